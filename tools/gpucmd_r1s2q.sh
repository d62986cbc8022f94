timeout 300 python tools/prof_mlmv.py
REPS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:bt_gemm_kernel -s 5 -c 3 -o gpurun_out/s2q_mlmv python tools/prof_mlmv.py > gpurun_out/s2q_ncu.log 2>&1; tail -2 gpurun_out/s2q_ncu.log
