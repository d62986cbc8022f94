timeout 300 python tools/prof_gram.py > gpurun_out/s2c_gram.log 2>&1; cat gpurun_out/s2c_gram.log
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:bt_gemm_kernel -c 4 -o gpurun_out/s2c_gram python tools/prof_gram.py > gpurun_out/s2c_ncu.log 2>&1; tail -3 gpurun_out/s2c_ncu.log
