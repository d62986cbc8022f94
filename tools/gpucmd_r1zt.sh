for t in 128 256 512 1024; do BT_CP_SMALL_THREADS=$t timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1_t$t.log 2>&1; echo "threads $t"; tail -1 gpurun_out/prof_c1_t$t.log; done
timeout 300 ncu --set full --clock-control none -k regex:cp_small_kernel -c 1 -o gpurun_out/prof_cp_small python tools/prof_c1.py > gpurun_out/ncu_cp_small.log 2>&1; tail -1 gpurun_out/ncu_cp_small.log
