# Q dimension tree: GPU tests, plain C5 bench, launch list, ncu --set full of the mode-1 tree kernel and the Q GEMM
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/c5_q.json 2> gpurun_out/c5_q.err || exit 1
tail -3 gpurun_out/c5_q.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5q.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_launch_c5q.log 2>&1; tail -1 gpurun_out/ncu_launch_c5q.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_p_ws_kernel -s 3 -c 1 -o gpurun_out/prof_c5q_tree python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_c5q_tree.log 2>&1; tail -1 gpurun_out/ncu_c5q_tree.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:bt_gemm_kernel<GemmCfg<128, 64, 16, 2, 2, 4, false, false" -s 3 -c 1 -o gpurun_out/prof_c5q_qgemm python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras > gpurun_out/ncu_c5q_qgemm.log 2>&1; tail -1 gpurun_out/ncu_c5q_qgemm.log
