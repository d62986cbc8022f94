timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1b.log 2>&1; cat gpurun_out/prof_c1b.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1b.csv python tools/prof_c1.py > gpurun_out/ncu_c1b.log 2>&1; tail -1 gpurun_out/ncu_c1b.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zi.log 2>&1; tail -3 gpurun_out/gpu_tests_zi.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_zi.json 2> gpurun_out/bench_zi.err; tail -1 gpurun_out/bench_zi.err
