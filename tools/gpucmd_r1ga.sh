timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; tail -1 gpurun_out/bench_ga.err
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_ga.log 2>&1; tail -3 gpurun_out/gpu_tests_ga.log
