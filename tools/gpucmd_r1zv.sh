timeout 300 python tools/bench_pinv.py 2>&1 | tail -12
timeout 300 python tools/prof_c4.py > gpurun_out/prof_c4b.log 2>&1; cat gpurun_out/prof_c4b.log
timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1j.log 2>&1; tail -2 gpurun_out/prof_c1j.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zv.log 2>&1; tail -4 gpurun_out/gpu_tests_zv.log
