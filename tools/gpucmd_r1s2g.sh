timeout 300 python tools/bench_prims.py 2>&1 | head -8
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2g_tests.log 2>&1; tail -5 gpurun_out/s2g_tests.log
timeout 300 python tools/prof_c2.py 2>&1 | head -4
timeout 300 python tools/prof_c3.py 2>&1 | grep -A3 "=="
