timeout 300 python tools/prof_c2.py 2>&1 | head -4
timeout 300 python tools/prof_c3.py 2>&1 | grep -A4 "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2h_tests.log 2>&1; tail -3 gpurun_out/s2h_tests.log
