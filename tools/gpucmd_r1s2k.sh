timeout 300 python tools/prof_gram.py
BT_GEMM_NO_MID=1 timeout 300 python tools/prof_gram.py | grep ttm
timeout 300 python tools/trace_tucker.py c3 2>&1 | grep "=="
timeout 300 python tools/trace_tucker.py c2 2>&1 | grep "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2k_tests.log 2>&1; tail -3 gpurun_out/s2k_tests.log
