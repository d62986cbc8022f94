timeout 300 python tools/trace_tucker.py c3 2>&1 | grep -v -i warn | grep -A6 "=="
timeout 300 python tools/trace_tucker.py c2 2>&1 | grep -v -i warn | grep -A6 "=="
BT_SUB_CHOLQR=0 timeout 300 python tools/trace_tucker.py c3 2>&1 | grep "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2o_tests.log 2>&1; tail -3 gpurun_out/s2o_tests.log
