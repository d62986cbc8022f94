timeout 300 python tools/trace_matvec.py c2 2>&1 | grep -v -i warn | head -8
BT_BLR_ROWS=0 timeout 300 python tools/trace_matvec.py c2 2>&1 | grep "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2n_tests.log 2>&1; tail -3 gpurun_out/s2n_tests.log
