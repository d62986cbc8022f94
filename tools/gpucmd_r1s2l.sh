timeout 300 python tools/trace_tucker.py c3 2>&1 | grep "=="
timeout 300 python tools/trace_tucker.py c2 2>&1 | grep "=="
BT_BASIS_DEBUG=1 timeout 300 python tools/prof_c3.py > gpurun_out/s2l_c3dbg.log 2>&1; tail -30 gpurun_out/s2l_c3dbg.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2l_tests.log 2>&1; tail -3 gpurun_out/s2l_tests.log
