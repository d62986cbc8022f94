timeout 300 python tools/prof_c2.py > gpurun_out/s2d_c2.log 2>&1; cat gpurun_out/s2d_c2.log
timeout 300 python tools/prof_c3.py > gpurun_out/s2d_c3.log 2>&1; cat gpurun_out/s2d_c3.log
BT_BASIS_DEBUG=1 timeout 300 python tools/prof_c2.py > gpurun_out/s2d_c2dbg.log 2>&1
BT_BASIS_DEBUG=1 timeout 300 python tools/prof_c3.py > gpurun_out/s2d_c3dbg.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2d_tests.log 2>&1; tail -15 gpurun_out/s2d_tests.log
