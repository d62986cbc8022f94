BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3b.log 2>&1; grep -v "^\[subspace" gpurun_out/prof_c3b.log | tail -30; grep "^\[subspace" gpurun_out/prof_c3b.log | head -20
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2c.log 2>&1; grep -v "^\[subspace" gpurun_out/prof_c2c.log | tail -14; grep "^\[subspace" gpurun_out/prof_c2c.log | head -12
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_w.log 2>&1; tail -15 gpurun_out/gpu_tests_w.log
