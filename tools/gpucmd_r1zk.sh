timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1c.log 2>&1; cat gpurun_out/prof_c1c.log
BT_CP_GRAPH=0 timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1d.log 2>&1; cat gpurun_out/prof_c1d.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zk.log 2>&1; tail -3 gpurun_out/gpu_tests_zk.log
