timeout 600 python -m pytest tests/test_gpu_detect.py tests/test_gpu_core.py -q -p no:cacheprovider > gpurun_out/gpu_tests_y.log 2>&1; tail -3 gpurun_out/gpu_tests_y.log
timeout 600 python tools/probe_write.py > gpurun_out/probe_write7.log 2>&1; cat gpurun_out/probe_write7.log
timeout 600 python tools/prof_detect.py > gpurun_out/prof_detect6.log 2>&1; cat gpurun_out/prof_detect6.log
