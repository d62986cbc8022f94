timeout 600 python -m pytest tests/test_gpu_detect.py tests/test_gpu_core.py -q -p no:cacheprovider > gpurun_out/gpu_tests_t.log 2>&1; tail -5 gpurun_out/gpu_tests_t.log
timeout 600 python tools/probe_write.py > gpurun_out/probe_write2.log 2>&1; cat gpurun_out/probe_write2.log
timeout 600 python tools/prof_detect.py > gpurun_out/prof_detect.log 2>&1; cat gpurun_out/prof_detect.log
