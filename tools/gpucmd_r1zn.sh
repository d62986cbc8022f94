timeout 600 python -m pytest tests/test_gpu_detect.py -q -p no:cacheprovider > gpurun_out/gpu_detect_zn.log 2>&1; tail -2 gpurun_out/gpu_detect_zn.log
timeout 600 python tools/prof_detect.py > gpurun_out/prof_detect8.log 2>&1; cat gpurun_out/prof_detect8.log
