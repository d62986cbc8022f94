timeout 900 python -m pytest tests/test_gpu_era.py -q -p no:cacheprovider > gpurun_out/gpu_era.log 2>&1; tail -30 gpurun_out/gpu_era.log
