timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zp.log 2>&1; tail -15 gpurun_out/gpu_tests_zp.log
