timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zm.log 2>&1; tail -3 gpurun_out/gpu_tests_zm.log
timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1g.log 2>&1; tail -2 gpurun_out/prof_c1g.log
timeout 600 python tools/probe_write.py > gpurun_out/probe_write8.log 2>&1; cat gpurun_out/probe_write8.log
timeout 600 python tools/prof_detect.py > gpurun_out/prof_detect7.log 2>&1; cat gpurun_out/prof_detect7.log
