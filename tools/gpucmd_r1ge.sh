timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_ge.log 2>&1; tail -8 gpurun_out/gpu_tests_ge.log
timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2j.log 2>&1; grep -A6 "total" gpurun_out/prof_c2j.log
timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3h.log 2>&1; grep -A3 "== " gpurun_out/prof_c3h.log
