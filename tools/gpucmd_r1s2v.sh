timeout 300 python tools/prof_c1_small.py
timeout 300 python tools/time_c1.py
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "cp or c1 or c4 or c5 or core or parallel" > gpurun_out/s2v_tests.log 2>&1; tail -3 gpurun_out/s2v_tests.log
