timeout 300 python tools/prof_mlmv.py
BT_GEMM_PERSIST=0 timeout 300 python tools/prof_mlmv.py
timeout 300 python tools/trace_matvec.py c4 2>&1 | grep -v -i warn | head -6
timeout 300 python tools/prof_gram.py
timeout 300 python tools/trace_tucker.py c3 2>&1 | grep "=="
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2r_tests.log 2>&1; tail -3 gpurun_out/s2r_tests.log
