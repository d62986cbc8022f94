BT_EIG_DEBUG=1 timeout 600 python tools/bench_eigx.py 2>&1 | tail -40
timeout 300 python tools/trace_tucker.py c3 2>&1 | grep -v -i Warn | tail -34
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2j_tests.log 2>&1; tail -3 gpurun_out/s2j_tests.log
