timeout 300 python tools/time_c1.py
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2w_tests.log 2>&1; tail -3 gpurun_out/s2w_tests.log
