timeout 300 python tools/prof_c1.py 2>&1 | tail -4
BT_CP_SMALL=0 timeout 300 python tools/prof_c1.py 2>&1 | tail -2
timeout 300 python tools/trace_tucker.py c1 2>&1 | grep -v -i warn | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2t_tests.log 2>&1; tail -3 gpurun_out/s2t_tests.log
