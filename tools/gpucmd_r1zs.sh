timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1h.log 2>&1; tail -3 gpurun_out/prof_c1h.log
BT_CP_SMALL=0 timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1i.log 2>&1; tail -1 gpurun_out/prof_c1i.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zs.log 2>&1; tail -12 gpurun_out/gpu_tests_zs.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke3.log 2>&1; tail -1 gpurun_out/smoke3.log
