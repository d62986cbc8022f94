timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zr.log 2>&1; tail -3 gpurun_out/gpu_tests_zr.log
timeout 1800 python bench.py > gpurun_out/bench_full5.json 2> gpurun_out/bench_full5.err; tail -2 gpurun_out/bench_full5.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke2.log 2>&1; tail -1 gpurun_out/smoke2.log
