timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zf.log 2>&1; tail -5 gpurun_out/gpu_tests_zf.log
timeout 1800 python bench.py > gpurun_out/bench_full4.json 2> gpurun_out/bench_full4.err; tail -3 gpurun_out/bench_full4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; cat gpurun_out/bench_ref2.json
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
