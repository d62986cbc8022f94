timeout 300 python tools/bench_eigx.py > gpurun_out/eigx.jsonl 2> gpurun_out/eigx.err; cat gpurun_out/eigx.jsonl; tail -3 gpurun_out/eigx.err
timeout 300 python tools/dmma_occupancy.py > gpurun_out/dmma_occ.jsonl 2>&1; cat gpurun_out/dmma_occ.jsonl
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; tail -2 gpurun_out/bench_f.err; python -c "import json; d=json.load(open('gpurun_out/bench_f.json')); print(d.get('extras'))"
