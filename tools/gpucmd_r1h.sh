timeout 300 python tools/bench_eigx.py > gpurun_out/eigx2.jsonl 2> gpurun_out/eigx2.err; cat gpurun_out/eigx2.jsonl | head -12; tail -3 gpurun_out/eigx2.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -B5 "Error" gpurun_out/gpu_tests.log | head -30
timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err; tail -2 gpurun_out/bench_h.err; python -c "import json; d=json.load(open('gpurun_out/bench_h.json')); print(d.get('extras'))"
