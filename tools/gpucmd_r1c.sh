timeout 300 python tools/bench_eig.py > gpurun_out/eig.jsonl 2> gpurun_out/eig.err; cat gpurun_out/eig.jsonl; tail -3 gpurun_out/eig.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -25 gpurun_out/gpu_tests.log
timeout 900 python bench.py --no-e2e --steps 3 --warmup 2 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; tail -3 gpurun_out/bench_c.err; python -c "import json; d=json.load(open('gpurun_out/bench_c.json')); print(d['value'], d['roofline'], d.get('extras'))"
