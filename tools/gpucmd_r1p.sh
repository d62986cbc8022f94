BT_EIG_DEBUG=1 timeout 300 python tools/prof_c2.py 2>&1 | tail -12
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -B10 "Error" gpurun_out/gpu_tests.log | head -60
timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/bench_p.json 2> gpurun_out/bench_p.err; python -c "import json; d=json.load(open('gpurun_out/bench_p.json')); print(d.get('extras'))"
