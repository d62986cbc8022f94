BT_BASIS_DEBUG=0 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3g.log 2>&1; grep -A4 "== " gpurun_out/prof_c3g.log | head -12
timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2h.log 2>&1; grep -A4 "total" gpurun_out/prof_c2h.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zc.log 2>&1; tail -5 gpurun_out/gpu_tests_zc.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_zc.json 2> gpurun_out/bench_zc.err; tail -1 gpurun_out/bench_zc.err; python -c "import json;d=json.loads(open('gpurun_out/bench_zc.json').read().strip().splitlines()[-1]);print(d.get('extras'))"
