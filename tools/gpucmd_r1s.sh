timeout 600 python -m pytest tests/test_gpu_detect.py tests/test_gpu_spd.py -q -p no:cacheprovider > gpurun_out/gpu_tests_s.log 2>&1; tail -15 gpurun_out/gpu_tests_s.log
timeout 600 python tools/probe_write.py > gpurun_out/probe_write.log 2>&1; cat gpurun_out/probe_write.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -2 gpurun_out/bench_s.err; python -c "import json;d=json.loads(open('gpurun_out/bench_s.json').read().strip().splitlines()[-1]);print(d.get('extras'))"
