timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/s2y_bench.json 2> gpurun_out/s2y_bench.err; echo exit $?
python -c "
import json
d = json.loads(open('gpurun_out/s2y_bench.json').read().strip().splitlines()[-1])
e = d['extras']; print({k: e[k] for k in e if k.startswith('c1')})
"
timeout 300 python tools/time_c1.py
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,pstate --format=csv
