timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/s3c.json 2>/dev/null
python -c "
import json
d = json.loads(open('gpurun_out/s3c.json').read().strip().splitlines()[-1])
e = d['extras']; print({k: round(e[k],2) for k in e if k.startswith('c4') or k.startswith('c1_cp')})
"
timeout 900 python bench.py --no-cpu --steps 2 --warmup 1 > gpurun_out/s3c2.json 2>/dev/null
python -c "
import json
d = json.loads(open('gpurun_out/s3c2.json').read().strip().splitlines()[-1])
e = d['extras']; print({k: round(e[k],2) for k in e if k.startswith('c4') or k.startswith('c1_cp')})
"
