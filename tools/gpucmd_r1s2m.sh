timeout 1500 python bench.py > gpurun_out/s2m_bench.json 2> gpurun_out/s2m_bench.err; echo bench exit $?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/s2m_bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["roofline"]["frac"], d["clocks"])
print(json.dumps(d.get("extras"), indent=0)[:2500])
PY
