timeout 1500 python bench.py > gpurun_out/s2x_bench.json 2> gpurun_out/s2x_bench.err; echo bench exit $?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/s2x_bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["roofline"]["frac"], d["clocks"], d["e2e"]["value"])
print(json.dumps(d.get("extras"), indent=0)[:3000])
print(json.dumps(d.get("extras_speedup_vs_cpu")))
PY
