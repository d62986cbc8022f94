timeout 1500 python bench.py > gpurun_out/s3d_bench.json 2> gpurun_out/s3d_bench.err; echo bench exit $?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/s3d_bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["roofline"]["frac"], d["clocks"], d["e2e"]["value"], d["cpu_baseline"]["value"])
e = d["extras"]; print({k: round(v, 3) if isinstance(v, float) else v for k, v in e.items()})
print(d.get("extras_speedup_vs_cpu"))
PY
