timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s3b_tests.log 2>&1; tail -3 gpurun_out/s3b_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err; echo bench exit $?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/s3b_bench.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["roofline"]["frac"], d["clocks"], d["e2e"]["value"], d["cpu_baseline"]["value"])
e = d["extras"]; print({k: round(v, 3) if isinstance(v, float) else v for k, v in e.items()})
print(d.get("extras_speedup_vs_cpu"))
PY
