timeout 300 python tools/bench_small_eig.py > gpurun_out/small_eig4.log 2>&1; cat gpurun_out/small_eig4.log | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['kind'], 'jac %.3f ms' % d.get('jacobi_ms', -1), 'syevx %.3f ms' % d['syevx_ms'], 'jres %.1e' % d.get('jacobi_resid', -1), 'jorth %.1e' % d.get('jacobi_orth', -1))
"
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3f.log 2>&1; grep -A4 "== " gpurun_out/prof_c3f.log | head -12
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2g.log 2>&1; grep -A4 "total" gpurun_out/prof_c2g.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_zb.log 2>&1; tail -5 gpurun_out/gpu_tests_zb.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_zb.json 2> gpurun_out/bench_zb.err; tail -1 gpurun_out/bench_zb.err
