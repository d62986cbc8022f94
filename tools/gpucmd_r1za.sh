timeout 300 python tools/bench_small_eig.py > gpurun_out/small_eig3.log 2>&1; cat gpurun_out/small_eig3.log | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['n'], d['kind'], 'jac %.3f ms' % d.get('jacobi_ms', -1), 'syevx %.3f ms' % d['syevx_ms'], 'jres %.1e' % d.get('jacobi_resid', -1))
"
