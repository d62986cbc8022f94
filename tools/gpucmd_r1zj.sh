timeout 300 python tools/bench_pinv.py 2>&1 | tail -14
