timeout 900 python tools/c4_debug.py 2>&1 | tail -12
