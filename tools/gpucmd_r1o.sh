BT_EIG_DEBUG=1 timeout 300 python tools/prof_c2.py 2>&1 | tail -30
