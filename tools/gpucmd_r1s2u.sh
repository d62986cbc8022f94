timeout 300 python tools/time_c1.py
BT_CP_SMALL=0 timeout 300 python tools/time_c1.py
