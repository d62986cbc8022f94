timeout 300 python tools/trace_tucker.py c3 2>&1 | grep -v Warning | tail -34
timeout 300 python tools/trace_tucker.py c2 2>&1 | grep -v Warning | tail -16
