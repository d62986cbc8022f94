timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1e.log 2>&1; tail -3 gpurun_out/prof_c1e.log
BT_CP_GRAPH=0 timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1f.log 2>&1; cat gpurun_out/prof_c1f.log
