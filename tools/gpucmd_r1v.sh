BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3.log 2>&1; cat gpurun_out/prof_c3.log | tail -40
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2b.log 2>&1; tail -25 gpurun_out/prof_c2b.log
