timeout 300 python tools/prof_c2.py > gpurun_out/s2b_c2.log 2>&1; cat gpurun_out/s2b_c2.log
BT_BASIS_DEBUG=1 timeout 300 python tools/prof_c2.py > gpurun_out/s2b_c2dbg.log 2>&1; tail -60 gpurun_out/s2b_c2dbg.log
timeout 300 python tools/prof_c3.py > gpurun_out/s2b_c3.log 2>&1; cat gpurun_out/s2b_c3.log
BT_BASIS_DEBUG=1 timeout 300 python tools/prof_c3.py > gpurun_out/s2b_c3dbg.log 2>&1; tail -60 gpurun_out/s2b_c3dbg.log
