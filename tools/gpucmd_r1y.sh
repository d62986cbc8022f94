timeout 300 python tools/bench_small_eig.py > gpurun_out/small_eig.log 2>&1; cat gpurun_out/small_eig.log | tail -8
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3d.log 2>&1; grep -A8 "== " gpurun_out/prof_c3d.log | head -20; grep -c subspace gpurun_out/prof_c3d.log
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2e.log 2>&1; grep -A6 "total" gpurun_out/prof_c2e.log
