timeout 300 python tools/bench_small_eig.py > gpurun_out/small_eig2.log 2>&1; cat gpurun_out/small_eig2.log | tail -8
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3e.log 2>&1; grep -A8 "== " gpurun_out/prof_c3e.log | head -20
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2f.log 2>&1; grep -A6 "total" gpurun_out/prof_c2f.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_z.log 2>&1; tail -15 gpurun_out/gpu_tests_z.log
