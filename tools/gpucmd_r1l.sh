BT_EIG_DEBUG=1 timeout 300 python tools/bench_eigx.py > gpurun_out/eigx6.jsonl 2> gpurun_out/eigx6.err; grep syevx gpurun_out/eigx6.err | awk 'NR%2==0' | head -12
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log; grep -B10 "Error" gpurun_out/gpu_tests.log | head -60
timeout 900 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; tail -2 gpurun_out/bench_l.err; python -c "import json; d=json.load(open('gpurun_out/bench_l.json')); print(d.get('extras'))"
export DIMS=2048,2048,256,64
timeout 120 python tools/tune_gemm.py > gpurun_out/prof_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_p_kernel -c 1 -o gpurun_out/prof_tree_v6 python tools/tune_gemm.py > gpurun_out/ncu_tree2.log 2>&1; tail -2 gpurun_out/ncu_tree2.log
