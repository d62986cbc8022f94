set -x
timeout 600 python -m pytest tests/test_gpu_reps.py -x -q -p no:cacheprovider > gpurun_out/gpu_reps.log 2>&1; tail -15 gpurun_out/gpu_reps.log
for T in 0 1 2 3 4 5; do BT_TREE_CFG=$T timeout 120 python tools/tune_gemm.py >> gpurun_out/tune.jsonl 2>>gpurun_out/tune.err; done
for G in 0 1 2 3 4; do BT_GEMM_CFG=$G timeout 120 python tools/tune_gemm.py >> gpurun_out/tune.jsonl 2>>gpurun_out/tune.err; done
cat gpurun_out/tune.jsonl
export DIMS=2048,2048,256,64
timeout 120 python tools/tune_gemm.py > gpurun_out/prof_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_p_kernel -c 1 -o gpurun_out/prof_tree python tools/tune_gemm.py > gpurun_out/ncu_tree.log 2>&1
tail -3 gpurun_out/ncu_tree.log
unset DIMS
timeout 600 python bench.py --no-e2e --no-cpu --steps 2 --warmup 1 > gpurun_out/bench_extras.json 2> gpurun_out/bench_extras.err; tail -3 gpurun_out/bench_extras.err
