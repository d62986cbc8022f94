for v in 6 9; do BT_TREE_CFG=$v timeout 900 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras > gpurun_out/bench_gb$v.json 2> gpurun_out/bench_gb$v.err; echo "variant $v"; tail -1 gpurun_out/bench_gb$v.err; done
BT_TREE_CFG=9 timeout 600 python -m pytest tests/test_gpu_core.py tests/test_gpu_parallel.py -q -x -p no:cacheprovider 2>&1 | tail -2
