# session-2 state check: GPU parity suite, smoke, full bench (both arms), launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2a_gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s2a_gpu_tests.log 2>&1; tail -15 gpurun_out/s2a_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; tail -2 gpurun_out/s2a_smoke.log
timeout 1500 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; echo bench exit $?; tail -c 3000 gpurun_out/s2a_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2a_ref.json 2> gpurun_out/s2a_ref.err; echo ref exit $?; cat gpurun_out/s2a_ref.json
