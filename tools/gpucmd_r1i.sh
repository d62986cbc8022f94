BT_EIG_DEBUG=1 timeout 300 python tools/bench_eigx.py > gpurun_out/eigx3.jsonl 2> gpurun_out/eigx3.err; grep syevx gpurun_out/eigx3.err | head -20
for T in 6; do BT_TREE_CFG=$T timeout 120 python tools/tune_gemm.py >> gpurun_out/tune3.jsonl 2>>gpurun_out/tune3.err; done; cat gpurun_out/tune3.jsonl
