for T in 1 5 6 7 8; do BT_TREE_CFG=$T timeout 120 python tools/tune_gemm.py >> gpurun_out/tune2.jsonl 2>>gpurun_out/tune2.err; done
for G in 4 5 6 7 2; do BT_TREE_CFG=1 BT_GEMM_CFG=$G timeout 120 python tools/tune_gemm.py >> gpurun_out/tune2.jsonl 2>>gpurun_out/tune2.err; done
for T in 1 6; do DIMS=255,255,255,16 BT_TREE_CFG=$T timeout 120 python tools/tune_gemm.py >> gpurun_out/tune2.jsonl 2>>gpurun_out/tune2.err; done
cat gpurun_out/tune2.jsonl
