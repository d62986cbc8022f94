timeout 300 python tools/trace_matvec.py c4 2>&1 | grep -v -i warn | head -8
BT_GEMM_FORCE=w timeout 300 python tools/trace_matvec.py c4 2>&1 | grep -v -i warn | head -8
