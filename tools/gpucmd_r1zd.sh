timeout 600 python tools/c4_gpu_fit.py 2>&1 | tail -6
