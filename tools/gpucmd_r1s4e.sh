timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
BT_BASIS_DEBUG=1 timeout 300 python tools/trace_tucker.py c3 > gpurun_out/trace_c3p.log 2>&1; grep -v Warn gpurun_out/trace_c3p.log | head -30
BT_PROJECTED=0 timeout 300 python tools/trace_tucker.py c3 > gpurun_out/trace_c3np.log 2>&1; grep "== c3" gpurun_out/trace_c3np.log
