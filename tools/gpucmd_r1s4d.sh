timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_gram.py > gpurun_out/prof_gram.log 2>&1; tail -15 gpurun_out/prof_gram.log
timeout 300 python tools/trace_tucker.py c3 > gpurun_out/trace_c3b.log 2>&1; grep -A4 "== c3" gpurun_out/trace_c3b.log
