BT_EIG_DEBUG=1 timeout 300 python tools/bench_eig.py > gpurun_out/eig2.jsonl 2> gpurun_out/eig2.err; cat gpurun_out/eig2.jsonl; grep -c sweep gpurun_out/eig2.err; head -60 gpurun_out/eig2.err
