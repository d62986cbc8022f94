timeout 300 python tools/prof_c1.py > gpurun_out/prof_c1.log 2>&1; cat gpurun_out/prof_c1.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python tools/prof_c1.py > gpurun_out/ncu_c1.log 2>&1; tail -1 gpurun_out/ncu_c1.log
timeout 900 python -m pytest tests/test_gpu_core.py -q -p no:cacheprovider > gpurun_out/gpu_core_zh.log 2>&1; tail -3 gpurun_out/gpu_core_zh.log
# plain run first (must exit 0), then one ncu --set full capture per map kernel
BT_GATHER_U=2 timeout 300 python tools/probe_write.py scatter > gpurun_out/maps_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -c 1 -o gpurun_out/prof_gather python tools/probe_write.py scatter > gpurun_out/ncu_gather.log 2>&1; tail -1 gpurun_out/ncu_gather.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter_kernel -c 2 -o gpurun_out/prof_scatter python tools/probe_write.py scatter > gpurun_out/ncu_scatter.log 2>&1; tail -1 gpurun_out/ncu_scatter.log
timeout 300 python tools/prof_detect.py > gpurun_out/detect_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"block_digest_kernel|block_match_kernel" -c 2 -o gpurun_out/prof_detect python tools/prof_detect.py > gpurun_out/ncu_detect.log 2>&1; tail -1 gpurun_out/ncu_detect.log
