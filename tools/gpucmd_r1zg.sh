# plain run first (must exit 0), then one ncu --set full capture per map kernel
BT_GATHER_U=2 timeout 300 python tools/probe_write.py scatter > gpurun_out/maps_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -c 1 -o gpurun_out/prof_gather python tools/probe_write.py scatter > gpurun_out/ncu_gather.log 2>&1; tail -1 gpurun_out/ncu_gather.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scatter_kernel -c 2 -o gpurun_out/prof_scatter python tools/probe_write.py scatter > gpurun_out/ncu_scatter.log 2>&1; tail -1 gpurun_out/ncu_scatter.log
timeout 300 python tools/prof_detect.py > gpurun_out/detect_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"block_digest_kernel|block_match_kernel" -c 2 -o gpurun_out/prof_detect python tools/prof_detect.py > gpurun_out/ncu_detect.log 2>&1; tail -1 gpurun_out/ncu_detect.log
