timeout 300 python tools/probe_write.py scatter > gpurun_out/maps_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_check_kernel|gather_rep_kernel" -c 2 -o gpurun_out/prof_gather2 python tools/probe_write.py scatter > gpurun_out/ncu_gather2.log 2>&1; tail -1 gpurun_out/ncu_gather2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"scatter_kernel|scatter_class_kernel" -c 2 -o gpurun_out/prof_scatter2 python tools/probe_write.py scatter > gpurun_out/ncu_scatter2.log 2>&1; tail -1 gpurun_out/ncu_scatter2.log
timeout 300 python tools/prof_detect.py > gpurun_out/detect_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"block_digest_kernel|block_match_kernel" -c 2 -o gpurun_out/prof_detect2 python tools/prof_detect.py > gpurun_out/ncu_detect2.log 2>&1; tail -1 gpurun_out/ncu_detect2.log
