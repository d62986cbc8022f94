timeout 300 python tools/prof_c4.py > gpurun_out/prof_c4.log 2>&1; cat gpurun_out/prof_c4.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python tools/prof_c4.py > gpurun_out/ncu_c4.log 2>&1; tail -1 gpurun_out/ncu_c4.log
