timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 2500 --log-file gpurun_out/c3_launches.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --kernel-events 0 > gpurun_out/c3_ncu.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/c3_launches.csv 30 > gpurun_out/c3_launches_summary.txt; head -32 gpurun_out/c3_launches_summary.txt
