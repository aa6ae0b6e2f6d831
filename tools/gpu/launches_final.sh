timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernel-events 0 --save-traj gpurun_out/traj.npy > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --warmup 0 --load-traj gpurun_out/traj.npy --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/launches.csv 45 > gpurun_out/launches_summary.txt; head -3 gpurun_out/launches_summary.txt
