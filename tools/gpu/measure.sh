set -x
timeout 600 python bench.py --steps 3 --warmup 3 --save-traj gpurun_out/traj.npy > gpurun_out/bench_c2.log 2>&1; echo rc=$?
timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --profile-only --warmup 0 --load-traj gpurun_out/traj.npy --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1; echo rc=$?
python tools/ncu_summary.py gpurun_out/launches.csv 45 > gpurun_out/launches_summary.txt; gzip -f gpurun_out/launches.csv
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 6 -c 1 -o gpurun_out/prof_gemm_qkv88 python tools/gemm_micro.py 88 qkv packed > gpurun_out/ncu_g1.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 6 -c 1 -o gpurun_out/prof_gemm_fc8 python tools/gemm_micro.py 8 fc packed > gpurun_out/ncu_g2.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_stream -s 2 -c 1 -o gpurun_out/prof_attn_c2v python tools/attn_bench.py one 8 11 256 36 > gpurun_out/ncu_a1.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_stream -s 2 -c 1 -o gpurun_out/prof_attn_c4 python tools/attn_bench.py one 64 9 8192 36 > gpurun_out/ncu_a2.log 2>&1; echo rc=$?
