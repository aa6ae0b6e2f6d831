# round-2 ncu evidence on the speculative generation itself (device loop): launch list + full captures
# (the device loop runs the same kernels inside conditional graph nodes, which ncu does not profile: the captures use --loop host)
timeout 600 python bench.py --steps 1 --warmup 1 --trace 0 --no-cpu-baseline --save-traj /tmp/traj_c2.npy > gpurun_out/r2_traj.log 2>&1; echo traj rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 8000 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --profile-only --warmup 0 --trace 0 \
  --load-traj /tmp/traj_c2.npy --loop host > gpurun_out/r2_launches_c2.log 2>&1
echo launches rc=$?
python tools/ncu_summary.py gpurun_out/r2_launches_c2.csv 40 > gpurun_out/r2_launches_c2_summary.txt; head -45 gpurun_out/r2_launches_c2_summary.txt
gzip -f gpurun_out/r2_launches_c2.csv
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_tc_kernel<\(int\)128, \(int\)0' -s 3 -c 1 -o gpurun_out/r2_gemm_qkv_verify python bench.py --profile-only --warmup 0 \
  --trace 0 --load-traj /tmp/traj_c2.npy --loop host > gpurun_out/r2_gemm_full.log 2>&1
echo gemm full rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:attn_stream_kernel<\(int\)16, \(int\)128' -s 300 -c 1 -o gpurun_out/r2_attn_c2 python bench.py --profile-only --warmup 0 \
  --trace 0 --load-traj /tmp/traj_c2.npy --loop host > gpurun_out/r2_attn_full.log 2>&1
echo attn full rc=$?
ls -la gpurun_out/*.ncu-rep
