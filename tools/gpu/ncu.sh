# ncu: launch list of the speculative generation + --set full captures.  The
# device loop runs the same kernels inside conditional graph nodes, which ncu
# does not profile, so these use --loop host.
timeout 600 python bench.py --steps 1 --warmup 1 --trace 0 --no-cpu-baseline --save-traj /tmp/traj_c2.npy > gpurun_out/ncu_traj.log 2>&1; echo traj rc=$?
A="--profile-only --warmup 0 --trace 0 --load-traj /tmp/traj_c2.npy --loop host"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 8000 --csv --log-file gpurun_out/ncu_launches_c2.csv python bench.py $A > gpurun_out/ncu_launches.log 2>&1; echo launches rc=$?
python tools/ncu_summary.py gpurun_out/ncu_launches_c2.csv 40 > gpurun_out/ncu_launches_c2_summary.txt; head -20 gpurun_out/ncu_launches_c2_summary.txt
gzip -f gpurun_out/ncu_launches_c2.csv
full() { out=$1; rx=$2; skip=$3; shift 3
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s $skip -c 1 \
    -o gpurun_out/$out "$@" > gpurun_out/$out.log 2>&1; echo $out rc=$?; }
full ncu_gemm_qkv_verify 'gemm_tc_kernel<\(int\)128, \(int\)0' 3 python bench.py $A
full ncu_attn_c2 'attn_stream_kernel<\(int\)16, \(int\)128' 300 python bench.py $A
full ncu_gemm_prefill_qkv 'gemm_tc_kernel<\(int\)128, \(int\)0' 0 python tools/prefill_bench.py 8 128 1
full ncu_gemm_prefill_o 'gemm_tc_kernel<\(int\)256, \(int\)1' 0 python tools/prefill_bench.py 8 128 1
ls -la gpurun_out/*.ncu-rep
full ncu_attn_q33 'attn_stream_kernel<\(int\)64, \(int\)128' 0 python tools/attn_bench.py one 64 33 8192 36
