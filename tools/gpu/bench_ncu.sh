set -x
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --save-traj gpurun_out/traj.npy > gpurun_out/bench.log 2>&1; echo rc=$?
tail -c 2500 gpurun_out/bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_stream -s 2 -c 1 -o gpurun_out/prof_attn_c2v python tools/attn_bench.py one 8 11 256 36 > gpurun_out/ncu_c2v.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 40 -c 4 -o gpurun_out/prof_gemm python tools/gemm_micro.py 88 qkv,o,fc,proj > gpurun_out/ncu_gemm.log 2>&1; echo rc=$?
