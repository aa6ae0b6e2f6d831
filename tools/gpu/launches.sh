# ncu launch lists (serialised, cold) of one profiled C2 generation: usage launches.sh <dtype> [count] [skip]
DT=${1:-bf16}; N=${2:-3000}; SKIP=${3:-0}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'gemm_tc|attn|quant_ctx|quant_amax|qkv_quant|ln_quant|embed|layernorm|row_stats|finalize|draft|cl_|combine|head_gather' \
  -s $SKIP -c $N --csv \
  --log-file gpurun_out/launches_$DT.csv python bench.py --profile-only --warmup 0 --trace 0 --dtype $DT > gpurun_out/launches_$DT.log 2>&1
echo ncu $DT rc=$?
python tools/ncu_summary.py gpurun_out/launches_$DT.csv 40 > gpurun_out/launches_${DT}_summary.txt 2>&1; head -42 gpurun_out/launches_${DT}_summary.txt
