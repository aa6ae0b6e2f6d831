# C4 attention sweep (all strategies, d_head 128 and 64) and C3 lines per strategy
timeout 1500 python tools/attn_bench.py all ragged,pad,split > gpurun_out/attn_sweep.jsonl 2> gpurun_out/attn_sweep.err; echo sweep rc=$? $(wc -l < gpurun_out/attn_sweep.jsonl)
for s in ragged pad split; do
  timeout 900 python bench.py --config c3 --steps 2 --warmup 2 --strategy $s --no-cpu-baseline > gpurun_out/bench_c3_$s.log 2>&1; echo c3 $s rc=$?
  grep "^{" gpurun_out/bench_c3_$s.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$s', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['mean_accepted'])"
done
