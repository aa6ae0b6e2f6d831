# C3 lines per attention strategy (PAD / SPLIT / RAGGED), BASELINE configs[2]
for s in ragged pad split; do
  timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --strategy $s --no-cpu-baseline > gpurun_out/bench_c3_$s.log 2>&1; echo c3 $s rc=$?
  grep "^{" gpurun_out/bench_c3_$s.log | tail -1 > gpurun_out/bench_c3_$s.jsonl
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_$s.jsonl')); print('$s', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['mean_accepted'], d['attention_roofline'].get('in_chain_ms_per_generation'), d['trace']['generation_ms'])"
done
