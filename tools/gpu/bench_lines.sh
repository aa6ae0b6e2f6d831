# bench lines (gpurun_out/line_*.jsonl): C2 device / host loop, C2 int8, C3 per strategy (+ sampled harness), C5
line() { name=$1; shift; timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/line_$name.log 2>&1
  grep "^{" gpurun_out/line_$name.log | tail -1 > gpurun_out/line_$name.jsonl
  python -c "
import json; d=json.load(open('gpurun_out/line_$name.jsonl')); print('$name', round(d['value'],1), {k: round(v,4) for k,v in d['per_seq_ms_per_token'].items()}, d.get('regular_decode_ms_per_token'), d['loop'])" 2>/dev/null || echo "$name failed"; }
line c2_device
line c2_host --loop host
line c2_int8 --dtype int8
for s in ragged pad split; do line c3_$s --config c3 --strategy $s; done
line c3_align --config c3 --align 0.874
line c5 --config c5
