# C2 / C3 bench lines: device loop (default) vs host loop
for lp in device host; do
  timeout 900 python bench.py --steps 3 --warmup 3 --loop $lp --no-cpu-baseline > gpurun_out/bench_c2_$lp.log 2>&1; echo c2 $lp rc=$?
  grep "^{" gpurun_out/bench_c2_$lp.log | tail -1 > gpurun_out/bench_c2_$lp.jsonl
  python -c "
import json; d=json.load(open('gpurun_out/bench_c2_$lp.jsonl')); print('c2 $lp', round(d['value'],1), d['per_seq_ms_per_token'], d['e2e']['value'], d['host_ms_per_generation'], d['loop'], d['roofline']['frac'], d['gpu_launches'])"
  tail -2 gpurun_out/bench_c2_$lp.log | grep -v "^{"
done
timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_device.log 2>&1; echo c3 rc=$?
grep "^{" gpurun_out/bench_c3_device.log | tail -1 > gpurun_out/bench_c3_device.jsonl
python -c "
import json; d=json.load(open('gpurun_out/bench_c3_device.jsonl')); print('c3 device', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['host_ms_per_generation'], d['loop'])"
