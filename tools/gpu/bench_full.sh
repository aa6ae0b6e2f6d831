timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo rc=$?
grep "^{" gpurun_out/bench_c2.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k in ['value','per_seq_ms_per_token','e2e','roofline','attention_roofline','cpu_baseline','clocks']: print(k, d.get(k))"
