timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo rc=$?
grep "^{" gpurun_out/bench_c3.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'])"
