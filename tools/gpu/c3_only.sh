timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo c3 rc=$?
grep "^{" gpurun_out/bench_c3.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['per_seq_ms_per_token']['all'], d['regular_decode_ms_per_token'])"
