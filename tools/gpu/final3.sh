timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo rc=$?
grep "^{" gpurun_out/bench_c2.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_seq_ms_per_token']['all'], d['roofline']['achieved_in_chain'], d['e2e']['value'], d['clocks'])"
timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo c3 rc=$?
grep "^{" gpurun_out/bench_c3.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['per_seq_ms_per_token']['all'])"
