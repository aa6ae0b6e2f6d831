timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo rc=$?
grep "^{" gpurun_out/bench_c2.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_seq_ms_per_token'], d['roofline']['frac'], d['roofline'].get('achieved_in_chain'), d['clocks'])"
