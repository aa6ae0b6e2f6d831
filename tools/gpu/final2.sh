timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo rc=$?
grep "^{" gpurun_out/bench_c2.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_seq_ms_per_token'], d['roofline']['frac'], d['roofline'].get('achieved_in_chain'), d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?; grep "^{" gpurun_out/bench_ref.log | tail -1 | cut -c1-300
