# full GPU suite + smoke + the default bench line (with cpu_baseline)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 "$@" > gpurun_out/tests_all.log 2>&1; echo tests rc=$?
grep -E "passed|failed" gpurun_out/tests_all.log | tail -3; grep -E "^FAILED" gpurun_out/tests_all.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench rc=$?
grep "^{" gpurun_out/bench_default.log | tail -1 > gpurun_out/bench_default.jsonl
python -c "
import json; d=json.load(open('gpurun_out/bench_default.jsonl')); print(d['value'], d['per_seq_ms_per_token'], d['e2e']['value'], d['roofline'].get('frac'), d['cpu_baseline']['value'], d['loop'], d['clocks'])"
