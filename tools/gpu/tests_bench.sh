# GPU box: full -m gpu suite, smoke, one short C2 bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 "$@" > gpurun_out/tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|rel err" gpurun_out/tests.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench rc=$?
grep "^{" gpurun_out/bench_c2.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['per_seq_ms_per_token'], d['e2e']['value'], d['clocks'])"
