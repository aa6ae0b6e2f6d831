timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -2 gpurun_out/t.log
for t in _ab/head .; do (cd $t && timeout 600 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --kernel-events 0 > /tmp/c3.log 2>&1); grep "^{" /tmp/c3.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value'],1), d['per_seq_ms_per_token']['all'], d['regular_decode_ms_per_token'])"; done
