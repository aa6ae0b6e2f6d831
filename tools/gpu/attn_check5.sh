timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -1 gpurun_out/t.log
for t in _ab/head .; do echo "== $t"; (cd $t && for a in "8 17 182 36" "8 25 276 36" "64 17 8192 36" "8 17 2048 36"; do timeout 120 python tools/attn_bench.py one $a 2>&1 | tail -1 | cut -c1-125; done); done
run() { (cd $1 && env $3 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b_$2.log 2>&1); python -c "
import json
l=[x for x in open('/tmp/b_$2.log') if x.startswith('{')][-1]; d=json.loads(l); print('$2', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4))"; }
run _ab/head head X=1; run . new X=1
