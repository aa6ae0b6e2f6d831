run() { (env $2 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b.log 2>&1); python -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')][-1]; d=json.loads(l); print('$1', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4))"; }
for i in 1 2 3; do run base X=1; run dF2 BASS_SPLIT_OVERRIDE=8192x2048:2; done
