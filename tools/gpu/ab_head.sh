run() { # dir tag
  (cd $1 && timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b_$2.log 2>&1)
  python -c "
import json
l=[x for x in open('/tmp/b_$2.log') if x.startswith('{')][-1]; d=json.loads(l)
print('$2', round(d['value'],1), {k: round(v,3) for k,v in d['per_seq_ms_per_token'].items()})"
}
for i in 1 2; do run _ab/head head; run . new; done
