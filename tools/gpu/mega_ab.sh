run() { (cd $1 && env $3 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b_$2.log 2>&1); python -c "
import json
l=[x for x in open('/tmp/b_$2.log') if x.startswith('{')][-1]; d=json.loads(l); print('$2', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4))" || tail -3 /tmp/b_$2.log; }
for i in 1 2; do run . base X=1; run . mega_draft BASS_MEGA=2; run . mega_all BASS_MEGA=1; done
