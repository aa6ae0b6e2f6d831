timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -5 gpurun_out/t.log
for i in 1 2; do for v in 0 1; do
BASS_LNFUSE=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b$v.log 2>&1; python -c "
import json
l=[x for x in open('/tmp/b$v.log') if x.startswith('{')][-1]; d=json.loads(l); print('lnfuse=$v', round(d['value'],1), d['per_seq_ms_per_token'])" || tail -3 /tmp/b$v.log
done; done
