for v in 1 0 1 0; do
BASS_PACK=$v timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench_pack$v.log 2>&1
python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_pack$v.log') if x.startswith('{')][-1]; d=json.loads(l)
print('pack=$v', round(d['value'],1), d['per_seq_ms_per_token'])"
done
