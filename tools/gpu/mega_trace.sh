BASS_MEGA=1 timeout 300 python tools/trace_gen.py > gpurun_out/trace_mega.txt 2>&1; echo rc=$?
head -30 gpurun_out/trace_mega.txt
BASS_MEGA=1 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench_mega.log 2>&1; echo rc=$?
python -c "
import json
l=[x for x in open('gpurun_out/bench_mega.log') if x.startswith('{')][-1]; d=json.loads(l); print('mega', round(d['value'],1), d['per_seq_ms_per_token'])"
