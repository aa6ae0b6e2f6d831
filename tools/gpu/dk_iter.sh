export BASS_GEMM_IMPL=dk
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/dk_tests1.log 2>&1; echo rc=$?
tail -5 gpurun_out/dk_tests1.log
timeout 300 python tools/gemm_micro.py 8,88,136 all packed > gpurun_out/gemm_dk.jsonl 2>&1; echo rc=$?
cut -c1-100 gpurun_out/gemm_dk.jsonl
for i in 1 2; do
BASS_GEMM_IMPL=dk timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench_dk.log 2>&1; echo rc=$?
python -c "
import json
l=[x for x in open('gpurun_out/bench_dk.log') if x.startswith('{')][-1]; d=json.loads(l)
print('dk', round(d['value'],1), d['per_seq_ms_per_token'])"
BASS_GEMM_IMPL=tc timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench_tc.log 2>&1; echo rc=$?
python -c "
import json
l=[x for x in open('gpurun_out/bench_tc.log') if x.startswith('{')][-1]; d=json.loads(l)
print('tc', round(d['value'],1), d['per_seq_ms_per_token'])"
done
