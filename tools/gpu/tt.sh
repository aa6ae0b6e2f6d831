timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -x -q > gpurun_out/t1.log 2>&1; echo rc=$?; tail -2 gpurun_out/t1.log
timeout 300 python tools/gemm_micro.py 136,152,176,200 qkv,o,fc,proj,d_qkv packed > gpurun_out/gemm_tt.jsonl 2>&1; echo rc=$?
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/bn.log 2>&1; python -c "
import json
l=[x for x in open('/tmp/bn.log') if x.startswith('{')][-1]; d=json.loads(l); print('new', round(d['value'],1), d['per_seq_ms_per_token'])"; done
