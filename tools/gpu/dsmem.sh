timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_decode.py -x -q > gpurun_out/t1.log 2>&1; echo rc=$?
tail -3 gpurun_out/t1.log
timeout 300 python tools/gemm_micro.py 8,88,136 all packed > gpurun_out/gemm_dsm.jsonl 2>&1; echo rc=$?
for i in 1 2; do (cd _ab/head && timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/bh.log 2>&1; python -c "
import json
l=[x for x in open('/tmp/bh.log') if x.startswith('{')][-1]; d=json.loads(l); print('head', round(d['value'],1), d['per_seq_ms_per_token'])")
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/bn.log 2>&1; python -c "
import json
l=[x for x in open('/tmp/bn.log') if x.startswith('{')][-1]; d=json.loads(l); print('new', round(d['value'],1), d['per_seq_ms_per_token'])"
done
