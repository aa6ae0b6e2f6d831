# sampling-path GPU tests and the C3 lines (PAD / SPLIT / RAGGED)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py tests/test_gpu_report.py -x -q -p no:cacheprovider 2>&1 | tail -3
for s in ragged pad split; do
  timeout 900 python bench.py --config c3 --steps 2 --warmup 2 --strategy $s --no-cpu-baseline > gpurun_out/bench_c3_$s.log 2>&1; echo c3 $s rc=$?
  grep "^{" gpurun_out/bench_c3_$s.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$s', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['mean_accepted'], d['trace']['classes'].get('gemm',{}).get('union_ms'), d['trace']['generation_ms'])"
done
