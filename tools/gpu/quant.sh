# INT8 W8A8: GPU parity tests, then C2 bench lines bf16 vs int8
timeout 1200 python -m pytest tests/test_gpu_quant.py -x -q -p no:cacheprovider "$@" > gpurun_out/quant_tests.log 2>&1; echo quant tests rc=$?
tail -15 gpurun_out/quant_tests.log
for dt in int8; do
  timeout 900 python bench.py --steps 3 --warmup 3 --dtype $dt --no-cpu-baseline > gpurun_out/bench_c2_$dt.log 2>&1; echo bench $dt rc=$?
  grep "^{" gpurun_out/bench_c2_$dt.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$dt', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['mean_accepted'], d['roofline'].get('frac'), d['trace']['classes'].get('gemm',{}).get('union_ms'), d['trace']['generation_ms'])"
  tail -3 gpurun_out/bench_c2_$dt.log
done
