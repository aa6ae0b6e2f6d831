# INT8: parity tests (quant + device loop), C2 int8 bench, split sweep of the main projections
timeout 1200 python -m pytest tests/test_gpu_quant.py tests/test_gpu_loop.py -x -q -p no:cacheprovider > gpurun_out/int8_tests.log 2>&1; echo int8 tests rc=$?
tail -3 gpurun_out/int8_tests.log; grep -B3 -A20 "^E  " gpurun_out/int8_tests.log | head -40
run() { timeout 600 python bench.py --dtype int8 --steps 2 --warmup 2 --no-cpu-baseline --trace 0 "$@" 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['per_seq_ms_per_token']['all'],4), round(d['regular_decode_ms_per_token'],4), round(d['value'],1))"; }
run
for s in 1 4 6; do run --split 13824x4608:$s; done
for s in 2 3 4; do run --split 4608x4608:$s; done
for s in 2 4; do run --split 18432x4608:$s; done
for s in 2 3 4 8; do run --split 4608x18432:$s; done
