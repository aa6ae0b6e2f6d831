# INT8 split tuning: baseline and combinations (main-model projection shapes)
run() { timeout 600 python bench.py --dtype int8 --steps 2 --warmup 2 --no-cpu-baseline --trace 0 "$@" 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('int8 [$*]', round(d['per_seq_ms_per_token']['all'],4), round(d['regular_decode_ms_per_token'],4), round(d['value'],1))"; }
run
run --split 18432x4608:2
run --split 18432x4608:2 --split 4608x4608:4 --split 4608x18432:4
run --split 18432x4608:2 --split 4608x4608:4 --split 4608x18432:4 --split 13824x4608:4
run --split 18432x4608:2 --split 4608x4608:4 --split 4608x18432:3
