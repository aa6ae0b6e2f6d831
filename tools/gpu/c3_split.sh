# C3 in-chain split-count sweep for the main projections (per-model override)
run() { timeout 600 python bench.py --config c3 --steps 1 --warmup 2 --no-cpu-baseline --trace 0 "$@" 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['per_seq_ms_per_token']['all'],4), round(d['regular_decode_ms_per_token'],4))"; }
run
for s in 2 3 4 5 8; do run --split 20480x5120:$s; done
for s in 1 4 5; do run --split 15360x5120:$s; done
for s in 4 8; do run --split 5120x5120:$s; done
for s in 4 8; do run --split 5120x20480:$s; done
