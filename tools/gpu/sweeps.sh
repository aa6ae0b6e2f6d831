# C4 attention sweep, INT8 split tuning, device vs host loop across acceptance regimes
timeout 2400 python tools/attn_bench.py all ragged,pad,split > gpurun_out/attn_sweep.jsonl 2> gpurun_out/attn_sweep.err; echo sweep rc=$? $(wc -l < gpurun_out/attn_sweep.jsonl)
run() { timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --trace 0 "$@" 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$*]', round(d['per_seq_ms_per_token']['all'],4), round(d['regular_decode_ms_per_token'],4), round(d['value'],1))"; }
run --dtype int8
for s in 1 2 4; do run --dtype int8 --split 18432x4608:$s; done
for a in 1.0 0.874 0.0; do for lp in device host; do run --align $a --loop $lp; done; done
# draft-model split counts in the real chain (profiles/r2/draft_split_sweep.txt: the defaults are the optimum)
for ov in 2048x2048:4 2048x8192:4 8192x2048:2 6144x2048:2 6144x2048:8; do run --split $ov; done
