# device vs host loop at different acceptance regimes (per-step overhead vs finished-slot waste)
for a in 1.0 0.874 0.0; do for lp in device host; do
  timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --trace 0 --align $a --loop $lp 2>/dev/null | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('align $a $lp', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4), d['steps_per_generation'], round(d['ms_per_step'],2))"
done; done
