# attention pipeline stamps (debug build): draft shape and verify shape
python tools/attn_bench.py one 8 1 182 16 2>&1 | tail -18
python tools/attn_bench.py one 8 11 182 36 2>&1 | tail -18
