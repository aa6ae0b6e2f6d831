# C4 attention sweep (SURVEY 8(d) grid, all strategies, d_head 128 and 64)
timeout 2400 python tools/attn_bench.py all ragged,pad,split > gpurun_out/attn_sweep.jsonl 2> gpurun_out/attn_sweep.err; echo sweep rc=$? $(wc -l < gpurun_out/attn_sweep.jsonl)
tail -3 gpurun_out/attn_sweep.err
