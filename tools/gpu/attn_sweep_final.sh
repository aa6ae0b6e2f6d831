timeout 1500 python tools/attn_bench.py all ragged,pad > gpurun_out/attn_sweep.jsonl 2> gpurun_out/attn_sweep.err; echo rc=$?; wc -l gpurun_out/attn_sweep.jsonl
