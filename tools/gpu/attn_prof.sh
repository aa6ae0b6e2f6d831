set -x
export BASS_ATTN_MODE=stream
timeout 600 python tools/attn_bench.py all ragged,pad > gpurun_out/attn_bench.jsonl 2>&1; echo rc=$?
grep c2 gpurun_out/attn_bench.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_stream -s 2 -c 1 -o gpurun_out/prof_attn_q17 python tools/attn_bench.py one 64 17 8192 36 > gpurun_out/ncu_q17.log 2>&1; echo rc=$?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_stream -s 2 -c 1 -o gpurun_out/prof_attn_c2v python tools/attn_bench.py one 8 11 256 36 > gpurun_out/ncu_c2v.log 2>&1; echo rc=$?
