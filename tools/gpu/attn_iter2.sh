timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/it_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/it_tests.log
timeout 600 python tools/attn_bench.py c2 ragged > gpurun_out/attn_c2.jsonl 2>&1; echo rc=$?
cut -c1-160 gpurun_out/attn_c2.jsonl
