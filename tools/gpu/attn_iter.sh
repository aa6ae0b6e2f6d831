set -x
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/it_tests1.log 2>&1; echo rc=$?
tail -3 gpurun_out/it_tests1.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/it_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/it_tests.log
timeout 600 python tools/attn_bench.py all ragged > gpurun_out/attn_bench.jsonl 2>&1; echo rc=$?
cat gpurun_out/attn_bench.jsonl | cut -c1-200
