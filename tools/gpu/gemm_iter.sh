timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/g_tests1.log 2>&1; echo rc=$?
tail -15 gpurun_out/g_tests1.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/g_tests.log
timeout 300 python tools/gemm_micro.py 8,16,88,264 > gpurun_out/gemm_sk.jsonl 2>&1; echo rc=$?
BASS_GEMM_IMPL=split timeout 300 python tools/gemm_micro.py 8,16,88,264 > gpurun_out/gemm_split.jsonl 2>&1; echo rc=$?
paste -d'|' <(cut -c1-110 gpurun_out/gemm_sk.jsonl) <(cut -c60-110 gpurun_out/gemm_split.jsonl)
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench.log
