timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/g_tests1.log 2>&1; echo rc=$?
tail -3 gpurun_out/g_tests1.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo rc=$?
tail -15 gpurun_out/g_tests.log
timeout 300 python tools/gemm_micro.py 8,88,136,264 all packed > gpurun_out/gemm_pk.jsonl 2>&1; echo rc=$?
cut -c1-100 gpurun_out/gemm_pk.jsonl
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench.log
timeout 300 python tools/trace_gen.py > gpurun_out/trace.txt 2>&1; echo rc=$?
head -40 gpurun_out/trace.txt
