timeout 300 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/m_tests1.log 2>&1; echo rc=$?
tail -20 gpurun_out/m_tests1.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/m_tests.log 2>&1; echo rc=$?
tail -5 gpurun_out/m_tests.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench_mega.log 2>&1; echo rc=$?
tail -c 1200 gpurun_out/bench_mega.log
