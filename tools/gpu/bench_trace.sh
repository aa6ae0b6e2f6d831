timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo rc=$?
tail -3 gpurun_out/g_tests.log
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench.log
timeout 300 python tools/trace_gen.py > gpurun_out/trace.txt 2>&1; echo rc=$?
head -40 gpurun_out/trace.txt
