timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo rc=$?
tail -c 2500 gpurun_out/bench_c3.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/bench_c2.log
