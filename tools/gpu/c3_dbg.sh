BASS_ATTN=simt PROMPT=128 NEW=128 timeout 300 python tools/repro_c3.py > gpurun_out/c3b.log 2>&1; echo rc=$?; tail -1 gpurun_out/c3b.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -2 gpurun_out/t.log
timeout 900 python bench.py --config c3 --steps 2 --warmup 2 > gpurun_out/bench_c3.log 2>&1; echo rc=$?; tail -c 1500 gpurun_out/bench_c3.log
