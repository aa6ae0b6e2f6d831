set -x
export BASS_ATTN_MODE=stream
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention > gpurun_out/st_tests1.log 2>&1; echo rc=$?
tail -5 gpurun_out/st_tests1.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/st_tests.log 2>&1; echo rc=$?
tail -5 gpurun_out/st_tests.log
timeout 300 python tools/attn_sweep.py 1,8,64 1,8,16,32 512,2048,8192 ragged,pad > gpurun_out/sweep_stream2.jsonl 2>&1; echo rc=$?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_stream2.log 2>&1; echo rc=$?
tail -c 1800 gpurun_out/bench_stream2.log
