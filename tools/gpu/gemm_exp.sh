for mu in 1 4 8; do
BASS_SK_MIN_UNITS=$mu timeout 300 python tools/gemm_micro.py 8,88 > gpurun_out/gemm_sk100_mu$mu.jsonl 2>&1; echo rc=$?
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --kernel-events 0 > gpurun_out/bench100.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/bench100.log | head -c 700
