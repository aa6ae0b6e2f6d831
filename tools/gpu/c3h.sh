# device-loop tests incl. the sampled harness; C3 with the point-mass harness (align 0.874) vs natural
timeout 1200 python -m pytest tests/test_gpu_loop.py -x -q -p no:cacheprovider > gpurun_out/loop_tests.log 2>&1; echo loop tests rc=$?
tail -3 gpurun_out/loop_tests.log; grep -B3 -A20 "^E  " gpurun_out/loop_tests.log | head -40
for a in 0.874; do
  timeout 900 python bench.py --config c3 --steps 2 --warmup 3 --align $a --no-cpu-baseline > gpurun_out/bench_c3_align.log 2>&1; echo c3 align rc=$?
  grep "^{" gpurun_out/bench_c3_align.log | tail -1 > gpurun_out/bench_c3_align.jsonl
  python -c "
import json; d=json.load(open('gpurun_out/bench_c3_align.jsonl')); print('c3 align', round(d['value'],1), d['per_seq_ms_per_token'], d['regular_decode_ms_per_token'], d['mean_accepted'], d['mean_draft_len'], d['tokens_per_step_per_seq'], d['loop'])"
  tail -3 gpurun_out/bench_c3_align.log | grep -v "^{"
done
