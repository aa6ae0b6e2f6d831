set -x
BASS_ATTN_MODE=chunk timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --save-traj gpurun_out/traj.npy > gpurun_out/bench_chunk.log 2>&1
tail -c 1500 gpurun_out/bench_chunk.log
timeout 600 python tools/attn_sweep.py 8,64 1,8,16 512,2048,8192 ragged,pad > gpurun_out/sweep_stream.jsonl 2>&1
BASS_ATTN_MODE=chunk timeout 600 python tools/attn_sweep.py 8,64 1,8,16 512,2048,8192 ragged,pad > gpurun_out/sweep_chunk.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_stream.csv python bench.py --profile-only --warmup 0 --load-traj gpurun_out/traj.npy --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1
python tools/ncu_summary.py gpurun_out/launches_stream.csv 40 > gpurun_out/launches_stream_summary.txt
head -45 gpurun_out/launches_stream_summary.txt
