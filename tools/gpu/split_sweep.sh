for s in 1 2 3 4 6 8; do
BASS_FORCE_SPLIT=$s timeout 150 python tools/gemm_micro.py 8,88,136 all packed > gpurun_out/ss_s${s}.jsonl 2>&1
done; echo done
