for nb in 1 2; do for s in 1 2 3 4 6 8; do
BASS_GEMM_NB=$nb BASS_FORCE_SPLIT=$s timeout 120 python tools/gemm_micro.py 8,88,136 all packed > gpurun_out/sw_nb${nb}_s${s}.jsonl 2>&1
done; done
echo done
