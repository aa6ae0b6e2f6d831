timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -1 gpurun_out/t.log
bash tools/gpu/attn_check.sh
