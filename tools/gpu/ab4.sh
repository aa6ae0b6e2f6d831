timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -2 gpurun_out/t.log
bash tools/gpu/ab3.sh
