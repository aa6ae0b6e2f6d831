nproc; free -g | head -2
timeout 1200 python -m pytest tests/test_gpu_headline.py -x -q -s --durations=10 -p no:cacheprovider "$@" > gpurun_out/headline.log 2>&1; echo rc=$?
grep -E "rel err|passed|failed|Error|assert" gpurun_out/headline.log | head -30; tail -15 gpurun_out/headline.log
