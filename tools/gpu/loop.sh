# device-resident loop: parity vs the host loop, then the decode suite (now on the device loop by default)
timeout 1200 python -m pytest tests/test_gpu_loop.py -x -q -p no:cacheprovider "$@" > gpurun_out/loop_tests.log 2>&1; echo loop tests rc=$?
grep -E "passed|failed|Error|error" gpurun_out/loop_tests.log | tail -5; grep -B5 -A25 "^E  " gpurun_out/loop_tests.log | head -60
timeout 1200 python -m pytest tests/test_gpu_decode.py tests/test_gpu_shard.py -x -q -p no:cacheprovider > gpurun_out/decode_tests.log 2>&1; echo decode tests rc=$?
tail -3 gpurun_out/decode_tests.log
