export BASS_GEMM_IMPL=dk
for t in "3 8" "2 16" "6 4"; do set -- $t
BASS_DK_TARGET=$1 BASS_DK_MIN_UNITS=$2 timeout 200 python tools/gemm_micro.py 8,88 all packed > gpurun_out/gemm_dk_$1_$2.jsonl 2>&1; echo rc=$?
done
BASS_DK_TARGET=3 BASS_DK_MIN_UNITS=8 timeout 200 python -m pytest tests/test_gpu_decode.py -x -q > gpurun_out/dk_tests1.log 2>&1; echo rc=$?
tail -3 gpurun_out/dk_tests1.log
