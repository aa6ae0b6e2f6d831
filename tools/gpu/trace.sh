timeout 300 python tools/trace_gen.py > gpurun_out/trace_sk.txt 2>&1; echo rc=$?
head -40 gpurun_out/trace_sk.txt
BASS_GEMM_IMPL=split BASS_PACK=0 timeout 300 python tools/trace_gen.py > gpurun_out/trace_split.txt 2>&1; echo rc=$?
head -40 gpurun_out/trace_split.txt
