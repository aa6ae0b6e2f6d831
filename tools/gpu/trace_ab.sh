(cd _ab/head && TRACE_CSV=/tmp/head.csv timeout 300 python tools/trace_gen.py > /tmp/head_trace.txt 2>&1); cp /tmp/head.csv gpurun_out/trace_head.csv
BASS_LNFUSE=0 TRACE_CSV=gpurun_out/trace_nofuse.csv timeout 300 python tools/trace_gen.py > gpurun_out/trace_nofuse.txt 2>&1
TRACE_CSV=gpurun_out/trace_fuse.csv timeout 300 python tools/trace_gen.py > gpurun_out/trace_fuse.txt 2>&1
head -8 /tmp/head_trace.txt; head -8 gpurun_out/trace_nofuse.txt; head -8 gpurun_out/trace_fuse.txt
