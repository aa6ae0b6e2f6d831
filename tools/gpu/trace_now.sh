TRACE_CSV=gpurun_out/trace_fuse.csv timeout 300 python tools/trace_gen.py > gpurun_out/trace_fuse.txt 2>&1
head -60 gpurun_out/trace_fuse.txt
