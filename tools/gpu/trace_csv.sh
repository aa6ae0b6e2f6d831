TRACE_CSV=gpurun_out/trace_launches.csv timeout 300 python tools/trace_gen.py > gpurun_out/trace.txt 2>&1; echo rc=$?
head -8 gpurun_out/trace.txt
