timeout 300 python tools/trace_gen.py > gpurun_out/trace_mega.txt 2>&1; echo rc=$?
head -70 gpurun_out/trace_mega.txt
