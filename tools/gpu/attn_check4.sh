timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo rc=$?; tail -1 gpurun_out/t.log
for t in _ab/head .; do echo "== $t"; (cd $t && for a in "8 33 182 36" "64 33 8192 36" "8 128 128 36" "8 33 2048 36"; do timeout 120 python tools/attn_bench.py one $a 2>&1 | tail -1 | cut -c1-125; done); done
