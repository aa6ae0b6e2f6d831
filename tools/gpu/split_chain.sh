# in-chain split-count sweep for the bench GEMM shapes (BASS_SPLIT_OVERRIDE)
run() { (env $2 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --kernel-events 0 > /tmp/b.log 2>&1); python -c "
import json
l=[x for x in open('/tmp/b.log') if x.startswith('{')][-1]; d=json.loads(l); print('$1', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4))"; }
run base X=1
for o in 4 8; do run O$o BASS_SPLIT_OVERRIDE=4608x4608:$o; done
for p in 4 8; do run P$p BASS_SPLIT_OVERRIDE=4608x18432:$p; done
run Q1 BASS_SPLIT_OVERRIDE=13824x4608:1
run Q3 BASS_SPLIT_OVERRIDE=13824x4608:3
run F1 BASS_SPLIT_OVERRIDE=18432x4608:1
run dQ3 BASS_SPLIT_OVERRIDE=6144x2048:3
run dQ6 BASS_SPLIT_OVERRIDE=6144x2048:6
run dF2 BASS_SPLIT_OVERRIDE=8192x2048:2
run dO4 BASS_SPLIT_OVERRIDE=2048x2048:4
run dP4 BASS_SPLIT_OVERRIDE=2048x8192:4
run base X=1
