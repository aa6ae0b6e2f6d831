# A/B the C2 bench between the in-tree libbass.so and tools/bin/libbass_base.so
# on the same box, alternating: usage  bash tools/gpu/ab.sh [rounds] [bench args]
R=${1:-2}; shift
for i in $(seq 1 $R); do
  for v in base new; do
    if [ $v = base ]; then export BASS_LIB=$PWD/tools/bin/libbass_base.so; else unset BASS_LIB; fi
    timeout 600 python bench.py --steps 3 --warmup 2 "$@" 2>/dev/null | grep "^{" | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), round(d['per_seq_ms_per_token']['all'],4))"
  done
done
