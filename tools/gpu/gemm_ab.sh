# A/B of the GEMM micro-benchmark: _ab/head vs working tree
Ms=${MS:-88,1100}
for t in _ab/head .; do echo "== $t"; (cd $t && timeout 300 python tools/gemm_micro.py $Ms qkv,o,fc,proj packed); done
