for tt in 256 192 160 128; do echo "== TT $tt"; BASS_BIG_TT=$tt timeout 300 python tools/gemm_micro.py 1100 qkv,o,fc,proj packed; done
