BASS_LIB=$PWD/paper_2404_15778_b200/probe_lib/libbass_g.so timeout 600 python tools/gemm_probe_chain.py ${GP:-qkv,o,fc,proj,d_proj} 2>&1 | tail -90
