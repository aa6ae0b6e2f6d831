BASS_LIB=$PWD/paper_2404_15778_b200/probe_lib/libbass.so timeout 300 python tools/attn_probe_chain.py 2>&1 | tail -17
