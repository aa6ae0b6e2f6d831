"""GEMM microbenchmark: the forward's projection shapes at decode / verify /
prefill M, back-to-back launches timed with CUDA events (bass_gemm_bench),
rotating over weight copies totalling > L2 so every launch streams HBM.
Prints one JSON line per shape with achieved algorithmic GB/s."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2404_15778_b200 as B  # noqa: E402
from paper_2404_15778_b200 import _lib as L  # noqa: E402

d, dd, V = 4608, 2048, 50272
SHAPES = {"qkv": (3 * d, d), "o": (d, d), "fc": (4 * d, d), "proj": (d, 4 * d), "head": (V, d),
          "d_qkv": (3 * dd, dd), "d_o": (dd, dd), "d_fc": (4 * dd, dd), "d_proj": (dd, 4 * dd),
          "d_head": (V, dd)}
Ms = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["8", "16", "88", "264"])]
only = sys.argv[2].split(",") if len(sys.argv) > 2 and sys.argv[2] != "all" else list(SHAPES)
# argv[3] == "packed": weights in the packed tile layout the model uses (mode 3 of bass_gemm_bench)
gmode = 3 if len(sys.argv) > 3 and sys.argv[3] == "packed" else L.GEMM_TC
reps = 40
hbm = 6545.9
handle = B.DeviceWeights(B.ModelConfig(1, 2, 128, 64, 256, 64), "bf16")
ctx = handle.ctx
for name in only:
    N, K = SHAPES[name]
    n_w = max(2, int(512e6 // (N * K * 2)) + 1)
    w = (torch.randn(n_w * N, K, device="cuda") * 0.02).bfloat16()
    for M in Ms:
        x = torch.randn(M, K, device="cuda").bfloat16()
        y = torch.empty(M, N, device="cuda")
        ms = C.c_double()
        ctx.check(ctx.lib.bass_gemm_bench(handle.handle, gmode, M, N, K, C.c_void_p(x.data_ptr()),
                                          C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()), reps, n_w,
                                          C.byref(ms)))
        t = ms.value / 1e3
        by = N * K * 2 + M * K * 2 + M * N * 4
        print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "us": round(t * 1e6, 2),
                          "GB/s": round(by / t / 1e9, 1), "frac": round(by / t / 1e9 / hbm, 3)}),
              flush=True)
    del w
