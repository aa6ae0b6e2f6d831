"""C4 ragged-attention sweep (BASELINE.json configs[3]): batch 1-64, draft
length k (q = k + 1 rows per sequence), context 512-8K, ragged (L_i ~
U[L/2, L]) vs equal lengths, RAGGED / PAD / SPLIT strategies.  H = 36,
d_head = 128, bf16 K/V/Q ~ N(0, 1).  Achieved GB/s = algorithmic bytes
(real K/V rows + Q in + O out) / CUDA-event time per call.
Prints one JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_15778_b200 as B  # noqa: E402

H, DH = 36, 128
HBM = 6545.9
ctx = B.CudaContext.default()
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)

batches = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,8,64").split(",")]
ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,8,16").split(",")]
Ls = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "512,2048,8192").split(",")]
strategies = (sys.argv[4] if len(sys.argv) > 4 else "ragged,pad").split(",")

for b in batches:
    for L in Ls:
        for ragged in (True, False):
            rng = np.random.default_rng(b * 100003 + L)
            lens = rng.integers(L // 2, L + 1, b) if ragged else np.full(b, L)
            stride = int(lens.max())
            K = torch.randn(b, H, stride, DH, device="cuda", dtype=torch.bfloat16)
            V = torch.randn(b, H, stride, DH, device="cuda", dtype=torch.bfloat16)
            for k in ks:
                q = k + 1
                cu = np.arange(b + 1) * q
                offs = (lens - q).tolist()
                Q = torch.randn(b * q, H, DH, device="cuda", dtype=torch.bfloat16)
                out = torch.empty_like(Q)
                by = sum(2 * H * int(n) * DH * 2 + 2 * H * q * DH * 2 for n in lens)
                for strat in strategies:
                    if strat == "split" and b > 8:
                        continue
                    best = float("inf")
                    for rep in range(4):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        B.attend_device(ctx, Q, K, V, cu, offs, strat, out=out)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        if rep:
                            best = min(best, e0.elapsed_time(e1) / 1e3)
                    gbs = by / best / 1e9
                    print(json.dumps({"b": b, "k": k, "L": L, "ragged": ragged, "strategy": strat,
                                      "us": round(best * 1e6, 1), "GB": round(by / 1e9, 4),
                                      "GB/s": round(gbs, 1), "frac": round(gbs / HBM, 3)}), flush=True)
            del K, V
            torch.cuda.empty_cache()
