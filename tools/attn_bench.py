"""Device-timed ragged attention sweep (BASELINE.json configs[3], C4) plus the
C2 decode shapes, through bass_attention_bench: one plan, back-to-back
launches timed with CUDA events, K/V copies rotated so the working set
exceeds L2 (as in the forward, where ~0.5 GB of weights stream between two
attention launches).  H = 36 (16 for the draft rows), d_head = 128 (and 64),
bf16 K/V/Q ~ N(0, 1).  Achieved GB/s = algorithmic bytes (real K/V rows + Q in +
O out) / device time per call.  One JSON line per point.

    python tools/attn_bench.py [sweep|c2|all] [strategies]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_15778_b200 as B  # noqa: E402
from paper_2404_15778_b200 import _lib as L  # noqa: E402
from paper_2404_15778_b200.attention import strategy_code  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


HBM = peak()
ctx = B.CudaContext.default()
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)


_KV = {}


def _kv(n, dh):
    """one pool of random K/V rows per d_head, reused across points (views)"""
    if _KV.get(dh) is None or _KV[dh][0].numel() < n:
        _KV[dh] = None
        torch.cuda.empty_cache()
        _KV[dh] = (torch.randn(n, device="cuda", dtype=torch.bfloat16),
                   torch.randn(n, device="cuda", dtype=torch.bfloat16))
    return _KV[dh][0][:n], _KV[dh][1][:n]


def point(lens, q_lens, H, strategy, tag, reps=20, dh=128):
    b = len(lens)
    stride = int(max(lens))
    kv_bytes = b * H * stride * dh * 2
    n_kv = max(1, min(16, int(300e6 // kv_bytes) + 1))
    K, V = _kv(n_kv * b * H * stride * dh, dh)
    cu = np.concatenate([[0], np.cumsum(q_lens)]).astype(np.int32)
    offs = np.array([n - q for n, q in zip(lens, q_lens)], dtype=np.int32)
    Q = torch.randn(int(cu[-1]), H, dh, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(Q)
    ms = C.c_double()
    torch.cuda.synchronize()
    ctx.check(ctx.lib.bass_attention_bench(ctx.handle, strategy_code(strategy), b, H, dh, L.ptr(cu, C.c_int32),
                                           L.ptr(offs, C.c_int32), C.c_void_p(Q.data_ptr()),
                                           C.c_void_p(K.data_ptr()), C.c_void_p(V.data_ptr()), stride, n_kv,
                                           C.c_void_p(out.data_ptr()), reps, C.byref(ms)))
    t = ms.value / 1e3
    by = sum(2 * H * int(n) * dh * 2 + 2 * H * int(q) * dh * 2 for n, q in zip(lens, q_lens))
    gbs = by / t / 1e9
    rec = {"tag": tag, "b": b, "H": H, "dh": dh, "q": int(max(q_lens)), "L": int(max(lens)), "strategy": strategy,
           "us": round(t * 1e6, 2), "MB": round(by / 1e6, 2), "GB/s": round(gbs, 1), "frac": round(gbs / HBM, 3)}
    print(json.dumps(rec), flush=True)
    return rec


def sweep(strategies):
    """SURVEY 8(d) C4 grid: b in {1..64}, L in {512..8K}, draft length k in
    {1, 2, 4, 8, 16} (q = k + 1) plus k = 32 (Alg. 1's limit); ragged lengths
    L_i ~ U[L/2, L] for every strategy (PAD streams the padding), equal
    lengths for the ragged kernel; d_head 64 (H = 36) on ragged lengths."""
    for b in (1, 2, 4, 8, 16, 32, 64):
        for Lc in (512, 1024, 2048, 4096, 8192):
            for ragged in (True, False):
                rng = np.random.default_rng(b * 100003 + Lc)
                lens = rng.integers(Lc // 2, Lc + 1, b) if ragged else np.full(b, Lc)
                for k in (1, 2, 4, 8, 16, 32):
                    for s in (strategies if ragged else ["ragged"]):
                        point(lens.tolist(), [k + 1] * b, 36, s, f"c4{'r' if ragged else 'e'}")
                    if ragged:
                        point(lens.tolist(), [k + 1] * b, 36, "ragged", "c4r-dh64", dh=64)


def c2(strategies):
    # the benchmark's attention launches: 128-token prompts, contexts 130-300,
    # main verify q = k+1 (H=36), draft decode q = 1-2 (H=16)
    rng = np.random.default_rng(7)
    for ctxlen in (160, 256):
        lens = (ctxlen + rng.integers(-24, 25, 8)).tolist()
        for s in strategies:
            for k in (4, 10, 16, 32):
                point(lens, [k + 1] * 8, 36, s, "c2-verify")
            point(lens, [1] * 8, 16, s, "c2-draft")
            point(lens, [1] * 8, 36, s, "c2-rd")
    for s in strategies:
        point([128] * 8, [128] * 8, 36, s, "c2-prefill")


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what == "one":   # python tools/attn_bench.py one b q L H [strategy [dh [reps]]]  (ncu captures)
        b, q, Lc, H = (int(a) for a in sys.argv[2:6])
        point([Lc] * b, [q] * b, H, sys.argv[6] if len(sys.argv) > 6 else "ragged", "one",
              reps=int(sys.argv[8]) if len(sys.argv) > 8 else 3, dh=int(sys.argv[7]) if len(sys.argv) > 7 else 128)
        sys.exit(0)
    strategies = (sys.argv[2] if len(sys.argv) > 2 else "ragged").split(",")
    if what in ("c2", "all"):
        c2(strategies)
    if what in ("sweep", "all"):
        sweep(strategies)
