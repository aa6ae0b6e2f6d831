"""Prompt prefill: the C2 main model's ragged forward over b
prompts of P tokens (the prompt step of a generation, ref:model.py:249-260,
engine.py:134), device-timed; per-kernel-class time (CUDA events between
launches: serialised, an upper bound), algorithmic flops, and the achieved
TFLOP/s against the measured dense bf16 peak.  Usage:
    python tools/prefill_bench.py [b] [P] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_15778_b200 as B  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    tf_peak = float(peaks.get("bf16_tflops") or peaks.get("bf16_dense_tflops") or 1637.0)
except Exception:
    tf_peak = 1637.0
cfg = B.ModelConfig(30, 36, 4608, 128, 50272, 2048)
ctx = B.CudaContext(0)
stream = torch.cuda.Stream()
ctx.set_stream(stream.cuda_stream)   # the events below bracket the context's own stream
w = B.DeviceWeights.random(cfg, 1000, ctx=ctx)
m = B.CudaModel(w, b, "ragged", capacity=P + 8)
rs = np.random.default_rng(0)
prompts = [rs.integers(0, cfg.vocab_size, P).tolist() for _ in range(b)]


def once(profile=False):
    for s in range(b):
        m.rollback(s, 0)
    if profile:
        ctx.profile(True)
    m.forward(list(range(b)), prompts, last_only=True)
    ctx.sync()
    if profile:
        out = ctx.profile_read()
        ctx.profile(False)
        return out
    return None


once()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = stream
times = []
for _ in range(reps):
    for s in range(b):
        m.rollback(s, 0)
    torch.cuda.synchronize()
    ev0.record(st)
    m.forward(list(range(b)), prompts, last_only=True)
    ev1.record(st)
    torch.cuda.synchronize()
    times.append(ev0.elapsed_time(ev1))
prof = once(profile=True)
ms = float(np.median(times))
d, L, V = cfg.d_model, cfg.n_layer, cfg.vocab_size
M = b * P
gemm_flops = 2.0 * M * L * 12 * d * d + 2.0 * b * d * V          # projections + last-row head
attn_flops = L * 4.0 * d * b * (P * (P + 1) / 2)                  # causal QK^T + PV
line = {"prefill": f"C2 main, {b} x {P} prompt tokens", "ms": round(ms, 3),
        "prompt_tokens_per_s": round(M / ms * 1e3, 1),
        "tflops_total": round((gemm_flops + attn_flops) / ms / 1e9, 1),
        "tflops_peak": tf_peak, "frac_total": round((gemm_flops + attn_flops) / ms / 1e9 / tf_peak, 3),
        "classes_serialised": {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                                   "tflops": round(v["flops"] / max(v["ms"], 1e-9) / 1e9, 1)}
                               for k, v in prof.items() if v["launches"]}}
print(json.dumps(line), flush=True)
