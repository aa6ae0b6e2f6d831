"""Golden vectors for the INT8 W8A8 path, produced by running the REFERENCE.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_quant.py

Writes tests/golden/quant.npz: known-answer cases of the quantizers and the
integer GEMM (ref:quant.py), the quantized payload / scales of whole model
matrices (ref:model.py:135-143), and quantized ragged-forward logits and a
greedy decode on two tiny models (ref:model.py:177-246 with `quantized`,
engine.py:120-197).  Pins oracle/quant.py and, through it, the device path.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from batchspec import attention as A          # noqa: E402
from batchspec import engine as E             # noqa: E402
from batchspec import model as M              # noqa: E402
from batchspec import quant as Q              # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MODELS = {"a": dict(n_layer=2, n_head=4, d_model=128, vocab_size=512, max_seq_len=256),
          "b": dict(n_layer=2, n_head=2, d_model=256, vocab_size=384, max_seq_len=256)}


def main():
    arr = {}
    rs = np.random.default_rng(21)
    # quantizer / GEMM known answers
    for c in range(6):
        m, k, n = int(rs.integers(1, 9)), 128, 128 * int(rs.integers(1, 3))
        a = rs.standard_normal((m, k)) * rs.uniform(0.1, 10)
        # weights on the float32 grid, like every model weight (ref:model.py:106-132)
        w = (rs.standard_normal((k, n)) * rs.uniform(0.01, 1)).astype(np.float32).astype(np.float64)
        if c == 0:
            w[:, 3] = 0.0              # all-zero channel: scale 1
            a[0] = 0.0                 # all-zero token
        aq, wq = Q.quantize_activations_per_token(a), Q.quantize_weights_per_channel(w)
        arr[f"k{c}_a"], arr[f"k{c}_w"] = a, w.astype(np.float32)
        arr[f"k{c}_ap"], arr[f"k{c}_as"] = aq.payload, aq.scales
        arr[f"k{c}_wp"], arr[f"k{c}_ws"] = wq.payload, wq.scales
        arr[f"k{c}_out"] = Q.int_gemm_dequant(aq, wq)
        t = rs.standard_normal((m, 64)) * rs.uniform(0.01, 50)
        arr[f"k{c}_t"], arr[f"k{c}_tfq"] = t, Q.fake_quant_per_head(t, 4)
    # whole models
    rs = np.random.default_rng(0)
    prompts = [rs.integers(0, 384, n).tolist() for n in (5, 1, 9, 3)]
    blocks = [rs.integers(0, 384, n).tolist() for n in (3, 7, 5, 1)]
    for i, p in enumerate(prompts):
        arr[f"prompt_{i}"] = np.asarray(p)
        arr[f"block_{i}"] = np.asarray(blocks[i])
    for key, geo in MODELS.items():
        cfg = M.desk_config(**geo)
        w = M.init_model(cfg, 5)
        qw = M.prepare_quantized(w)
        for name in ("wq", "w_proj"):
            t = qw.blocks[1][name]
            arr[f"{key}_{name}1_p"], arr[f"{key}_{name}1_s"] = t.payload, t.scales
        arr[f"{key}_head_p"], arr[f"{key}_head_s"] = qw.head.payload, qw.head.scales
        for strat in (A.AttentionStrategy.PAD, A.AttentionStrategy.SPLIT):
            main = M.MainModel(w, 4, strat, quantized=True)
            for i, p in enumerate(prompts):
                arr[f"{key}_{strat.value}_prefill_{i}"] = main.prefill(i, p)
            out = main.forward([0, 1, 2, 3], blocks)
            for i, o in enumerate(out):
                arr[f"{key}_{strat.value}_block_{i}"] = o
        req = E.GenerationRequest(prompts=[p[:4] or [1] for p in prompts], max_new_tokens=24,
                                  temperature=0.0)
        res = E.decode_regular(M.MainModel(w, 4, quantized=True), req)
        for i, t in enumerate(res.tokens):
            arr[f"{key}_greedy_{i}"] = np.asarray(t)
    np.savez_compressed(os.path.join(OUT, "quant.npz"), **arr)
    print("wrote", os.path.join(OUT, "quant.npz"), len(arr), "arrays")


if __name__ == "__main__":
    main()
