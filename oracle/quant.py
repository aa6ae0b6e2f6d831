"""INT8 W8A8 numerics, restated in numpy — TEST INFRASTRUCTURE ONLY.

Restates the reference's quantized inference path
(ref:quant.py:19-129, model.py:135-143 prepare_quantized, model.py:160-164
``_linear``, model.py:219-222 fake-quant of q/k/v): symmetric scale-only
int8, one scale per weight output channel, per activation row, per
(token, head) for q/k/v; the GEMM accumulates the int8 payloads exactly in
int64 and applies both scales in one dequantizing epilogue.  Pinned by
``tests/golden/quant.npz`` (outputs of the reference itself,
``tests/golden/make_golden_quant.py``).
"""

from __future__ import annotations

import numpy as np

from .ragged import (Geometry, RaggedCache, _heads, _unheads, attend_pad,
                     attend_split, gelu_erf, layer_norm)

QMAX = 127                                   # ref:quant.py:19


def round_half_away(x):
    """ref:quant.py:44-45."""
    return np.sign(x) * np.floor(np.abs(x) + 0.5)


def quantize_groups(x, group_max):
    """ref:quant.py:48-52: zero-max groups get scale 1."""
    scales = np.where(group_max > 0, group_max / QMAX, 1.0)
    payload = np.clip(round_half_away(x / scales), -QMAX, QMAX)
    return payload.astype(np.int8), scales


def quantize_weights(w):
    """[d_in, d_out] -> (payload int8, scales [d_out]) (ref:quant.py:55-63)."""
    w = np.asarray(w, dtype=np.float64)
    p, s = quantize_groups(w, np.abs(w).max(axis=0, keepdims=True))
    return p, s[0]


def quantize_tokens(a):
    """[tokens, d] -> (payload, scales [tokens]) (ref:quant.py:66-74)."""
    a = np.asarray(a, dtype=np.float64)
    p, s = quantize_groups(a, np.abs(a).max(axis=1, keepdims=True))
    return p, s[:, 0]


def fake_quant_heads(t, n_head):
    """Round trip through per-(token, head) int8 (ref:quant.py:77-89, 126-129)."""
    t = np.asarray(t, dtype=np.float64)
    n, d = t.shape
    g = t.reshape(n, n_head, d // n_head)
    p, s = quantize_groups(g, np.abs(g).max(axis=2, keepdims=True))
    return (p.astype(np.float64) * s).reshape(n, d)


def int_gemm_dequant(ap, as_, wp, ws):
    """acc * s_token * s_channel (ref:quant.py:98-123).  The reference
    accumulates in int64; every partial sum of int8 x int8 products here is an
    integer below 2^53 (127^2 * K for K <= 5e11), so the float64 BLAS product
    of the payloads is the same exact integer in any summation order."""
    acc = ap.astype(np.float64) @ wp.astype(np.float64)
    return acc * as_[:, None] * ws[None, :]


def prepare(w: dict) -> dict:
    """Per-channel payload/scales of every matrix (ref:model.py:135-143)."""
    keys = ("wq", "wk", "wv", "wo", "w_fc", "w_proj")
    return {"layers": [{k: quantize_weights(lay[k]) for k in keys} for lay in w["layers"]],
            "head": quantize_weights(w["head"])}


def _linear(x, qw):
    """ref:model.py:160-164 with a QuantTensor."""
    ap, as_ = quantize_tokens(x)
    return int_gemm_dequant(ap, as_, *qw)


def forward_ragged_int8(w: dict, qw: dict, cache: RaggedCache, slots, blocks,
                        strategy: str = "pad"):
    """``forward_ragged`` on the quantized path (ref:model.py:177-246 with
    ``quantized``): same structure, every linear through ``_linear`` above and
    q / k / v fake-quantized per (token, head) before the cache and attention."""
    g: Geometry = w["geometry"]
    offs = [cache.length(s) for s in slots]
    xs = [np.asarray(w["tok_emb"][np.asarray(blk)], dtype=np.float64)
          + w["pos_emb"][np.arange(off, off + len(blk))] for blk, off in zip(blocks, offs)]
    attend = attend_pad if strategy == "pad" else attend_split
    for li, lay in enumerate(w["layers"]):
        ql = qw["layers"][li]
        qs = []
        for i, s in enumerate(slots):
            h = layer_norm(xs[i], lay["ln1_g"], lay["ln1_b"])
            q = fake_quant_heads(_linear(h, ql["wq"]), g.n_head)
            k = fake_quant_heads(_linear(h, ql["wk"]), g.n_head)
            v = fake_quant_heads(_linear(h, ql["wv"]), g.n_head)
            cache.append(s, li, _heads(k, g.n_head), _heads(v, g.n_head))
            qs.append(_heads(q, g.n_head))
        kv = [cache.view(s, li) for s in slots]
        ctx = attend(qs, [a for a, _ in kv], [b for _, b in kv], offs)
        for i in range(len(slots)):
            xs[i] = xs[i] + _linear(_unheads(ctx[i]), ql["wo"])
            h2 = layer_norm(xs[i], lay["ln2_g"], lay["ln2_b"])
            xs[i] = xs[i] + _linear(gelu_erf(_linear(h2, ql["w_fc"])), ql["w_proj"])
    return [_linear(layer_norm(x, w["lnf_g"], w["lnf_b"]), qw["head"]) for x in xs]
