"""Reference-identical weights at benchmark geometries, streamed tensor by tensor.

The reference's `init_model` (ref:model.py:106-132) draws every tensor from one
`default_rng(seed)` stream in a fixed order: token_emb [V,d], pos_emb [S,d],
then per layer wq, wk, wv, wo [d,d], w_fc [d,4d], w_proj [4d,d], then head
[d,V]; each draw is `normal(0, 0.02)` cast to float32.  numpy's normal draws
are chunk-invariant (two successive calls equal one
concatenated call), so the tensors can be produced one at a time in that
order without holding the whole fp64 model (65 GB for the 7.8B shape).

Every value is then rounded to the bf16 grid (round-to-nearest-even; SURVEY
App. A.2): the device stores bf16 weights, and the oracle fed the *same*
rounded values is the parity reference.  Arrays are kept in float32 (bf16
values are exact there); the oracle upcasts to float64 inside its matmuls.

Test infrastructure only (imports the oracle's geometry type; never imported
by the product package).
"""

from __future__ import annotations

import numpy as np

from oracle import ragged as OR

INIT_STD = OR.INIT_STD
LAYER_ORDER = ("wq", "wk", "wv", "wo", "w_fc", "w_proj")


def bf16_round(a) -> np.ndarray:
    """float32 round-to-nearest-even onto the bf16 grid (returned as float32)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    u = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


def layer_shapes(g: OR.Geometry):
    d, ff = g.d_model, g.d_ff
    return {"wq": (d, d), "wk": (d, d), "wv": (d, d), "wo": (d, d), "w_fc": (d, ff),
            "w_proj": (ff, d)}


def stream_init(g: OR.Geometry, seed: int):
    """Yield (name, layer, float32 bf16-rounded array) in the reference's draw order.

    name in {"tok_emb", "pos_emb", "head"} (layer None) or a LAYER_ORDER key.
    """
    rng = np.random.default_rng(seed)

    def draw(shape):
        return bf16_round(rng.normal(0.0, INIT_STD, size=shape).astype(np.float32))

    yield "tok_emb", None, draw((g.vocab_size, g.d_model))
    yield "pos_emb", None, draw((g.max_seq_len, g.d_model))
    shapes = layer_shapes(g)
    for li in range(g.n_layer):
        for k in LAYER_ORDER:
            yield k, li, draw(shapes[k])
    yield "head", None, draw((g.d_model, g.vocab_size))


def init_dict(g: OR.Geometry, seed: int) -> dict:
    """The oracle's weight dict (ref names) with bf16-rounded float32 arrays."""
    d = g.d_model
    w = {"layers": [{"ln1_g": np.ones(d), "ln1_b": np.zeros(d), "ln2_g": np.ones(d),
                     "ln2_b": np.zeros(d)} for _ in range(g.n_layer)],
         "lnf_g": np.ones(d), "lnf_b": np.zeros(d), "geometry": g}
    for name, li, arr in stream_init(g, seed):
        if li is None:
            w[name] = arr
        else:
            w["layers"][li][name] = arr
    return w


# oracle dict key -> libbass tensor id name (paper_2404_15778_b200._lib W_*)
TENSOR_IDS = {"tok_emb": "W_TOK_EMB", "pos_emb": "W_POS_EMB", "head": "W_HEAD", "wq": "W_WQ",
              "wk": "W_WK", "wv": "W_WV", "wo": "W_WO", "w_fc": "W_FC", "w_proj": "W_PROJ",
              "ln1_g": "W_LN1_G", "ln1_b": "W_LN1_B", "ln2_g": "W_LN2_G", "ln2_b": "W_LN2_B",
              "lnf_g": "W_LNF_G", "lnf_b": "W_LNF_B"}


def upload(dw, name: str, layer, arr) -> None:
    """Put one reference-layout tensor into a DeviceWeights."""
    from paper_2404_15778_b200 import _lib as L
    dw._put(getattr(L, TENSOR_IDS[name]), 0 if layer is None else layer, arr)


def upload_unit_norms(dw, g: OR.Geometry) -> None:
    d = g.d_model
    one, zero = np.ones(d, np.float32), np.zeros(d, np.float32)
    for li in range(g.n_layer):
        for k, v in (("ln1_g", one), ("ln1_b", zero), ("ln2_g", one), ("ln2_b", zero)):
            upload(dw, k, li, v)
    upload(dw, "lnf_g", None, one)
    upload(dw, "lnf_b", None, zero)


def oracle_layer(x: np.ndarray, lay: dict, g: OR.Geometry) -> np.ndarray:
    """One pre-LN block over a single sequence's prompt (prefill, causal over
    itself), float64 — ref:model.py:211-245 for one sequence, offset 0."""
    h = OR.layer_norm(x, lay.get("ln1_g", 1.0), lay.get("ln1_b", 0.0))
    q, k, v = h @ lay["wq"], h @ lay["wk"], h @ lay["wv"]
    ctx = OR.attend_split([OR._heads(q, g.n_head)], [OR._heads(k, g.n_head)],
                          [OR._heads(v, g.n_head)], [0])[0]
    x = x + OR._unheads(ctx) @ lay["wo"]
    h2 = OR.layer_norm(x, lay.get("ln2_g", 1.0), lay.get("ln2_b", 0.0))
    return x + OR.gelu_erf(h2 @ lay["w_fc"]) @ lay["w_proj"]


def row_rel_err(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """max|got - want| / max|want| per logits row (SURVEY 7.2(1) metric)."""
    got, want = np.atleast_2d(got), np.atleast_2d(want)
    return np.abs(got - want).max(axis=1) / np.abs(want).max(axis=1)
