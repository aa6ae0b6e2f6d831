"""Ragged decoder forward, KV store and PAD/SPLIT attention, restated in numpy.

The model (ref:model.py:1-260) is a pre-LN GELU decoder in float64 with
weights drawn on the float32 grid, learned absolute positions, untied head,
no linear biases, LN eps 1e-5.  Dense layers run per sequence exactly as the
reference does (ref:model.py:211-245) so that this file's CPU timing is the
reference's cost structure; only attention sees the whole ragged batch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
from scipy.special import erf

LN_EPS = 1e-5          # ref:model.py:31
INIT_STD = 0.02        # ref:model.py:32
PAD_MASK = -1e9        # ref:attention.py:27

LAYER_KEYS = ("wq", "wk", "wv", "wo", "w_fc", "w_proj")


@dataclass(frozen=True)
class Geometry:
    """ref:model.py:36-62 (same validation)."""

    n_layer: int
    n_head: int
    d_model: int
    d_head: int
    vocab_size: int
    max_seq_len: int

    def __post_init__(self):
        for k in ("n_layer", "n_head", "d_model", "d_head", "vocab_size",
                  "max_seq_len"):
            if getattr(self, k) < 1:
                raise ValueError(f"{k} must be >= 1")
        if self.d_model != self.n_head * self.d_head:
            raise ValueError("d_model must equal n_head * d_head")

    @property
    def d_ff(self):
        return 4 * self.d_model


def init_weights(g: Geometry, seed: int) -> dict:
    """Seeded N(0, 0.02) init on the float32 grid (ref:model.py:106-132).

    Draw order (one default_rng(seed) stream): token_emb [V,d], pos_emb
    [S,d], then per layer wq, wk, wv, wo [d,d], w_fc [d,4d], w_proj [4d,d],
    then head [d,V].  LN gains 1, biases 0.  Matrices are input-major
    (``x @ W``).
    """
    rng = np.random.default_rng(seed)

    def draw(shape):
        return rng.normal(0.0, INIT_STD, size=shape).astype(np.float32) \
                  .astype(np.float64)

    d, ff = g.d_model, g.d_ff
    w = {"tok_emb": draw((g.vocab_size, d)), "pos_emb": draw((g.max_seq_len, d))}
    layers = []
    for _ in range(g.n_layer):
        lay = {"ln1_g": np.ones(d), "ln1_b": np.zeros(d),
               "ln2_g": np.ones(d), "ln2_b": np.zeros(d)}
        for k, shape in (("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)),
                         ("wo", (d, d)), ("w_fc", (d, ff)),
                         ("w_proj", (ff, d))):
            lay[k] = draw(shape)
        layers.append(lay)
    w["layers"] = layers
    w["lnf_g"], w["lnf_b"] = np.ones(d), np.zeros(d)
    w["head"] = draw((d, g.vocab_size))
    w["geometry"] = g
    return w


class RaggedCache:
    """Per-(layer, slot) K/V with independent lengths (ref:kv_cache.py:23-128).

    Storage grows by doubling (ref:kv_cache.py:51-61); rollback only moves
    the length, so rolled-back rows are overwritten by the next append.
    """

    def __init__(self, n_layer, n_slot, n_head, d_head):
        self.shape = (n_head, d_head)
        self.n_layer, self.n_slot = n_layer, n_slot
        self.len = np.zeros((n_layer, n_slot), dtype=np.int64)
        self.k = [[np.empty((n_head, 0, d_head)) for _ in range(n_slot)]
                  for _ in range(n_layer)]
        self.v = [[np.empty((n_head, 0, d_head)) for _ in range(n_slot)]
                  for _ in range(n_layer)]

    def append(self, slot, layer, k, v):
        """k, v: [n_head, n, d_head] (ref:kv_cache.py:63-84)."""
        if k.ndim != 3 or (k.shape[0], k.shape[2]) != self.shape \
                or v.shape != k.shape:
            raise ValueError("geometry mismatch")
        n0, n = int(self.len[layer, slot]), k.shape[1]
        cap = self.k[layer][slot].shape[1]
        if n0 + n > cap:
            new_cap = max(n0 + n, 2 * cap, 16)
            for store in (self.k, self.v):
                grown = np.empty((self.shape[0], new_cap, self.shape[1]))
                grown[:, :n0] = store[layer][slot][:, :n0]
                store[layer][slot] = grown
        self.k[layer][slot][:, n0:n0 + n] = k
        self.v[layer][slot][:, n0:n0 + n] = v
        self.len[layer, slot] = n0 + n

    def view(self, slot, layer):
        n = int(self.len[layer, slot])
        return self.k[layer][slot][:, :n], self.v[layer][slot][:, :n]

    def length(self, slot):
        col = set(self.len[:, slot].tolist())
        if len(col) != 1:
            raise RuntimeError(f"slot {slot}: divergent layer lengths")
        return col.pop()

    def truncate(self, slot, n):
        """ref:kv_cache.py:93-104."""
        if n < 0 or n > int(self.len[:, slot].min()):
            raise ValueError(f"truncate to {n} outside [0, length]")
        self.len[:, slot] = n


def layer_norm(x, g, b):
    """ref:model.py:150-153 (population variance)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * g + b


def gelu_erf(x):
    """Exact-erf GELU (ref:model.py:156-157)."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def _masked_softmax(scores, offset):
    """Row t may see key s <= offset + t (ref:attention.py:85-93)."""
    _, nq, nk = scores.shape
    ok = np.arange(nk)[None, :] <= offset + np.arange(nq)[:, None]
    s = np.where(ok, scores, -np.inf)
    e = np.exp(s - s.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def attend_split(qs, ks, vs, offs):
    """Per-sequence GEMMs (ref:attention.py:96-104)."""
    c = math.sqrt(qs[0].shape[2])
    out = []
    for q, k, v, off in zip(qs, ks, vs, offs):
        p = _masked_softmax(np.matmul(q, np.swapaxes(k, 1, 2)) / c, off)
        out.append(np.matmul(p, v))
    return out


def attend_pad(qs, ks, vs, offs):
    """Pad Q/K/V to the batch maxima, one batched GEMM per stage, softmax on
    each sequence's unpadded slice (ref:attention.py:107-137)."""
    nb, nh, dh = len(qs), qs[0].shape[0], qs[0].shape[2]
    c = math.sqrt(dh)
    nq = [q.shape[1] for q in qs]
    nk = [k.shape[1] for k in ks]
    Q = np.zeros((nb, nh, max(nq), dh))
    K = np.zeros((nb, nh, max(nk), dh))
    V = np.zeros_like(K)
    for i in range(nb):
        Q[i, :, :nq[i]] = qs[i]
        K[i, :, :nk[i]] = ks[i]
        V[i, :, :nk[i]] = vs[i]
    S = np.matmul(Q, np.swapaxes(K, 2, 3)) / c
    P = np.zeros_like(S)
    for i in range(nb):
        S[i, :, :, nk[i]:] += PAD_MASK
        P[i, :, :nq[i], :nk[i]] = _masked_softmax(S[i, :, :nq[i], :nk[i]],
                                                  offs[i])
    O = np.matmul(P, V)
    return [O[i, :, :nq[i]] for i in range(nb)]


def _heads(x, nh):
    t, d = x.shape
    return x.reshape(t, nh, d // nh).transpose(1, 0, 2)


def _unheads(x):
    nh, t, dh = x.shape
    return x.transpose(1, 0, 2).reshape(t, nh * dh)


def forward_ragged(w: dict, cache: RaggedCache, slots, blocks,
                   strategy: str = "pad"):
    """Run ragged token blocks through the model (ref:model.py:177-246).

    ``blocks[i]`` extends slot ``slots[i]``; returns a [len_i, V] float64
    logits array per slot and appends every new position's K/V.
    """
    g: Geometry = w["geometry"]
    if len(slots) != len(blocks) or not slots:
        raise ValueError("active_seqs and new_tokens must align and be non-empty")
    offs = []
    for s, blk in zip(slots, blocks):
        if len(blk) < 1:
            raise ValueError(f"sequence {s}: empty token block")
        off = cache.length(s)
        if off + len(blk) > g.max_seq_len:
            raise ValueError(f"sequence {s}: context {off + len(blk)} "
                             f"exceeds max_seq_len {g.max_seq_len}")
        offs.append(off)
    xs = []
    for s, blk, off in zip(slots, blocks, offs):
        ids = np.asarray(blk, dtype=np.int64)
        if ids.min() < 0 or ids.max() >= g.vocab_size:
            raise ValueError(f"sequence {s}: token id outside vocab")
        # float64 residual stream even when the tables are stored on a
        # narrower grid (bf16-rounded float32 parity weights)
        xs.append(np.asarray(w["tok_emb"][ids], dtype=np.float64)
                  + w["pos_emb"][np.arange(off, off + len(blk))])
    attend = attend_pad if strategy == "pad" else attend_split
    for li, lay in enumerate(w["layers"]):
        qs = []
        for i, s in enumerate(slots):
            h = layer_norm(xs[i], lay["ln1_g"], lay["ln1_b"])
            q, k, v = h @ lay["wq"], h @ lay["wk"], h @ lay["wv"]
            cache.append(s, li, _heads(k, g.n_head), _heads(v, g.n_head))
            qs.append(_heads(q, g.n_head))
        kv = [cache.view(s, li) for s in slots]
        ctx = attend(qs, [a for a, _ in kv], [b for _, b in kv], offs)
        for i in range(len(slots)):
            xs[i] = xs[i] + _unheads(ctx[i]) @ lay["wo"]
            h2 = layer_norm(xs[i], lay["ln2_g"], lay["ln2_b"])
            xs[i] = xs[i] + gelu_erf(h2 @ lay["w_fc"]) @ lay["w_proj"]
    return [layer_norm(x, w["lnf_g"], w["lnf_b"]) @ w["head"] for x in xs]
