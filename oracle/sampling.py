"""Distribution shaping, inverse-CDF sampling and the accept/resample rule.

Restates ref:sampling.py:69-146 over plain float64 vectors (no wrapper
types).  Uniforms come from `KeyedStreams`, the same numpy construction as
ref:sampling.py:53-66; `oracle.rng` restates that construction bit-exactly
for the device implementation.
"""

from __future__ import annotations

import numpy as np

from .rng import M64, ROLE_DRAFT, ROLE_VERIFY


def shape_probs(logits, temperature: float, top_p: float) -> np.ndarray:
    """Temperature + nucleus shaping (ref:sampling.py:69-104).

    T == 0: one-hot on the first argmax.  Otherwise softmax(z / T) with
    max-subtraction; keep the shortest prefix in (descending probability,
    ascending id) order whose running sum reaches ``top_p``
    (left-searchsorted, clamped to the last index); renormalise.
    """
    if not 0.0 < top_p <= 1.0:
        raise ValueError(f"top_p must be in (0, 1], got {top_p}")
    if temperature < 0.0:
        raise ValueError(f"temperature must be >= 0, got {temperature}")
    z = np.asarray(logits, dtype=np.float64)
    if not np.isfinite(z).any():
        raise ValueError("all logits are -inf; distribution undefined")
    out = np.zeros_like(z)
    if temperature == 0.0:
        out[int(np.argmax(z))] = 1.0
        return out
    z = z / temperature
    z = z - z[np.isfinite(z)].max()
    e = np.exp(z)
    e[~np.isfinite(e)] = 0.0
    full = e / e.sum()
    ids = np.arange(full.size)
    rank = np.lexsort((ids, -full))
    run = np.cumsum(full[rank])
    last = min(int(np.searchsorted(run, top_p, side="left")), full.size - 1)
    kept = rank[: last + 1]
    out[kept] = full[kept]
    return out / out.sum()


def inverse_cdf(probs: np.ndarray, u: float) -> int:
    """ref:sampling.py:107-115: right-searchsorted of u * total in id order."""
    c = np.cumsum(probs)
    return min(int(np.searchsorted(c, u * c[-1], side="right")),
               probs.size - 1)


def accept_or_resample(q: np.ndarray, p: np.ndarray, tok: int,
                       draw) -> tuple[bool, int | None]:
    """ref:sampling.py:118-146.

    ``draw()`` yields successive uniforms of one keyed generator: the first
    is the accept test ``u * p(x) < q(x)``, the second (only on rejection)
    samples normalize(max(q - p, 0)).
    """
    px = float(p[tok])
    if px <= 0.0:
        raise ValueError(f"draft token {tok} has zero draft probability")
    qx = float(q[tok])
    if draw() * px < qx:
        return True, None
    r = np.maximum(q - p, 0.0)
    tot = r.sum()
    if tot <= 0.0:
        raise ValueError("residual is empty: q <= p everywhere")
    return False, inverse_cdf(r / tot, draw())


class KeyedStreams:
    """Per-(seed, sequence id, role, position) generators (ref:sampling.py:53-66)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & M64

    def gen(self, seq_id: int, role: int, counter: int):
        key = (self.seed, int(seq_id), int(role), int(counter))
        g = np.random.default_rng(np.random.SeedSequence(entropy=key))
        return g.random

    def draft(self, seq_id, pos):
        return self.gen(seq_id, ROLE_DRAFT, pos)

    def verify(self, seq_id, pos):
        return self.gen(seq_id, ROLE_VERIFY, pos)
