"""Bounded CPU timing of the reference algorithm (the oracle port) at full
benchmark shape — used ONLY by bench.py's cpu_baseline leg and its
`--impl reference` arm (timing the port, never checking or shipping it).

A full 7.8B-class step does not fit this budget (~21 s per 30-layer verify
on 8 cores), so one speculative step is measured piecewise at full
width with the reference's own per-sequence cost structure
(ref:model.py:211-245, ref:engine.py:249-271) and extrapolated by layer count:

  T_step = L_main * t_layer(main, verify block) + t_head(main, verify rows)
         + k * (L_draft * t_layer(draft, 1-row block) + t_head(draft, 1 row))

`time_generation_pieces` adds the first step's prompt blocks (the reference
prefills inside step 1's ragged block, ref:engine.py:248, 268), so a whole
generation's time is composed from an exact per-step draft-length schedule:

  T_gen = T_prefill + sum_steps [t_verify + l_step * t_draft_token]
"""

from __future__ import annotations

import time

import numpy as np

from .ragged import Geometry, RaggedCache, attend_pad, gelu_erf, layer_norm


def _rand(rng, shape):
    return rng.standard_normal(shape, dtype=np.float32).astype(np.float64) * 0.02


def _layer(rng, d):
    return {"ln1_g": np.ones(d), "ln1_b": np.zeros(d), "ln2_g": np.ones(d), "ln2_b": np.zeros(d),
            "wq": _rand(rng, (d, d)), "wk": _rand(rng, (d, d)), "wv": _rand(rng, (d, d)),
            "wo": _rand(rng, (d, d)), "w_fc": _rand(rng, (d, 4 * d)), "w_proj": _rand(rng, (4 * d, d))}


def _time_layer(g: Geometry, lay, xs, cache, slots, offs):
    """One decoder layer over per-sequence row blocks, as ref:model.py:211-239."""
    nh = g.n_head
    t0 = time.perf_counter()
    qs = []
    for i, s in enumerate(slots):
        h = layer_norm(xs[i], lay["ln1_g"], lay["ln1_b"])
        q, k, v = h @ lay["wq"], h @ lay["wk"], h @ lay["wv"]
        sh = lambda a: a.reshape(a.shape[0], nh, -1).transpose(1, 0, 2)
        cache.append(s, 0, sh(k), sh(v))
        qs.append(sh(q))
    kv = [cache.view(s, 0) for s in slots]
    ctx = attend_pad(qs, [a for a, _ in kv], [b for _, b in kv], offs)
    for i in range(len(slots)):
        xs[i] = xs[i] + ctx[i].transpose(1, 0, 2).reshape(xs[i].shape) @ lay["wo"]
        h2 = layer_norm(xs[i], lay["ln2_g"], lay["ln2_b"])
        xs[i] = xs[i] + gelu_erf(h2 @ lay["w_fc"]) @ lay["w_proj"]
    return time.perf_counter() - t0


def _time_head(head, xs):
    t0 = time.perf_counter()
    for x in xs:
        layer_norm(x, np.ones(x.shape[1]), np.zeros(x.shape[1])) @ head
    return time.perf_counter() - t0


def time_spec_step(main: Geometry, draft: Geometry, batch: int, ctx_len: int, k: int,
                   seed: int = 0, repeats: int = 1) -> dict:
    """Measure the pieces of one speculative step on the host cores."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, g, rows in (("main", main, k + 1), ("draft", draft, 1)):
        lay = _layer(rng, g.d_model)
        head = _rand(rng, (g.d_model, g.vocab_size))
        best_l, best_h = float("inf"), float("inf")
        for _ in range(repeats):
            cache = RaggedCache(1, batch, g.n_head, g.d_head)
            for s in range(batch):   # committed context already cached
                kv = rng.standard_normal((g.n_head, ctx_len, g.d_head))
                cache.append(s, 0, kv, kv)
            xs = [rng.standard_normal((rows, g.d_model)) for _ in range(batch)]
            best_l = min(best_l, _time_layer(g, lay, xs, cache, list(range(batch)),
                                             [ctx_len] * batch))
            best_h = min(best_h, _time_head(head, xs))
        out[name] = {"t_layer_s": best_l, "t_head_s": best_h, "rows_per_seq": rows}
        del lay, head
    t_step = main.n_layer * out["main"]["t_layer_s"] + out["main"]["t_head_s"] + \
        k * (draft.n_layer * out["draft"]["t_layer_s"] + out["draft"]["t_head_s"])
    out["t_step_s"] = t_step
    return out


def time_generation_pieces(main: Geometry, draft: Geometry, batch: int, prompt: int, ctx_len: int,
                           k: int, seed: int = 0) -> dict:
    """Host-core times of the pieces a generation is made of (full width, one
    layer each, extrapolated by layer count): the verify forward of a
    (k+1)-row block per sequence at context `ctx_len`, one draft token (1-row
    block), and the prompt blocks of step 1 (main: prompt + k rows, draft:
    prompt rows) from an empty cache."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, g, rows, ctx in (("verify", main, k + 1, ctx_len), ("draft_token", draft, 1, ctx_len),
                               ("prefill_main", main, prompt + k, 0), ("prefill_draft", draft, prompt, 0)):
        lay = _layer(rng, g.d_model)
        head = _rand(rng, (g.d_model, g.vocab_size))
        cache = RaggedCache(1, batch, g.n_head, g.d_head)
        if ctx:
            for s_ in range(batch):
                kv = rng.standard_normal((g.n_head, ctx, g.d_head))
                cache.append(s_, 0, kv, kv)
        xs = [rng.standard_normal((rows, g.d_model)) for _ in range(batch)]
        t_l = _time_layer(g, lay, xs, cache, list(range(batch)), [ctx] * batch)
        # logits of the rows the step consumes: all k+1 verify rows, one per
        # draft forward (the last prompt row)
        t_h = _time_head(head, [x[-(k + 1):] if name == "prefill_main" else x[-1:] if name != "verify" else x
                                for x in xs])
        out[name] = g.n_layer * t_l + t_h
        del lay, head, cache, xs
    return out
