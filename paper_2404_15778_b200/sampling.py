"""Device sampling primitives (ref:sampling.py:53-146) exposed for parity
tests and for the generic host loop: keyed uniforms, shaping + inverse-CDF
sampling, and accept/resample — each one CUDA launch through libbass."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

ROLE_DRAFT = "draft"
ROLE_VERIFY = "verify"
_ROLE_CODES = {ROLE_DRAFT: 0, ROLE_VERIFY: 1}


def device_uniforms(ctx, seed, sids, roles, counters) -> np.ndarray:
    """[n, 2]: first two draws of default_rng(SeedSequence((seed, sid, role, ctr)))."""
    sid = np.ascontiguousarray(np.asarray(sids, dtype=np.int64))
    ctr = np.ascontiguousarray(np.asarray(counters, dtype=np.int64))
    rl = np.ascontiguousarray(np.asarray([_ROLE_CODES.get(r, r) for r in roles], dtype=np.int32))
    out = np.empty((sid.size, 2), dtype=np.float64)
    ctx.check(ctx.lib.bass_rng_uniforms(ctx.handle, sid.size, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        L.ptr(sid, C.c_int64), L.ptr(rl, C.c_int32),
                                        L.ptr(ctr, C.c_int64), L.ptr(out, C.c_double)))
    return out


def device_shape_sample(ctx, logits, temperature, top_p, u, want_probs=False):
    """Shape rows of logits and draw one token per row with uniform u[row]."""
    lg = np.ascontiguousarray(np.atleast_2d(np.asarray(logits, dtype=np.float32)))
    uu = np.ascontiguousarray(np.broadcast_to(np.asarray(u, dtype=np.float64), (lg.shape[0],)))
    tok = np.empty(lg.shape[0], dtype=np.int32)
    probs = np.empty(lg.shape, dtype=np.float64) if want_probs else None
    ctx.check(ctx.lib.bass_shape_sample(ctx.handle, lg.shape[0], lg.shape[1], L.ptr(lg, C.c_float),
                                        float(temperature), float(top_p), L.ptr(uu, C.c_double),
                                        L.ptr(tok, C.c_int32),
                                        L.ptr(probs, C.c_double) if want_probs else None))
    return (tok, probs) if want_probs else tok


def device_accept(ctx, q_logits, p_logits, temperature, top_p, tokens, seed, sids, counters):
    """Accept/resample decisions: (accepted[n] bool, corrected[n] int, -1 if accepted)."""
    ql = np.ascontiguousarray(np.atleast_2d(np.asarray(q_logits, dtype=np.float32)))
    pl = np.ascontiguousarray(np.atleast_2d(np.asarray(p_logits, dtype=np.float32)))
    n, V = ql.shape
    tk = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
    sid = np.ascontiguousarray(np.asarray(sids, dtype=np.int64))
    ctr = np.ascontiguousarray(np.asarray(counters, dtype=np.int64))
    acc = np.empty(n, dtype=np.int32)
    cor = np.empty(n, dtype=np.int32)
    ctx.check(ctx.lib.bass_accept(ctx.handle, n, V, L.ptr(ql, C.c_float), L.ptr(pl, C.c_float),
                                  float(temperature), float(top_p), L.ptr(tk, C.c_int32),
                                  int(seed) & 0xFFFFFFFFFFFFFFFF, L.ptr(sid, C.c_int64),
                                  L.ptr(ctr, C.c_int64), L.ptr(acc, C.c_int32),
                                  L.ptr(cor, C.c_int32)))
    return acc.astype(bool), cor
