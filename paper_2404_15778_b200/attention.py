"""Ragged attention strategies (ref:attention.py:30-154) on the GPU.

PAD and SPLIT keep the reference's meaning (`AttentionStrategy`,
ref:attention.py:30-32): PAD is one launch over the batch padded to the
longest query block and the longest history (padded keys masked to an exact
zero probability, so the padded work is real and wasted, as in the paper);
SPLIT is one launch per sequence.  RAGGED (new) is a single launch over an
exact work list — no padding, no per-sequence launches.  All three produce
bitwise-identical context vectors because a row's reduction order is fixed
by absolute key positions.
"""

from __future__ import annotations

import ctypes as C
import enum

import numpy as np

from . import _lib as L


class AttentionStrategy(enum.Enum):
    PAD = "pad"
    SPLIT = "split"
    RAGGED = "ragged"


def strategy_code(s) -> int:
    s = AttentionStrategy(s.value if isinstance(s, enum.Enum) else s)
    return {AttentionStrategy.PAD: L.PAD, AttentionStrategy.SPLIT: L.SPLIT,
            AttentionStrategy.RAGGED: L.RAGGED}[s]


def attend_device(ctx, q, k, v, cu_q, offsets, strategy=AttentionStrategy.RAGGED, out=None):
    """Ragged attention over torch CUDA tensors.

    q: [M, H, dh]; k, v: [n_seq, H, stride, dh] (sequence i's history in
    entry i); cu_q: CSR row offsets (host ints); offsets[i]: committed length
    before sequence i's block.  dtype bf16 or fp32.  Returns [M, H, dh].
    """
    import torch

    if q.dtype == torch.bfloat16:
        code = L.BF16
    elif q.dtype == torch.float32:
        code = L.F32
    else:
        raise ValueError("q/k/v must be bf16 or fp32")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("attend_device needs CUDA tensors")
    n_seq, H, stride, dh = k.shape
    cu = np.ascontiguousarray(np.asarray(cu_q, dtype=np.int32))
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32))
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, device=q.device)
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    torch.cuda.synchronize(q.device)
    ctx.check(ctx.lib.bass_attention(ctx.handle, strategy_code(strategy), code, n_seq, H, dh,
                                     L.ptr(cu, C.c_int32), L.ptr(off, C.c_int32),
                                     C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                     C.c_void_p(v.data_ptr()), stride, C.c_void_p(out.data_ptr())))
    return out
