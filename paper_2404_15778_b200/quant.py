"""INT8 W8A8 path (ref:quant.py:19-129) on the device.

The quantized inference path itself runs inside the forward of an int8
model (`DeviceWeights(..., dtype="int8")`, `RunConfig(quant_enabled=True)`):
weights are quantized per output channel on the device when they are
uploaded, activations per token by the row kernels in front of every
projection, and the projections are tcgen05 kind::i8 GEMMs.  This module
exposes the reference's data type and its integer GEMM for parity and
microbenchmarks; quantizing is host-free and happens on the device.
"""

from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib as L

QMAX = 127   # ref:quant.py:19


class GroupAxis(enum.Enum):
    """ref:quant.py:22-25."""
    PER_CHANNEL = "per_channel"
    PER_TOKEN = "per_token"
    PER_HEAD_TOKEN = "per_head_token"


@dataclass(frozen=True)
class QuantTensor:
    """ref:quant.py:28-41 (same validation)."""

    payload: np.ndarray
    scales: np.ndarray
    axis: GroupAxis
    n_head: int = 1

    def __post_init__(self):
        if self.payload.dtype != np.int8:
            raise ValueError("payload must be int8")
        if np.abs(self.payload.astype(np.int16)).max(initial=0) > QMAX:
            raise ValueError("payload out of [-127, 127]")
        if (np.asarray(self.scales) <= 0).any():
            raise ValueError("scales must be positive")


def int_gemm_dequant(aq: QuantTensor, wq: QuantTensor, ctx=None) -> np.ndarray:
    """out[t, c] = (sum_i aq[t, i] wq[i, c]) * scale_t * scale_c on the tcgen05
    kind::i8 GEMM (ref:quant.py:98-123, no bias / residual).  Returns fp32."""
    from .model import CudaContext
    if aq.axis is not GroupAxis.PER_TOKEN:
        raise ValueError("activations must be quantized per token")
    if wq.axis is not GroupAxis.PER_CHANNEL:
        raise ValueError("weights must be quantized per output channel")
    if aq.payload.shape[1] != wq.payload.shape[0]:
        raise ValueError(f"inner dims differ: {aq.payload.shape} @ {wq.payload.shape}")
    ctx = ctx or CudaContext.default()
    a = np.ascontiguousarray(aq.payload, dtype=np.int8)
    w = np.ascontiguousarray(wq.payload, dtype=np.int8)
    sa = np.ascontiguousarray(aq.scales, dtype=np.float64)
    sw = np.ascontiguousarray(wq.scales, dtype=np.float64)
    (M, K), N = a.shape, w.shape[1]
    out = np.empty((M, N), dtype=np.float32)
    ctx.check(ctx.lib.bass_int_gemm_dequant(ctx.handle, M, N, K, L.ptr(a, C.c_int8), L.ptr(sa, C.c_double),
                                            L.ptr(w, C.c_int8), L.ptr(sw, C.c_double), L.ptr(out, C.c_float)))
    return out
