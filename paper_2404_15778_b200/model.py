"""Device models behind the reference's LogitsProvider protocol.

`CudaModel` replaces `MainModel` (ref:model.py:288-332): it owns device
weights (libbass `bass_model`) and a ragged device KV cache (`bass_kv`), and
its `forward` runs the whole ragged block on the GPU.  Logits come back to
the host only because the protocol returns numpy arrays; the device-resident
decode path (`decode_speculative` with two CudaModels) never copies them.
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .attention import AttentionStrategy, strategy_code


@dataclass(frozen=True)
class ModelConfig:
    """ref:model.py:36-62 (same fields and validation)."""

    n_layer: int
    n_head: int
    d_model: int
    d_head: int
    vocab_size: int
    max_seq_len: int

    def __post_init__(self):
        for name in ("n_layer", "n_head", "d_model", "d_head", "vocab_size", "max_seq_len"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.d_model % self.n_head != 0:
            raise ValueError(f"d_model {self.d_model} not divisible by n_head {self.n_head}")
        if self.d_model != self.n_head * self.d_head:
            raise ValueError(f"d_model {self.d_model} != n_head {self.n_head} * d_head {self.d_head}")

    @property
    def d_ff(self) -> int:
        return 4 * self.d_model

    def geometry(self) -> L.Geometry:
        return L.Geometry(self.n_layer, self.n_head, self.d_model, self.d_head,
                          self.vocab_size, self.max_seq_len)


def desk_config(n_layer=4, n_head=8, d_model=256, vocab_size=512, max_seq_len=1024) -> ModelConfig:
    return ModelConfig(n_layer, n_head, d_model, d_model // n_head, vocab_size, max_seq_len)


class CudaContext:
    """One libbass context (device + stream) per GPU per process."""

    _default: dict[int, "CudaContext"] = {}

    def __init__(self, device: int = 0):
        self.lib = L.lib()
        h = C.c_void_p()
        L.check(self.lib.bass_ctx_create(device, C.byref(h)))
        self.handle, self.device = h, device

    @classmethod
    def default(cls, device: int = 0) -> "CudaContext":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def check(self, rc):
        L.check(rc, self.handle)

    @property
    def launches(self) -> int:
        return int(self.lib.bass_ctx_launches(self.handle))

    def sync(self):
        self.check(self.lib.bass_ctx_sync(self.handle))

    def set_stream(self, cuda_stream_ptr: int):
        """Enqueue libbass work on a caller stream (e.g. torch.cuda.Stream.cuda_stream)."""
        self.check(self.lib.bass_ctx_set_stream(self.handle, C.c_void_p(cuda_stream_ptr)))

    def transfer_bytes(self) -> tuple[int, int]:
        h, d = C.c_int64(), C.c_int64()
        self.check(self.lib.bass_ctx_transfer_bytes(self.handle, C.byref(h), C.byref(d)))
        return h.value, d.value

    PROFILE_CLASSES = ("gemm", "attention", "norm", "sampling")

    def profile(self, enable: bool):
        """Start (and reset) / stop per-kernel-class CUDA-event timing."""
        self.check(self.lib.bass_ctx_profile(self.handle, 1 if enable else 0))

    def algo_read(self) -> dict:
        """Cumulative algorithmic work per kernel class (launches, bytes, flops)."""
        out = {}
        for i, name in enumerate(self.PROFILE_CLASSES):
            n, by, fl = C.c_int64(), C.c_double(), C.c_double()
            self.check(self.lib.bass_ctx_algo_read(self.handle, i, C.byref(n), C.byref(by), C.byref(fl)))
            out[name] = {"launches": n.value, "bytes": by.value, "flops": fl.value}
        return out

    def trace(self, records: int):
        """Enable (records > 0, capacity) / disable (0) the per-CTA timeline trace."""
        self.check(self.lib.bass_trace_enable(self.handle, int(records)))

    def trace_read(self, max_records: int):
        """Records {t0, t1, smid, tag} (globaltimer ns) of the traced launches
        since enable, as an int64 [n, 4] array; resets the trace."""
        buf = np.zeros(int(max_records) * 4, np.uint64)
        n = C.c_int64()
        self.check(self.lib.bass_trace_read(self.handle, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            int(max_records), C.byref(n)))
        return buf[: 4 * n.value].reshape(-1, 4).astype(np.int64)

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(self.PROFILE_CLASSES):
            n, ms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            self.check(self.lib.bass_ctx_profile_read(self.handle, i, C.byref(n), C.byref(ms),
                                                      C.byref(by), C.byref(fl)))
            out[name] = {"launches": n.value, "ms": ms.value, "bytes": by.value,
                         "flops": fl.value}
        return out


def _dtype_code(dtype) -> int:
    if dtype in ("bf16", "bfloat16", L.BF16):
        return L.BF16
    if dtype in ("fp32", "float32", L.F32):
        return L.F32
    if dtype in ("int8", "w8a8", L.INT8):
        return L.INT8
    raise ValueError(f"unknown dtype {dtype!r}")


_LAYER_IDS = {"ln1_gain": L.W_LN1_G, "ln1_bias": L.W_LN1_B, "wq": L.W_WQ, "wk": L.W_WK,
              "wv": L.W_WV, "wo": L.W_WO, "ln2_gain": L.W_LN2_G, "ln2_bias": L.W_LN2_B,
              "w_fc": L.W_FC, "w_proj": L.W_PROJ}
_ORACLE_NAMES = {"token_emb": "tok_emb", "pos_emb": "pos_emb", "head": "head",
                 "ln_f_gain": "lnf_g", "ln_f_bias": "lnf_b", "ln1_gain": "ln1_g",
                 "ln1_bias": "ln1_b", "ln2_gain": "ln2_g", "ln2_bias": "ln2_b"}


def _reference_arrays(weights):
    """(config, top-level arrays, per-layer arrays) in the reference's names,
    from a reference `ModelWeights` object or an equivalent dict."""
    if isinstance(weights, dict):
        g = weights["geometry"]
        name = lambda k: _ORACLE_NAMES.get(k, k)
        top = {k: weights[name(k)] for k in ("token_emb", "pos_emb", "head", "ln_f_gain",
                                            "ln_f_bias")}
        layers = [{k: lay[name(k)] for k in _LAYER_IDS} for lay in weights["layers"]]
    else:
        g = weights.config
        top = {k: getattr(weights, k) for k in ("token_emb", "pos_emb", "head", "ln_f_gain",
                                               "ln_f_bias")}
        layers = [{k: getattr(b, k) for k in _LAYER_IDS} for b in weights.blocks]
    cfg = ModelConfig(g.n_layer, g.n_head, g.d_model, g.d_head, g.vocab_size, g.max_seq_len)
    return cfg, top, layers


class DeviceWeights:
    """A model's weights resident in HBM (ref:model.py:87-95 ModelWeights)."""

    def __init__(self, config: ModelConfig, dtype="bf16", ctx: CudaContext | None = None):
        self.config, self.ctx = config, ctx or CudaContext.default()
        self.dtype = _dtype_code(dtype)
        h = C.c_void_p()
        g = config.geometry()
        self.ctx.check(self.ctx.lib.bass_model_create(self.ctx.handle, C.byref(g), self.dtype,
                                                      C.byref(h)))
        self.handle = h

    # weight upload from reference-layout host arrays (input-major [in, out])
    def _put(self, tensor, layer, arr):
        a = np.ascontiguousarray(np.asarray(arr, dtype=np.float32))
        self.ctx.check(self.ctx.lib.bass_model_set_weight(self.handle, tensor, layer,
                                                          L.ptr(a, C.c_float), a.size))

    _SHAPES = {L.W_TOK_EMB: lambda c: (c.vocab_size, c.d_model), L.W_POS_EMB: lambda c: (c.max_seq_len, c.d_model),
               L.W_HEAD: lambda c: (c.d_model, c.vocab_size), L.W_WQ: lambda c: (c.d_model, c.d_model),
               L.W_WK: lambda c: (c.d_model, c.d_model), L.W_WV: lambda c: (c.d_model, c.d_model),
               L.W_WO: lambda c: (c.d_model, c.d_model), L.W_FC: lambda c: (c.d_model, 4 * c.d_model),
               L.W_PROJ: lambda c: (4 * c.d_model, c.d_model)}

    def get(self, tensor: int, layer: int = 0) -> np.ndarray:
        """One tensor back in the reference layout (float32 values as stored)."""
        shape = self._SHAPES.get(tensor, lambda c: (c.d_model,))(self.config)
        out = np.empty(shape, dtype=np.float32)
        self.ctx.check(self.ctx.lib.bass_model_get_weight(self.handle, tensor, layer, L.ptr(out, C.c_float),
                                                          out.size))
        return out

    @classmethod
    def from_reference(cls, weights, dtype="bf16", ctx=None) -> "DeviceWeights":
        """Upload a reference `ModelWeights` (or the oracle's dict) to the device."""
        cfg, top, layers = _reference_arrays(weights)
        dw = cls(cfg, dtype, ctx)
        for name, tid in (("token_emb", L.W_TOK_EMB), ("pos_emb", L.W_POS_EMB),
                          ("ln_f_gain", L.W_LNF_G), ("ln_f_bias", L.W_LNF_B), ("head", L.W_HEAD)):
            dw._put(tid, 0, top[name])
        for i, lay in enumerate(layers):
            for name, tid in _LAYER_IDS.items():
                dw._put(tid, i, lay[name])
        return dw

    @classmethod
    def init_model(cls, config: ModelConfig, seed: int, dtype="bf16", ctx=None) -> "DeviceWeights":
        """The reference's `init_model(config, seed)` (ref:model.py:106-132),
        value for value: one `default_rng(seed)` stream, N(0, 0.02) drawn on
        the float32 grid in the reference's order (token_emb, pos_emb, per
        layer wq wk wv wo w_fc w_proj, head), LN gains 1 / biases 0.  numpy's
        normal draws are chunk-invariant, so each tensor is drawn, uploaded
        (converted to `dtype` on the device) and dropped in turn — the fp64
        model is never materialised (65 GB at the 7.8B shape)."""
        dw = cls(config, dtype, ctx)
        rng = np.random.default_rng(seed)
        d, v, s, ff = config.d_model, config.vocab_size, config.max_seq_len, config.d_ff

        def draw(shape):
            return rng.normal(0.0, 0.02, size=shape).astype(np.float32)

        dw._put(L.W_TOK_EMB, 0, draw((v, d)))
        dw._put(L.W_POS_EMB, 0, draw((s, d)))
        one, zero = np.ones(d, np.float32), np.zeros(d, np.float32)
        for li in range(config.n_layer):
            for tid, shape in ((L.W_WQ, (d, d)), (L.W_WK, (d, d)), (L.W_WV, (d, d)), (L.W_WO, (d, d)),
                               (L.W_FC, (d, ff)), (L.W_PROJ, (ff, d))):
                dw._put(tid, li, draw(shape))
            for tid, val in ((L.W_LN1_G, one), (L.W_LN1_B, zero), (L.W_LN2_G, one), (L.W_LN2_B, zero)):
                dw._put(tid, li, val)
        dw._put(L.W_LNF_G, 0, one)
        dw._put(L.W_LNF_B, 0, zero)
        dw._put(L.W_HEAD, 0, draw((d, v)))
        return dw

    @classmethod
    def random(cls, config: ModelConfig, seed: int, dtype="bf16", std=0.02, ctx=None):
        """Device-side N(0, std) init for benchmark-scale shapes."""
        dw = cls(config, dtype, ctx)
        dw.ctx.check(dw.ctx.lib.bass_model_init_random(dw.handle, seed, std))
        return dw

    def gemm(self, x, w, mode: int = L.GEMM_TC):
        """Y = x @ w.T on the device with this model's GEMM kernels (torch
        CUDA tensors in the model dtype, contiguous; returns fp32 [M, N])."""
        import torch
        M, K = x.shape
        N = w.shape[0]
        x, w = x.contiguous(), w.contiguous()
        y = torch.empty((M, N), dtype=torch.float32, device=x.device)
        torch.cuda.synchronize(x.device)
        self.ctx.check(self.ctx.lib.bass_gemm(self.handle, mode, M, N, K, C.c_void_p(x.data_ptr()),
                                              C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr())))
        return y

    def qweight(self, tensor: int, layer: int = 0):
        """INT8 models: (payload [in, out] int8, scales [out] fp64) of one matrix
        as quantized on the device (ref:model.py:135-143, quant.py:55-63)."""
        shape = self._SHAPES[tensor](self.config)
        p = np.empty(shape, dtype=np.int8)
        s = np.empty(shape[1], dtype=np.float64)
        self.ctx.check(self.ctx.lib.bass_model_get_qweight(self.handle, tensor, layer, L.ptr(p, C.c_int8),
                                                           L.ptr(s, C.c_double), p.size))
        return p, s

    def set_split(self, N: int, K: int, splits: int):
        """Split-K count for the (N, K) projection (0: default rule)."""
        self.ctx.check(self.ctx.lib.bass_model_set_split(self.handle, N, K, splits))

    def set_gemm(self, mode: int):
        self.ctx.check(self.ctx.lib.bass_model_set_gemm(self.handle, mode))

    @property
    def nbytes(self) -> int:
        return int(self.ctx.lib.bass_model_weight_bytes(self.handle))

    def __del__(self):
        try:
            if getattr(self, "handle", None) and L.alive():
                self.ctx.lib.bass_model_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


class CudaModel:
    """LogitsProvider over device weights and a device ragged KV cache.

    ref:model.py:263-332.  Two calls with identical committed state and
    inputs return identical logits (all device reductions are in a fixed,
    batch-independent order).
    """

    def __init__(self, weights: DeviceWeights, n_seq: int,
                 strategy: AttentionStrategy = AttentionStrategy.PAD, capacity: int | None = None):
        self.weights = weights
        self.ctx = weights.ctx
        self.strategy = strategy
        self.n_seq = n_seq
        self.capacity = capacity or weights.config.max_seq_len
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.bass_kv_create(weights.handle, n_seq, self.capacity, C.byref(h)))
        self.kv = h

    @property
    def config(self) -> ModelConfig:
        return self.weights.config

    @property
    def vocab_size(self) -> int:
        return self.config.vocab_size

    @property
    def max_seq_len(self) -> int:
        return self.config.max_seq_len

    def lengths(self) -> list[int]:
        out = np.zeros(self.n_seq, dtype=np.int32)
        self.ctx.lib.bass_kv_lengths(self.kv, L.ptr(out, C.c_int32))
        return out.tolist()

    def length(self, seq: int) -> int:
        return self.lengths()[seq]

    def forward(self, active_seqs, new_tokens, last_only: bool = False):
        if len(active_seqs) != len(new_tokens) or not active_seqs:
            raise ValueError("active_seqs and new_tokens must align and be non-empty")
        slots = np.asarray(active_seqs, dtype=np.int32)
        lens = [len(t) for t in new_tokens]
        for s, n in zip(active_seqs, lens):
            if n < 1:
                raise ValueError(f"sequence {s}: empty token block")
        cu = np.zeros(len(lens) + 1, dtype=np.int32)
        cu[1:] = np.cumsum(lens)
        toks = np.asarray([t for blk in new_tokens for t in blk], dtype=np.int64)
        if toks.min() < 0 or toks.max() >= self.vocab_size:
            bad = next(s for s, blk in zip(active_seqs, new_tokens)
                       if min(blk) < 0 or max(blk) >= self.vocab_size)
            raise ValueError(f"sequence {bad}: token id outside vocab")
        toks = toks.astype(np.int32)
        rows = len(lens) if last_only else int(cu[-1])
        out = np.empty((rows, self.vocab_size), dtype=np.float32)
        self.ctx.check(self.ctx.lib.bass_forward_ragged(
            self.weights.handle, self.kv, len(lens), L.ptr(slots, C.c_int32), L.ptr(cu, C.c_int32),
            L.ptr(toks, C.c_int32), strategy_code(self.strategy), 1 if last_only else 0,
            L.ptr(out, C.c_float)))
        if last_only:
            return [out[i:i + 1].astype(np.float64) for i in range(len(lens))]
        return [out[cu[i]:cu[i + 1]].astype(np.float64) for i in range(len(lens))]

    def prefill(self, seq: int, prompt) -> np.ndarray:
        if len(prompt) == 0:
            raise ValueError("empty prompt: prefill needs at least one token")
        if self.length(seq) != 0:
            raise ValueError(f"sequence {seq} already has cached context")
        return self.forward([seq], [list(prompt)])[0][-1]

    def rollback(self, seq: int, length: int) -> None:
        s = np.asarray([seq], dtype=np.int32)
        n = np.asarray([length], dtype=np.int32)
        self.ctx.check(self.ctx.lib.bass_kv_truncate(self.kv, 1, L.ptr(s, C.c_int32),
                                                     L.ptr(n, C.c_int32)))

    def __del__(self):
        try:
            if getattr(self, "kv", None) and L.alive():
                self.ctx.lib.bass_kv_destroy(self.kv)
                self.kv = None
        except Exception:
            pass


class CudaAlignedDraft:
    """`SyntheticAlignedDraft` (ref:model.py:335-415) over a CudaModel.

    The inner forward runs on the GPU; the per-row perturbation is the
    reference's keyed blake2b draw over the token history (host bookkeeping,
    parity harness only — the benchmark uses the device-side override of
    `bass_gen_request.align`).
    """

    def __init__(self, weights: DeviceWeights, alignment: float, perturb_seed: int, n_seq: int,
                 strategy: AttentionStrategy = AttentionStrategy.PAD):
        if not 0.0 <= alignment <= 1.0:
            raise ValueError(f"alignment must be in [0, 1], got {alignment}")
        self.alignment, self.perturb_seed = float(alignment), int(perturb_seed)
        self.inner = CudaModel(weights, n_seq, strategy)
        self._hist = [[] for _ in range(n_seq)]

    vocab_size = property(lambda self: self.inner.vocab_size)
    max_seq_len = property(lambda self: self.inner.max_seq_len)

    def _draw(self, prefix):
        msg = self.perturb_seed.to_bytes(8, "little", signed=True) + \
            np.asarray(prefix, dtype=np.int64).tobytes()
        dg = hashlib.blake2b(msg, digest_size=16).digest()
        return int.from_bytes(dg[:8], "little") / 2.0 ** 64, \
            int.from_bytes(dg[8:], "little") % self.vocab_size

    def _mix(self, seq, raw, base):
        if self.alignment == 1.0:
            return raw
        out = raw.copy()
        for j in range(raw.shape[0]):
            u, y = self._draw(self._hist[seq][:base + j + 1])
            if u >= self.alignment:
                out[j] = -np.inf
                out[j, y] = 0.0
        return out

    def prefill(self, seq, prompt):
        base = len(self._hist[seq])
        raw = self.inner.prefill(seq, prompt)
        self._hist[seq] = list(prompt)
        return self._mix(seq, raw[None, :], base + len(prompt) - 1)[0]

    def forward(self, active_seqs, new_tokens):
        outs = []
        for s, toks, raw in zip(active_seqs, new_tokens, self.inner.forward(active_seqs, new_tokens)):
            base = len(self._hist[s])
            self._hist[s].extend(toks)
            outs.append(self._mix(s, raw, base))
        return outs

    def rollback(self, seq, length):
        self.inner.rollback(seq, length)
        del self._hist[seq][length:]

    def length(self, seq):
        return self.inner.length(seq)

    def lengths(self):
        return self.inner.lengths()
