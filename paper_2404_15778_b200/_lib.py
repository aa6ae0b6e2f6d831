"""ctypes binding of libbass.so (include/bass.h).

The CUDA library is the product: if it is missing or fails to load, every
entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BASS_LIB", os.path.join(_HERE, "libbass.so"))

BASS_OK, BASS_ERR_VALUE, BASS_ERR_CUDA, BASS_ERR_MEMORY, BASS_ERR_STATE = 0, -1, -2, -3, -4
BF16, F32, INT8 = 0, 1, 2
PAD, SPLIT, RAGGED = 0, 1, 2
GEMM_AUTO, GEMM_SIMT, GEMM_TC = 0, 1, 2
LOOP_HOST, LOOP_DEVICE = 0, 1
(W_TOK_EMB, W_POS_EMB, W_LN1_G, W_LN1_B, W_WQ, W_WK, W_WV, W_WO, W_LN2_G, W_LN2_B,
 W_FC, W_PROJ, W_LNF_G, W_LNF_B, W_HEAD) = range(15)

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
i8p = C.POINTER(C.c_int8)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class Geometry(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_layer", "n_head", "d_model", "d_head",
                                         "vocab_size", "max_seq_len")]


class GenRequest(C.Structure):
    _fields_ = [("batch", C.c_int32), ("prompt_tokens", i32p), ("prompt_offsets", i32p),
                ("max_new_tokens", C.c_int32), ("temperature", C.c_double),
                ("top_p", C.c_double), ("eos_token", C.c_int32), ("seed", C.c_uint64),
                ("sequence_ids", i64p), ("ctl_fixed", C.c_int32), ("l0", C.c_int32),
                ("incre", C.c_int32), ("mod", C.c_int32), ("limit", C.c_int32), ("s0", C.c_int32),
                ("align", C.c_double), ("align_seed", C.c_uint64), ("align_tokens", i32p)]


class GenResult(C.Structure):
    _fields_ = [("tokens", i32p), ("logprobs", f64p), ("n_tokens", i32p),
                ("finish_reason", i32p), ("completion_step", i32p), ("finish_wall_s", f64p),
                ("max_steps", C.c_int32), ("n_steps", C.c_int32), ("step_draft_len", i32p),
                ("step_accepted", i32p), ("step_emitted", i32p), ("step_kv_len", i32p),
                ("step_wall_s", f64p), ("main_forward_calls", C.c_int64),
                ("draft_forward_calls", C.c_int64), ("wall_s", C.c_double),
                ("final_l_draft", C.c_int32), ("final_s", C.c_int32),
                ("host_enqueue_s", C.c_double), ("sync_wait_s", C.c_double)]


# name -> (restype, argtypes); every symbol include/bass.h declares
SIGNATURES = {
    "bass_version": (C.c_int, []),
    "bass_device_arch": (C.c_int, [C.c_int]),
    "bass_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "bass_ctx_destroy": (C.c_int, [vp]),
    "bass_ctx_set_stream": (C.c_int, [vp, vp]),
    "bass_ctx_sync": (C.c_int, [vp]),
    "bass_last_error": (C.c_char_p, [vp]),
    "bass_ctx_launches": (C.c_int64, [vp]),
    "bass_ctx_transfer_bytes": (C.c_int, [vp, i64p, i64p]),
    "bass_ctx_profile": (C.c_int, [vp, C.c_int]),
    "bass_ctx_profile_read": (C.c_int, [vp, C.c_int, i64p, f64p, f64p, f64p]),
    "bass_ctx_algo_read": (C.c_int, [vp, C.c_int, i64p, f64p, f64p]),
    "bass_model_create": (C.c_int, [vp, C.POINTER(Geometry), C.c_int, C.POINTER(vp)]),
    "bass_model_destroy": (C.c_int, [vp]),
    "bass_model_set_weight": (C.c_int, [vp, C.c_int, C.c_int, f32p, C.c_int64]),
    "bass_model_get_weight": (C.c_int, [vp, C.c_int, C.c_int, f32p, C.c_int64]),
    "bass_model_init_random": (C.c_int, [vp, C.c_uint64, C.c_float]),
    "bass_model_get_qweight": (C.c_int, [vp, C.c_int, C.c_int, i8p, f64p, C.c_int64]),
    "bass_int_gemm_dequant": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, i8p, f64p, i8p, f64p, f32p]),
    "bass_model_set_gemm": (C.c_int, [vp, C.c_int]),
    "bass_model_weight_bytes": (C.c_int64, [vp]),
    "bass_model_set_split": (C.c_int, [vp, C.c_int, C.c_int, C.c_int]),
    "bass_kv_create": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "bass_kv_destroy": (C.c_int, [vp]),
    "bass_kv_lengths": (C.c_int, [vp, i32p]),
    "bass_kv_truncate": (C.c_int, [vp, C.c_int, i32p, i32p]),
    "bass_forward_ragged": (C.c_int, [vp, vp, C.c_int, i32p, i32p, i32p, C.c_int, C.c_int, f32p]),
    "bass_gemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
    "bass_gemm_bench": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, C.c_int,
                                  C.c_int, f64p]),
    "bass_attention": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p,
                                 vp, vp, vp, C.c_int, vp]),
    "bass_attention_bench": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, vp, vp, vp, C.c_int,
                                       C.c_int, vp, C.c_int, f64p]),
    "bass_trace_enable": (C.c_int, [vp, C.c_int64]),
    "bass_trace_read": (C.c_int, [vp, C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_int64)]),
    "bass_rng_uniforms": (C.c_int, [vp, C.c_int, C.c_uint64, i64p, i32p, i64p, f64p]),
    "bass_shape_sample": (C.c_int, [vp, C.c_int, C.c_int, f32p, C.c_double, C.c_double, f64p,
                                    i32p, f64p]),
    "bass_accept": (C.c_int, [vp, C.c_int, C.c_int, f32p, f32p, C.c_double, C.c_double, i32p,
                              C.c_uint64, i64p, i64p, i32p, i32p]),
    "bass_engine_create": (C.c_int, [vp, vp, vp, vp, C.POINTER(vp)]),
    "bass_engine_destroy": (C.c_int, [vp]),
    "bass_engine_set_strategy": (C.c_int, [vp, C.c_int]),
    "bass_engine_set_loop": (C.c_int, [vp, C.c_int]),
    "bass_engine_loop_info": (C.c_int, [vp, i32p, i32p, i64p]),
    "bass_spec_generate": (C.c_int, [vp, C.POINTER(GenRequest), C.POINTER(GenResult)]),
    "bass_regular_generate": (C.c_int, [vp, C.POINTER(GenRequest), C.POINTER(GenResult)]),
}

_lib = None
_alive = True


def _at_exit():
    global _alive
    _alive = False   # process teardown: the driver reclaims device memory


import atexit  # noqa: E402
atexit.register(_at_exit)


def alive() -> bool:
    return _alive


class BassError(RuntimeError):
    pass


def lib():
    """Load libbass.so once; raise (never fall back) when it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BassError(f"libbass.so not found at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _lib = L
    return _lib


def check(rc: int, ctx=None):
    """Map a C status to the reference's exception classes."""
    if rc == BASS_OK:
        return
    msg = lib().bass_last_error(ctx).decode() if ctx else f"libbass error {rc}"
    if rc == BASS_ERR_VALUE:
        raise ValueError(msg)
    raise BassError(msg)


def ptr(arr, ctype):
    """numpy array -> ctypes pointer (array must stay alive and contiguous)."""
    return arr.ctypes.data_as(C.POINTER(ctype))
