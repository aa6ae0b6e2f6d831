"""BASSCKPT weights straight to the device (ref:checkpoint.py).

The reference's container (ref:checkpoint.py:1-8): magic "BASSCKPT", format
version u32, array count u32, then per array: name length u32, UTF-8 name,
rank u32, dims u32 each, dtype tag u32 (0 = float32 LE), raw data; all
little-endian.  `load_checkpoint` reads it through a memory map and uploads
each float32 array as it is found (`bass_model_set_weight`: transposed,
converted to the model dtype and packed on the device), so a 7.8B-class
checkpoint never exists as float64 on the host (ref:checkpoint.py:91-143
builds a float64 `ModelWeights`).  Validation and error texts follow the
reference (`CheckpointError`: bad magic, version, dtype tag, unexpected
array, shape mismatch, missing arrays, truncated file).

`save_checkpoint` writes the same format from a `DeviceWeights` (read back
in the reference layout with `bass_model_get_weight`) or from a reference /
oracle weight object, so files round-trip with the reference's loader.
"""

from __future__ import annotations

import mmap
import struct
from pathlib import Path

import numpy as np

from . import _lib as L

MAGIC = b"BASSCKPT"
FORMAT_VERSION = 1
DTYPE_FLOAT32 = 0


class CheckpointError(ValueError):
    """ref:checkpoint.py:26-27."""


_LAYER_FIELDS = (("attn_norm.gain", L.W_LN1_G), ("attn_norm.bias", L.W_LN1_B), ("wq", L.W_WQ),
                 ("wk", L.W_WK), ("wv", L.W_WV), ("wo", L.W_WO), ("ffn_norm.gain", L.W_LN2_G),
                 ("ffn_norm.bias", L.W_LN2_B), ("w_fc", L.W_FC), ("w_proj", L.W_PROJ))


def manifest(config) -> dict:
    """name -> (shape, tensor id, layer) in the reference's file order
    (ref:checkpoint.py:30-49)."""
    d, v, s, f = config.d_model, config.vocab_size, config.max_seq_len, 4 * config.d_model
    shapes = {"attn_norm.gain": (d,), "attn_norm.bias": (d,), "wq": (d, d), "wk": (d, d),
              "wv": (d, d), "wo": (d, d), "ffn_norm.gain": (d,), "ffn_norm.bias": (d,),
              "w_fc": (d, f), "w_proj": (f, d)}
    out = {"token_embedding": ((v, d), L.W_TOK_EMB, 0), "position_embedding": ((s, d), L.W_POS_EMB, 0)}
    for i in range(config.n_layer):
        for k, tid in _LAYER_FIELDS:
            out[f"layer{i}.{k}"] = (shapes[k], tid, i)
    out["final_norm.gain"] = ((d,), L.W_LNF_G, 0)
    out["final_norm.bias"] = ((d,), L.W_LNF_B, 0)
    out["output_head"] = ((d, v), L.W_HEAD, 0)
    return out


def iter_checkpoint(path, config):
    """Yield (name, float32 array view, tensor id, layer) for every array of
    a checkpoint, validated against `config` as the reference loader does.
    The arrays are zero-copy views of a read-only memory map."""
    expected = manifest(config)
    seen = set()
    with open(path, "rb") as fh:
        size = fh.seek(0, 2)
        if size == 0:
            raise CheckpointError("truncated checkpoint")
        mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
    buf = memoryview(mm)
    pos = 0

    def take(n):
        nonlocal pos
        if pos + n > len(buf):
            raise CheckpointError("truncated checkpoint")
        b = buf[pos:pos + n]
        pos += n
        return b

    if bytes(take(len(MAGIC))) != MAGIC:
        raise CheckpointError("bad magic: not a checkpoint file")
    version, count = struct.unpack("<II", take(8))
    if version != FORMAT_VERSION:
        raise CheckpointError(f"unsupported format version {version}")
    for _ in range(count):
        (name_len,) = struct.unpack("<I", take(4))
        name = bytes(take(name_len)).decode("utf-8")
        (rank,) = struct.unpack("<I", take(4))
        shape = struct.unpack(f"<{rank}I", take(4 * rank))
        (tag,) = struct.unpack("<I", take(4))
        if tag != DTYPE_FLOAT32:
            raise CheckpointError(f"{name}: unsupported dtype tag {tag}")
        n_elem = int(np.prod(shape, dtype=np.int64)) if rank else 1
        raw = take(4 * n_elem)
        if name not in expected:
            raise CheckpointError(f"unexpected array {name!r}")
        if tuple(shape) != expected[name][0]:
            raise CheckpointError(f"{name}: shape {tuple(shape)} does not match config {expected[name][0]}")
        seen.add(name)
        _, tid, layer = expected[name]
        yield name, np.frombuffer(raw, dtype="<f4").reshape(shape), tid, layer
    missing = set(expected) - seen
    if missing:
        raise CheckpointError(f"missing arrays: {sorted(missing)}")


def load_checkpoint(path, config, dtype="bf16", ctx=None):
    """Checkpoint -> `DeviceWeights` (ref:checkpoint.py:91-143, device-resident)."""
    from .model import DeviceWeights
    dw = DeviceWeights(config, dtype, ctx)
    for _, arr, tid, layer in iter_checkpoint(path, config):
        dw._put(tid, layer, arr)
    return dw


def _reference_tensors(weights):
    """name -> float array from a DeviceWeights, a reference ModelWeights or
    the oracle's dict."""
    from .model import DeviceWeights, _reference_arrays
    if isinstance(weights, DeviceWeights):
        cfg = weights.config
        return cfg, ((name, weights.get(tid, layer)) for name, (_, tid, layer) in manifest(cfg).items())
    cfg, top, layers = _reference_arrays(weights)
    ref_names = {"token_embedding": "token_emb", "position_embedding": "pos_emb",
                 "final_norm.gain": "ln_f_gain", "final_norm.bias": "ln_f_bias", "output_head": "head"}
    lay_names = {"attn_norm.gain": "ln1_gain", "attn_norm.bias": "ln1_bias", "ffn_norm.gain": "ln2_gain",
                 "ffn_norm.bias": "ln2_bias"}

    def gen():
        for name in manifest(cfg):
            if name.startswith("layer"):
                i, k = name[5:].split(".", 1)
                yield name, layers[int(i)][lay_names.get(k, k)]
            else:
                yield name, top[ref_names[name]]
    return cfg, gen()


def save_checkpoint(weights, path) -> None:
    """ref:checkpoint.py:65-79 (same byte layout)."""
    cfg, tensors = _reference_tensors(weights)
    names = list(manifest(cfg))
    with open(Path(path), "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<II", FORMAT_VERSION, len(names)))
        for name, arr in tensors:
            data = np.ascontiguousarray(arr, dtype="<f4")
            enc = name.encode("utf-8")
            fh.write(struct.pack("<I", len(enc)))
            fh.write(enc)
            fh.write(struct.pack("<I", data.ndim))
            fh.write(struct.pack(f"<{data.ndim}I", *data.shape))
            fh.write(struct.pack("<I", DTYPE_FLOAT32))
            fh.write(data.tobytes())


__all__ = ["CheckpointError", "load_checkpoint", "save_checkpoint", "iter_checkpoint", "manifest",
           "MAGIC", "FORMAT_VERSION"]
