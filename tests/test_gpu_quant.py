"""GPU parity of the INT8 W8A8 path (ref:quant.py:19-129,
model.py:135-143, 160-164, 219-222) through the C ABI.

* the tcgen05 kind::i8 GEMM with its dequantizing epilogue equals the
  reference's int_gemm_dequant rounded to fp32, bit for bit (the s32
  accumulation and the split-K reduction are exact integer sums; the scaling
  is the reference's fp64 product), at golden and headline shapes;
* device weight quantization equals the reference's payload and scales bit
  for bit;
* quantized ragged-forward logits match the reference's (golden, fp64) within
  the quantization-flip tolerance below — the residual stream, LayerNorm
  statistics and attention run in fp32 / bf16 on the device;
* greedy speculative == greedy regular on the int8 device path.
"""

import os

import numpy as np
import pytest

from oracle import engine as OE
from oracle import quant as OQ
from oracle import ragged as OR

pytestmark = pytest.mark.gpu

MODELS = {"a": OR.Geometry(2, 4, 128, 32, 512, 256), "b": OR.Geometry(2, 2, 256, 128, 384, 256)}


@pytest.fixture(scope="module")
def B():
    import paper_2404_15778_b200 as B
    return B


@pytest.fixture(scope="module")
def z(golden_dir):
    return np.load(os.path.join(golden_dir, "quant.npz"))


def _qt(B, p, s, axis):
    return B.QuantTensor(np.ascontiguousarray(p, dtype=np.int8), np.asarray(s, dtype=np.float64), axis)


def test_int_gemm_golden_bitwise(B, z):
    for c in range(6):
        out = B.int_gemm_dequant(_qt(B, z[f"k{c}_ap"], z[f"k{c}_as"], B.GroupAxis.PER_TOKEN),
                                 _qt(B, z[f"k{c}_wp"], z[f"k{c}_ws"], B.GroupAxis.PER_CHANNEL))
        np.testing.assert_array_equal(out, z[f"k{c}_out"].astype(np.float32))


@pytest.mark.parametrize("M,K,N", [(1, 4608, 13824), (88, 4608, 4608), (264, 18432, 4608),
                                   (300, 1024, 640), (17, 2048, 50272), (1100, 4608, 4608)])
def test_int_gemm_exact_at_model_shapes(B, M, K, N):
    rs = np.random.default_rng(M + K + N)
    a = rs.standard_normal((M, K)) * rs.uniform(0.5, 3, (M, 1))
    w = rs.standard_normal((K, N)).astype(np.float32).astype(np.float64) * 0.02
    ap, as_ = OQ.quantize_tokens(a)
    wp, ws = OQ.quantize_weights(w)
    want = OQ.int_gemm_dequant(ap, as_, wp, ws).astype(np.float32)
    got = B.int_gemm_dequant(_qt(B, ap, as_, B.GroupAxis.PER_TOKEN), _qt(B, wp, ws, B.GroupAxis.PER_CHANNEL))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("key", ["a", "b"])
def test_device_weight_quantization_bitwise(B, z, key):
    cfg = B.ModelConfig(*[getattr(MODELS[key], f) for f in ("n_layer", "n_head", "d_model", "d_head",
                                                              "vocab_size", "max_seq_len")])
    dw = B.DeviceWeights.init_model(cfg, 5, "int8")
    for name, tid in (("wq", B.model.L.W_WQ), ("w_proj", B.model.L.W_PROJ)):
        p, s = dw.qweight(tid, 1)
        np.testing.assert_array_equal(p, z[f"{key}_{name}1_p"])
        np.testing.assert_array_equal(s, z[f"{key}_{name}1_s"])
    p, s = dw.qweight(B.model.L.W_HEAD)
    np.testing.assert_array_equal(p, z[f"{key}_head_p"])
    np.testing.assert_array_equal(s, z[f"{key}_head_s"])
    # get_weight returns the dequantized values payload * scale
    hw = dw.get(B.model.L.W_HEAD)
    np.testing.assert_array_equal(hw, (p.astype(np.float64) * s[None, :]).astype(np.float32))


# Tolerance: the int8 path is a discontinuous function of its inputs (every
# quantizer rounds to a grid), so the device's fp32 LayerNorm / bf16
# embeddings, q / k / v and attention context move a few payloads by one step
# against the fp64 reference; tests/test_oracle_quant.py shows the REFERENCE
# itself moves by 2.2 % on average and up to 3.3-3.8 % (max over a row) under
# the bf16 embedding rounding alone at d = 128, and by 3.3 % / 4.3 % at the
# C2 width (d = 4608); the device measures 2.2 % / 3.2 % and 3.6 % / 4.2 %.
# The bound is therefore 8e-2 per row (max) and 5e-2 on the mean row error —
# a wrong scale, layout or rounding rule moves rows by tens of percent.
INT8_ROW_MAX, INT8_ROW_MEAN = 8e-2, 5e-2


def _row_errs(got, want):
    got, want = np.atleast_2d(got), np.atleast_2d(want)
    return list(np.abs(got - want).max(axis=1) / np.abs(want).max(axis=1))


@pytest.mark.parametrize("key", ["a", "b"])
@pytest.mark.parametrize("strategy", ["pad", "split", "ragged"])
def test_int8_forward_logits_vs_reference(B, z, key, strategy):
    g = MODELS[key]
    cfg = B.ModelConfig(g.n_layer, g.n_head, g.d_model, g.d_head, g.vocab_size, g.max_seq_len)
    dm = B.CudaModel(B.DeviceWeights.init_model(cfg, 5, "int8"), 4, strategy)
    prompts = [z[f"prompt_{i}"].tolist() for i in range(4)]
    blocks = [z[f"block_{i}"].tolist() for i in range(4)]
    ref = "split" if strategy == "split" else "pad"
    errs = []
    for i, p in enumerate(prompts):
        errs += _row_errs(dm.prefill(i, p), z[f"{key}_{ref}_prefill_{i}"])
    for i, o in enumerate(dm.forward([0, 1, 2, 3], blocks)):
        errs += _row_errs(o, z[f"{key}_{ref}_block_{i}"])
    assert max(errs) < INT8_ROW_MAX and np.mean(errs) < INT8_ROW_MEAN, (max(errs), np.mean(errs))


@pytest.mark.parametrize("key", ["a", "b"])
def test_int8_greedy_decode_vs_reference_and_spec_equals_regular(B, z, key):
    g = MODELS[key]
    cfg = B.ModelConfig(g.n_layer, g.n_head, g.d_model, g.d_head, g.vocab_size, g.max_seq_len)
    dw = B.DeviceWeights.init_model(cfg, 5, "int8")
    prompts = [z[f"prompt_{i}"].tolist()[:4] or [1] for i in range(4)]
    # teacher-forced greedy agreement on the reference's int8 greedy
    # trajectories (the structure of ref tests/test_acceptance.py:330-350):
    # every position's device argmax vs the reference's token.  A random-init
    # model's top logits are near-ties, so the quantization-flip noise above
    # changes some argmaxes: the reference itself agrees with its bf16-rounded
    # embeddings at 0.90 (a) / 0.94 (b) (tests/test_oracle_quant.py); >= 0.8.
    agree = total = 0
    for i, p in enumerate(prompts):
        ref = z[f"{key}_greedy_{i}"].tolist()
        out = B.CudaModel(dw, 1).forward([0], [p + ref])[0]
        agree += int((out[len(p) - 1:-1].argmax(axis=1) == np.asarray(ref)).sum())
        total += len(ref)
    assert agree >= 0.8 * total, (agree, total)
    req = B.GenerationRequest(prompts, 24, temperature=0.0)
    reg = B.decode_regular(B.CudaModel(dw, 4), req)
    spec = B.decode_speculative(B.CudaModel(dw, 4), B.CudaModel(dw, 4), req, B.AdaptiveDraftController())
    assert spec.tokens == reg.tokens


def test_int8_headline_shape_layer_vs_oracle(B):
    """One full-width C2 layer + head (d 4608, H 36, V 50272) on the int8
    path vs the oracle's int8 forward on the same reference-init weights."""
    g = OR.Geometry(1, 36, 4608, 128, 50272, 512)
    cfg = B.ModelConfig(1, 36, 4608, 128, 50272, 512)
    w = OR.init_weights(g, 2)
    dm = B.CudaModel(B.DeviceWeights.from_reference(w, "int8"), 2)
    om = OE.OracleModel(w, 2, quantized=True)
    rs = np.random.default_rng(9)
    prompts = [rs.integers(0, 50272, n).tolist() for n in (24, 9)]
    errs = []
    for s, p in enumerate(prompts):
        errs += _row_errs(dm.prefill(s, p), om.prefill(s, p))
    blocks = [rs.integers(0, 50272, n).tolist() for n in (11, 1)]
    for a, b in zip(dm.forward([0, 1], blocks), om.forward([0, 1], blocks)):
        errs += _row_errs(a, b)
    assert max(errs) < INT8_ROW_MAX and np.mean(errs) < INT8_ROW_MEAN, (max(errs), np.mean(errs))
    del cfg
