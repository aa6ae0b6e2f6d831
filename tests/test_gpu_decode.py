"""GPU parity of the full hot path: ragged forward (teacher-forced logits) and
the decode loops (device-resident and host-loop paths) against the
reference's golden runs and the oracle.

Parity ladder: fp32 mode (true FFMA) reproduces the fp64
reference's tokens exactly; bf16 mode matches the oracle fed the same
bf16-rounded weights within 1e-2 relative per logits row, and bf16 greedy
speculative == bf16 greedy regular on the GPU.
"""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import engine as OE
from oracle import ragged as OR

pytestmark = pytest.mark.gpu

TINY = OR.Geometry(2, 4, 64, 16, 96, 256)
C1_MAIN = OR.Geometry(2, 4, 128, 32, 512, 1024)
C1_DRAFT = OR.Geometry(1, 4, 128, 32, 512, 1024)


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def B():
    import paper_2404_15778_b200 as B
    return B


def _bf16_round(w):
    import torch
    out = {}
    for k, v in w.items():
        if k == "layers":
            out[k] = [{kk: torch.tensor(vv).bfloat16().double().numpy() if kk.startswith("w")
                       else vv for kk, vv in lay.items()} for lay in v]
        elif isinstance(v, np.ndarray) and k in ("tok_emb", "pos_emb", "head"):
            out[k] = torch.tensor(v).bfloat16().double().numpy()
        else:
            out[k] = v
    return out


@pytest.mark.parametrize("strategy", ["pad", "split", "ragged"])
def test_forward_fp32_matches_reference_golden(B, golden_dir, strategy):
    z = np.load(os.path.join(golden_dir, "forward.npz"))
    meta = _load(golden_dir, "forward.json")
    w = OR.init_weights(TINY, 5)
    m = B.CudaModel(B.DeviceWeights.from_reference(w, "fp32"), 4, strategy)
    for s, p in enumerate(meta["prompts"]):
        got = m.prefill(s, p)
        want = z[f"pad_prefill_{s}"]
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
    outs = m.forward([0, 1, 2, 3], meta["blocks"])
    for s in range(4):
        want = z[f"pad_block_{s}"]
        assert outs[s].shape == want.shape
        assert np.abs(outs[s] - want).max() <= 1e-5 * np.abs(want).max()
    assert m.lengths() == [7, 8, 11, 4]


def test_forward_bf16_within_1e2_of_oracle_on_rounded_weights(B):
    g = OR.Geometry(4, 8, 512, 64, 2048, 512)
    w = _bf16_round(OR.init_weights(g, 11))
    rng = np.random.default_rng(4)
    prompts = [rng.integers(0, 2048, n).tolist() for n in (40, 7, 120, 64)]
    blocks = [rng.integers(0, 2048, n).tolist() for n in (8, 8, 1, 33)]
    om = OE.OracleModel(w, 4)
    dm = B.CudaModel(B.DeviceWeights.from_reference(w, "bf16"), 4)
    for s, p in enumerate(prompts):
        om.prefill(s, p)
        dm.prefill(s, p)
    ref = om.forward([0, 1, 2, 3], blocks)
    got = dm.forward([0, 1, 2, 3], blocks)
    worst = 0.0
    for a, b in zip(got, ref):
        err = np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)
        worst = max(worst, float(err.max()))
    assert worst < 1e-2, worst


def test_forward_batch_invariance_and_block_equals_sequential(B):
    g = OR.Geometry(2, 4, 256, 64, 1000, 256)
    w = OR.init_weights(g, 3)
    dw = B.DeviceWeights.from_reference(w, "bf16")
    a, b = B.CudaModel(dw, 3), B.CudaModel(dw, 3)
    for m in (a, b):
        m.prefill(0, [1, 2, 3])
        m.prefill(1, [4, 5])
        m.prefill(2, [9, 9, 9, 9])
    together = a.forward([0, 1, 2], [[7, 8, 9], [11], [3, 4]])
    alone = [b.forward([s], [t])[0] for s, t in ((0, [7, 8, 9]), (1, [11]), (2, [3, 4]))]
    for x, y in zip(together, alone):
        assert np.array_equal(x, y)          # bitwise: row-independent kernels
    c = B.CudaModel(dw, 1)
    c.prefill(0, [1, 2, 3])
    seq = [c.forward([0], [[t]])[0][0] for t in (7, 8, 9)]
    assert np.array_equal(np.stack(seq), together[0])


def test_rollback_then_reappend_is_bitwise(B):
    g = OR.Geometry(2, 4, 128, 32, 300, 128)
    dw = B.DeviceWeights.from_reference(OR.init_weights(g, 1), "bf16")
    m = B.CudaModel(dw, 1)
    m.prefill(0, [5, 6, 7])
    first = m.forward([0], [[1, 2, 3, 4]])[0]
    m.rollback(0, 3)
    assert m.length(0) == 3
    again = m.forward([0], [[1, 2, 3, 4]])[0]
    assert np.array_equal(first, again)
    with pytest.raises(ValueError):
        m.rollback(0, 99)


def test_error_contracts(B):
    g = OR.Geometry(1, 2, 64, 32, 64, 8)
    m = B.CudaModel(B.DeviceWeights.from_reference(OR.init_weights(g, 1), "fp32"), 1)
    with pytest.raises(ValueError, match="empty prompt"):
        m.prefill(0, [])
    m.prefill(0, [1, 2])
    with pytest.raises(ValueError, match="cached context"):
        m.prefill(0, [1, 2])
    with pytest.raises(ValueError, match="max_seq_len"):
        m.forward([0], [[1] * 9])
    with pytest.raises(ValueError, match="vocab"):
        m.forward([0], [[99]])


def _check(res, ref, steps=True):
    assert res.tokens == ref["tokens"]
    assert res.finish_reason == ref["finish_reason"]
    assert res.completion_step == ref["completion_step"]
    assert res.main_forward_calls == ref["main_calls"]
    assert res.draft_forward_calls == ref["draft_calls"]
    for a, b in zip(res.logprobs, ref["logprobs"]):
        np.testing.assert_allclose(a, b, rtol=0, atol=2e-4)
    if steps:
        assert len(res.steps) == len(ref["steps"])
        for s, r in zip(res.steps, ref["steps"]):
            assert s.draft_length == r["draft_length"]
            assert list(s.slots) == r["slots"]
            assert list(s.accepted) == r["accepted"]
            assert [list(e) for e in s.emitted] == r["emitted"]
            assert list(s.finished) == r["finished"]
            assert list(s.kv_lengths) == r["kv_lengths"]


@pytest.mark.parametrize("strategy", ["pad", "split"])
def test_c1_greedy_device_path_matches_reference(B, golden_dir, strategy):
    d = _load(golden_dir, "decode.json")
    wm, wd = OR.init_weights(C1_MAIN, 0), OR.init_weights(C1_DRAFT, 1)
    dwm, dwd = B.DeviceWeights.from_reference(wm, "fp32"), B.DeviceWeights.from_reference(wd, "fp32")
    req = B.GenerationRequest(d["c1_prompts"], 64, temperature=0.0)
    reg = B.decode_regular(B.CudaModel(dwm, 4, strategy), req)
    _check(reg, d["runs"][f"c1_regular_{strategy}"], steps=False)
    main, draft = B.CudaModel(dwm, 4, strategy), B.CudaModel(dwd, 4, strategy)
    spec = B.decode_speculative(main, draft, req, B.FixedDraftController(4))
    _check(spec, d["runs"][f"c1_spec_{strategy}"])
    for s in range(4):
        committed = len(d["c1_prompts"][s]) + len(spec.tokens[s])
        assert main.length(s) == committed - 1
        assert committed - 2 <= draft.length(s) <= committed - 1


def test_c1_synthetic_aligned_draft_host_loop(B, golden_dir):
    d = _load(golden_dir, "decode.json")
    dwm = B.DeviceWeights.from_reference(OR.init_weights(C1_MAIN, 0), "fp32")
    req = B.GenerationRequest(d["c1_prompts"], 64, temperature=0.0)
    spec = B.decode_speculative(B.CudaModel(dwm, 4), B.CudaAlignedDraft(dwm, 0.8, 17, 4), req,
                                B.AdaptiveDraftController())
    _check(spec, d["runs"]["c1_spec_synth08"])


def test_tiny_sampled_device_path_matches_reference(B, golden_dir):
    d = _load(golden_dir, "decode.json")
    tw = B.DeviceWeights.from_reference(OR.init_weights(TINY, 1234), "fp32")
    req = B.GenerationRequest(d["tiny_prompts"], 12, temperature=0.7, top_p=0.9, seed=1234)
    res = B.decode_regular(B.CudaModel(tw, 2), req)
    _check(res, d["runs"]["tiny_regular_sampled"], steps=False)
    assert res.tokens == [[38, 32, 87, 74, 67, 27, 25, 29, 14, 19, 1, 62],
                          [76, 95, 58, 30, 94, 4, 73, 41, 86, 32, 41, 19]]
    dw = B.DeviceWeights.from_reference(OR.init_weights(OR.Geometry(1, 4, 64, 16, 96, 256), 99),
                                        "fp32")
    sreq = B.GenerationRequest(d["eos_prompts"], 30, temperature=1.0, top_p=0.95, seed=8,
                               eos_token=7, sequence_ids=[5, 0, 11])
    ctl = B.AdaptiveDraftController(B.DraftLengthParams(l0=3, incre=2, mod=10, limit=8))
    spec = B.decode_speculative(B.CudaModel(tw, 3), B.CudaModel(dw, 3), sreq, ctl)
    _check(spec, d["runs"]["tiny_spec_sampled_realdraft"])
    reg = B.decode_regular(B.CudaModel(tw, 3), sreq)
    _check(reg, d["runs"]["tiny_regular_sampled_eos"], steps=False)


def test_tiny_sampled_synthetic_host_loop(B, golden_dir):
    d = _load(golden_dir, "decode.json")
    tw = B.DeviceWeights.from_reference(OR.init_weights(TINY, 1234), "fp32")
    req = B.GenerationRequest(d["tiny_prompts"], 40, temperature=0.7, top_p=0.9, seed=1234)
    spec = B.decode_speculative(B.CudaModel(tw, 2), B.CudaAlignedDraft(tw, 0.8, 1234 + 17, 2), req,
                                B.AdaptiveDraftController())
    _check(spec, d["runs"]["tiny_spec_sampled"])


def test_device_and_host_loops_agree_sampled(B):
    """The device-resident loop and the host loop over the same CudaModels."""
    from paper_2404_15778_b200 import engine as E
    g = OR.Geometry(2, 4, 128, 32, 700, 256)
    gd = OR.Geometry(1, 4, 128, 32, 700, 256)
    dwm = B.DeviceWeights.from_reference(OR.init_weights(g, 21), "bf16")
    dwd = B.DeviceWeights.from_reference(OR.init_weights(gd, 22), "bf16")
    rng = np.random.default_rng(9)
    prompts = [rng.integers(0, 700, int(n)).tolist() for n in (5, 17, 9, 30)]
    for temp, top_p in ((0.0, 1.0), (0.9, 0.95), (0.3, 0.8)):
        req = B.GenerationRequest(prompts, 24, temperature=temp, top_p=top_p, seed=3, eos_token=11)
        dev = B.decode_speculative(B.CudaModel(dwm, 4), B.CudaModel(dwd, 4), req,
                                   B.AdaptiveDraftController(B.DraftLengthParams(l0=4, limit=12)))
        host = E._host_speculative(B.CudaModel(dwm, 4), B.CudaModel(dwd, 4), req,
                                   B.AdaptiveDraftController(B.DraftLengthParams(l0=4, limit=12)))
        assert dev.tokens == host.tokens
        assert [s.accepted for s in dev.steps] == [s.accepted for s in host.steps]
        assert dev.draft_forward_calls == host.draft_forward_calls


def test_bf16_greedy_speculative_equals_regular(B):
    g = OR.Geometry(4, 8, 512, 64, 4096, 512)
    gd = OR.Geometry(1, 8, 512, 64, 4096, 512)
    dwm = B.DeviceWeights.from_reference(OR.init_weights(g, 7), "bf16")
    dwd = B.DeviceWeights.from_reference(OR.init_weights(gd, 8), "bf16")
    rng = np.random.default_rng(2)
    prompts = [rng.integers(0, 4096, int(n)).tolist() for n in rng.integers(4, 60, 8)]
    req = B.GenerationRequest(prompts, 48, temperature=0.0)
    base = B.decode_regular(B.CudaModel(dwm, 8), req)
    spec = B.decode_speculative(B.CudaModel(dwm, 8), B.CudaModel(dwd, 8), req,
                                B.AdaptiveDraftController())
    assert spec.tokens == base.tokens
    # self-draft (draft = main weights): everything accepted, still identical
    spec2 = B.decode_speculative(B.CudaModel(dwm, 8), B.CudaModel(dwm, 8), req,
                                 B.AdaptiveDraftController())
    assert spec2.tokens == base.tokens
    assert sum(sum(s.accepted) for s in spec2.steps) > 0


def test_engine_validation_messages(B):
    g = OR.Geometry(1, 2, 64, 32, 64, 40)
    dw = B.DeviceWeights.from_reference(OR.init_weights(g, 2), "fp32")
    req = B.GenerationRequest([[1, 2, 3]], 20, temperature=0.0)
    with pytest.raises(ValueError, match="context overflow"):
        B.decode_speculative(B.CudaModel(dw, 1), B.CudaModel(dw, 1), req,
                             B.AdaptiveDraftController())
    g2 = OR.Geometry(1, 2, 64, 32, 80, 40)
    dw2 = B.DeviceWeights.from_reference(OR.init_weights(g2, 2), "fp32")
    with pytest.raises(ValueError, match="vocab"):
        B.decode_speculative(B.CudaModel(dw, 1), B.CudaModel(dw2, 1), req,
                             B.AdaptiveDraftController())
    with pytest.raises(ValueError, match="max_seq_len"):
        B.decode_regular(B.CudaModel(dw, 1), B.GenerationRequest([list(range(30))], 20))


def test_bf16_dh128_tcgen05_attention_path(B):
    """d_head = 128 routes attention through the TMA + tcgen05 kernel: logits
    within 1e-2 of the oracle (bf16-rounded weights), batch-invariant, and
    greedy speculative == regular."""
    g = OR.Geometry(3, 4, 512, 128, 1500, 600)
    gd = OR.Geometry(1, 4, 512, 128, 1500, 600)
    w = _bf16_round(OR.init_weights(g, 31))
    rng = np.random.default_rng(6)
    prompts = [rng.integers(0, 1500, n).tolist() for n in (150, 7, 300, 64)]
    blocks = [rng.integers(0, 1500, n).tolist() for n in (9, 9, 1, 33)]
    om = OE.OracleModel(w, 4)
    dwm = B.DeviceWeights.from_reference(w, "bf16")
    dm = B.CudaModel(dwm, 4)
    for s, p in enumerate(prompts):
        om.prefill(s, p)
        dm.prefill(s, p)
    ref = om.forward([0, 1, 2, 3], blocks)
    got = dm.forward([0, 1, 2, 3], blocks)
    for a, b in zip(got, ref):
        err = np.abs(a - b).max(axis=1) / np.abs(b).max(axis=1)
        assert float(err.max()) < 1e-2, float(err.max())
    solo = B.CudaModel(dwm, 4)
    solo.prefill(2, prompts[2])
    assert np.array_equal(solo.forward([2], [blocks[2]])[0], got[2])
    dwd = B.DeviceWeights.from_reference(OR.init_weights(gd, 32), "bf16")
    req = B.GenerationRequest([p[:40] for p in prompts], 40, temperature=0.0)
    base = B.decode_regular(B.CudaModel(dwm, 4), req)
    spec = B.decode_speculative(B.CudaModel(dwm, 4), B.CudaModel(dwm, 4), req,
                                B.AdaptiveDraftController())
    assert spec.tokens == base.tokens
    spec2 = B.decode_speculative(B.CudaModel(dwm, 4), B.CudaModel(dwd, 4), req,
                                 B.AdaptiveDraftController())
    assert spec2.tokens == base.tokens


def test_folded_layernorm_matches_unfused(B):
    """Default bf16 path (LayerNorms folded into the tcgen05 QKV / FC / head
    GEMM epilogues, centred row statistics produced by the residual
    epilogues) vs the same bf16 weights on the SIMT GEMMs with separate
    two-pass LayerNorm kernels: logits within 1e-2 per row, and greedy
    speculative == regular on the folded path."""
    from paper_2404_15778_b200 import _lib as L
    g = OR.Geometry(3, 4, 512, 128, 1500, 600)
    w = _bf16_round(OR.init_weights(g, 51))
    rng = np.random.default_rng(8)
    prompts = [rng.integers(0, 1500, n).tolist() for n in (40, 9, 70, 25)]
    blocks = [rng.integers(0, 1500, n).tolist() for n in (5, 1, 12, 3)]
    outs = []
    for mode in (L.GEMM_AUTO, L.GEMM_SIMT):
        dw = B.DeviceWeights.from_reference(w, "bf16")
        dw.set_gemm(mode)
        m = B.CudaModel(dw, 4)
        for s, p in enumerate(prompts):
            m.prefill(s, p)
        outs.append(np.concatenate(m.forward([0, 1, 2, 3], blocks)))
    err = np.abs(outs[1] - outs[0]).max(axis=1) / np.abs(outs[1]).max(axis=1)
    assert float(err.max()) < 1e-2, float(err.max())
    dw = B.DeviceWeights.from_reference(w, "bf16")
    dd = B.DeviceWeights.from_reference(_bf16_round(OR.init_weights(OR.Geometry(1, 4, 512, 128, 1500, 600), 52)),
                                        "bf16")
    req = B.GenerationRequest(prompts, 24, temperature=0.0)
    base = B.decode_regular(B.CudaModel(dw, 4), req)
    spec = B.decode_speculative(B.CudaModel(dw, 4), B.CudaModel(dd, 4), req, B.AdaptiveDraftController())
    assert spec.tokens == base.tokens


def test_draft_self_speculation_accepts_every_proposal(B):
    """Draft == main (same bf16 weights, separate caches), greedy, natural
    acceptance: every proposal is the main model's own greedy token (rows are
    bitwise batch-invariant), so every step accepts its whole draft.  Exercises
    the greedy draft pick from the folded LM head's per-tile argmax partials
    (a wrong pick would be rejected)."""
    w = B.DeviceWeights.from_reference(_bf16_round(OR.init_weights(OR.Geometry(2, 4, 512, 128, 1500, 600), 71)),
                                       "bf16")
    rng = np.random.default_rng(12)
    prompts = [rng.integers(0, 1500, n).tolist() for n in (33, 20, 57)]
    main_m, draft_m = B.CudaModel(w, 3), B.CudaModel(w, 3)
    eng = B.CudaEngine(main_m, draft_m)
    req = B.GenerationRequest(prompts, 20, temperature=0.0, sequence_ids=[0, 1, 2])
    res, _ = eng.run(req, B.FixedDraftController(4), speculative=True)[:2]
    steps = list(res.steps)
    assert len(steps) >= 2
    for s in steps[:-1]:   # the last step may be clipped at max_new_tokens
        assert all(a == s.draft_length for a in s.accepted), (s.step_index, s.accepted, s.draft_length)


def test_timeline_trace_records_every_cta(B):
    """bass_trace_enable / bass_trace_read: one record per CTA of every traced
    launch, with ordered timestamps and valid SM ids."""
    import ctypes as C
    w = _bf16_round(OR.init_weights(OR.Geometry(2, 4, 512, 128, 1500, 600), 61))
    m = B.CudaModel(B.DeviceWeights.from_reference(w, "bf16"), 2)
    ctx = m.ctx
    ctx.check(ctx.lib.bass_trace_enable(ctx.handle, 1 << 16))
    m.prefill(0, list(range(1, 30)))
    buf = np.zeros((1 << 16) * 4, np.uint64)
    n = C.c_int64()
    ctx.check(ctx.lib.bass_trace_read(ctx.handle, buf.ctypes.data_as(C.POINTER(C.c_uint64)), 1 << 16, C.byref(n)))
    ctx.check(ctx.lib.bass_trace_enable(ctx.handle, 0))
    rec = buf[: 4 * n.value].reshape(-1, 4).astype(np.int64)
    assert n.value > 0
    assert (rec[:, 1] >= rec[:, 0]).all() and (rec[:, 0] > 0).all()
    assert (rec[:, 2] < 1024).all()
    classes = set((rec[:, 3] & 15).tolist())
    assert {1, 2} <= classes   # GEMM, attention (the LayerNorms are folded into the GEMMs)


def test_sequence_ids_beyond_int32_and_long_drafts_match_oracle(B):
    """Contract fidelity (ref:engine.py:36-61 accepts any non-negative id;
    ref:draft_control.py:17-29 any limit >= 1): sequence ids above 2^32 key
    the per-sequence RNG exactly like the reference, and a fixed draft of 70
    tokens (beyond any fixed emit buffer) runs; sampled, fp32 parity mode,
    tokens / logprobs / step counters equal to the oracle engine."""
    g = OR.Geometry(1, 4, 64, 16, 96, 512)
    tw = B.DeviceWeights.from_reference(OR.init_weights(TINY, 1234), "fp32")
    dwt = OR.init_weights(g, 99)
    dw = B.DeviceWeights.from_reference(dwt, "fp32")
    prompts = [[3, 5, 7, 9], [11, 2], [40, 41, 42]]
    sids = [2 ** 40 + 3, 5, 2 ** 62 + 17]
    ref = OE.run_speculative(OE.OracleModel(OR.init_weights(TINY, 1234), 3), OE.OracleModel(dwt, 3),
                             OE.Request(prompts, 90, temperature=0.9, top_p=0.95, seed=77, sequence_ids=sids),
                             oracle.FixedLength(70))
    req = B.GenerationRequest(prompts, 90, temperature=0.9, top_p=0.95, seed=77, sequence_ids=sids)
    got = B.decode_speculative(B.CudaModel(tw, 3, capacity=256), B.CudaModel(dw, 3, capacity=256), req,
                               B.FixedDraftController(70))
    assert got.tokens == ref.tokens
    for a, b in zip(got.logprobs, ref.logprobs):
        assert np.allclose(a, b, rtol=0, atol=2e-4)
    assert got.main_forward_calls == ref.main_calls and got.draft_forward_calls == ref.draft_calls


def test_align_override_sampled_point_mass_and_providers_stay_usable(B):
    """The keyed acceptance override in sampled decoding turns each draft row
    into a point mass on its proposal (cl_draft_sample_kernel), so the verify
    never meets a zero draft probability; the caches end at the committed
    prefix and the providers stay usable (ref:engine.py:358-360)."""
    from paper_2404_15778_b200 import engine as E
    tw = B.DeviceWeights.from_reference(OR.init_weights(TINY, 1234), "fp32")
    main, draft = B.CudaModel(tw, 2), B.CudaModel(tw, 2)
    eng = E.CudaEngine(main, draft)
    req = B.GenerationRequest([[1, 2, 3], [4, 5]], 8, temperature=0.5)
    res = eng.run(req, B.FixedDraftController(3), speculative=True, align=0.5,
                  align_tokens=np.zeros((2, 8), np.int32))[0]
    assert all(len(t) == 8 for t in res.tokens)
    assert all(0 <= t < TINY.vocab_size for seq in res.tokens for t in seq)
    assert main.lengths() == [3 + 8 - 1, 2 + 8 - 1]
    for m in (main, draft):
        for s_ in range(2):
            m.rollback(s_, 0)
    res = B.decode_speculative(main, draft, req, B.FixedDraftController(3))
    assert all(len(t) == 8 for t in res.tokens)
