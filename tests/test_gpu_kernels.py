"""GPU parity of the standalone kernels against the oracle and the reference's
golden vectors: device RNG (bit-exact), shaping / sampling / accept
(identical decisions), ragged attention PAD / SPLIT / RAGGED."""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import ragged as OR
from oracle import rng as ORNG
from oracle import sampling as OS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2404_15778_b200 as B
    return B.CudaContext.default(0)


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


def test_device_rng_bit_exact(ctx, golden_dir):
    from paper_2404_15778_b200 import device_uniforms
    rows = _load(golden_dir, "rng.json")
    by_seed = {}
    for r in rows:
        by_seed.setdefault(r[0], []).append(r)
    for seed, rs in by_seed.items():
        u = device_uniforms(ctx, seed, [r[1] for r in rs], [r[2] for r in rs], [r[3] for r in rs])
        assert u.tolist() == [[r[4], r[5]] for r in rs]
    # 100k random keys vs the integer restatement (itself pinned to numpy)
    rng = np.random.default_rng(0)
    n = 100_000
    sid = rng.integers(0, 2**31 - 1, n)
    role = rng.integers(0, 2, n)
    ctr = rng.integers(0, 2**40, n)
    u = device_uniforms(ctx, 987654321987, sid, role, ctr)
    for i in rng.integers(0, n, 400):
        assert ORNG.keyed_uniforms(987654321987, sid[i], role[i], ctr[i], 2) == u[i].tolist()


def _f(x):
    return float("-inf") if x == "-inf" else x


def test_shape_sample_golden(ctx, golden_dir):
    from paper_2404_15778_b200 import device_shape_sample
    for c in _load(golden_dir, "sampling.json")["shape"]:
        logits = np.array([_f(x) for x in c["logits"]], dtype=np.float32)
        # the oracle on the same fp32-cast logits is the exact comparison
        want = OS.shape_probs(logits.astype(np.float64), c["t"], c["top_p"])
        tok, probs = device_shape_sample(ctx, logits, c["t"], c["top_p"], [c["u"]], want_probs=True)
        np.testing.assert_allclose(probs[0], want, rtol=1e-12, atol=1e-15)
        assert int(tok[0]) == OS.inverse_cdf(want, c["u"])


def test_shape_hand_cases(ctx):
    from paper_2404_15778_b200 import device_shape_sample
    _, p = device_shape_sample(ctx, np.array([0.0, 0.0, np.log(2.0)]), 1.0, 0.5, [0.3], True)
    np.testing.assert_allclose(p[0], [0, 0, 1], atol=1e-12)
    _, p = device_shape_sample(ctx, np.zeros(4), 1.0, 0.5, [0.3], True)
    np.testing.assert_allclose(p[0], [.5, .5, 0, 0], atol=1e-12)
    _, p = device_shape_sample(ctx, np.array([1.0, 3.0, 2.0]), 0.0, 0.9, [0.3], True)
    np.testing.assert_array_equal(p[0], [0, 1, 0])
    with pytest.raises(ValueError):
        device_shape_sample(ctx, np.full(4, -np.inf), 1.0, 0.9, [0.5])


def test_shape_sample_large_vocab_decisions(ctx):
    """V = 50272 rows (7.8B vocab): identical sampled tokens to the oracle."""
    from paper_2404_15778_b200 import device_shape_sample
    rng = np.random.default_rng(1)
    V, n = 50272, 48
    logits = (rng.standard_normal((n, V)) * 1.4).astype(np.float32)
    u = rng.random(n)
    for t, p in ((0.2, 0.95), (1.0, 1.0), (0.7, 0.9), (1.5, 0.5)):
        tok, probs = device_shape_sample(ctx, logits, t, p, u, want_probs=True)
        for i in range(n):
            want = OS.shape_probs(logits[i].astype(np.float64), t, p)
            assert int(tok[i]) == OS.inverse_cdf(want, u[i])
            # the nucleus tail may differ where numpy's sequential running sum
            # reaches top_p within rounding of the last elements (~1e-16 mass)
            np.testing.assert_allclose(probs[i], want, rtol=1e-6, atol=1e-9)


def test_accept_golden(ctx, golden_dir):
    from paper_2404_15778_b200 import device_accept
    cases = _load(golden_dir, "sampling.json")["accept"]
    for c in cases:
        ql = np.asarray(c["q_logits"], dtype=np.float32)
        pl = np.asarray(c["p_logits"], dtype=np.float32)
        q = OS.shape_probs(ql.astype(np.float64), c["t"], c["top_p"])
        p = OS.shape_probs(pl.astype(np.float64), c["t"], c["top_p"])
        ks = OS.KeyedStreams(c["seed"])
        tok = OS.inverse_cdf(p, ks.draft(c["sid"], c["ctr"])())
        ok, fix = OS.accept_or_resample(q, p, tok, ks.verify(c["sid"], c["ctr"]))
        acc, cor = device_accept(ctx, ql, pl, c["t"], c["top_p"], [tok], c["seed"], [c["sid"]],
                                 [c["ctr"]])
        assert bool(acc[0]) == ok
        if not ok:
            assert int(cor[0]) == fix


def test_accept_large_vocab_decisions(ctx):
    from paper_2404_15778_b200 import device_accept
    rng = np.random.default_rng(2)
    V, n = 50272, 64
    ql = (rng.standard_normal((n, V)) * 1.4).astype(np.float32)
    pl = (ql + rng.standard_normal((n, V)) * 0.5).astype(np.float32)
    t, tp, seed = 0.7, 0.95, 4242
    sids, ctrs = rng.integers(0, 64, n), rng.integers(0, 4000, n)
    toks = []
    for i in range(n):
        p = OS.shape_probs(pl[i].astype(np.float64), t, tp)
        toks.append(OS.inverse_cdf(p, OS.KeyedStreams(seed).draft(sids[i], ctrs[i])()))
    acc, cor = device_accept(ctx, ql, pl, t, tp, toks, seed, sids, ctrs)
    for i in range(n):
        q = OS.shape_probs(ql[i].astype(np.float64), t, tp)
        p = OS.shape_probs(pl[i].astype(np.float64), t, tp)
        ok, fix = OS.accept_or_resample(q, p, toks[i], OS.KeyedStreams(seed).verify(sids[i], ctrs[i]))
        assert bool(acc[i]) == ok and (ok or int(cor[i]) == fix)


def _workload_to_device(qs, ks, vs, dtype):
    import torch
    nb, H, dh = len(qs), qs[0].shape[0], qs[0].shape[2]
    stride = max(k.shape[1] for k in ks)
    K = np.zeros((nb, H, stride, dh))
    Vv = np.zeros_like(K)
    for i in range(nb):
        K[i, :, :ks[i].shape[1]] = ks[i]
        Vv[i, :, :vs[i].shape[1]] = vs[i]
    Q = np.concatenate([q.transpose(1, 0, 2) for q in qs], axis=0)    # [M, H, dh]
    cu = np.concatenate([[0], np.cumsum([q.shape[1] for q in qs])])
    dev = lambda a: torch.tensor(a, dtype=dtype, device="cuda")
    return dev(Q), dev(K), dev(Vv), cu


@pytest.mark.parametrize("strategy", ["pad", "split", "ragged"])
def test_attention_golden_fp32(ctx, golden_dir, strategy):
    import torch
    from paper_2404_15778_b200 import attend_device
    z = np.load(os.path.join(golden_dir, "attention.npz"))
    for c in range(6):
        offs = z[f"c{c}_off"].tolist()
        qs = [z[f"c{c}_{i}_q"] for i in range(len(offs))]
        if qs[0].shape[2] not in (16, 32, 64, 128):
            continue
        ks = [z[f"c{c}_{i}_k"] for i in range(len(offs))]
        vs = [z[f"c{c}_{i}_v"] for i in range(len(offs))]
        Q, K, Vv, cu = _workload_to_device(qs, ks, vs, torch.float32)
        out = attend_device(ctx, Q, K, Vv, cu, offs, strategy).cpu().numpy()
        for i in range(len(offs)):
            want = z[f"c{c}_{i}_pad"].transpose(1, 0, 2)
            np.testing.assert_allclose(out[cu[i]:cu[i + 1]], want, rtol=2e-5, atol=2e-5)


@pytest.mark.parametrize("dh", [128, 64])
def test_attention_strategies_bitwise_equal_bf16(ctx, dh):
    """tcgen05 stream attention (d_head 128 and 64): PAD == SPLIT == RAGGED
    bitwise, within 1e-2 of the oracle on the bf16-rounded inputs; blocks up
    to 65 rows (two NQ = 64 query tiles), histories past one 1024-key split."""
    import torch
    from paper_2404_15778_b200 import attend_device
    rng = np.random.default_rng(3 + dh)
    H = 36 if dh == 128 else 12
    q_lens = [1, 8, 17, 3, 33, 5, 9, 2] + ([65, 1] if dh == 64 else [])
    kv = [int(rng.integers(q, 1500)) for q in q_lens]
    qs = [rng.standard_normal((H, q, dh)) for q in q_lens]
    ks = [rng.standard_normal((H, n, dh)) for n in kv]
    vs = [rng.standard_normal((H, n, dh)) for n in kv]
    offs = [n - q for n, q in zip(kv, q_lens)]
    Q, K, Vv, cu = _workload_to_device(qs, ks, vs, torch.bfloat16)
    outs = [attend_device(ctx, Q, K, Vv, cu, offs, s) for s in ("pad", "split", "ragged")]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    # vs the oracle on the bf16-rounded inputs
    r = lambda a: torch.tensor(a).bfloat16().double().numpy()
    want = OR.attend_split([r(q) for q in qs], [r(k) for k in ks], [r(v) for v in vs], offs)
    got = outs[2].double().cpu().numpy()
    for i in range(len(q_lens)):
        w = want[i].transpose(1, 0, 2)
        err = np.abs(got[cu[i]:cu[i + 1]] - w).max() / np.abs(w).max()
        assert err < 1e-2, err


@pytest.mark.parametrize("q_max", [16, 32, 65])
def test_attention_tile_classes_long_histories(ctx, q_max):
    """Each query-tile build (NQ = 16 with its long-history 3-stage ring,
    NQ = 32 and NQ = 64 with K streamed ahead of V, two NQ = 64 tiles per
    block in split-major item order) over histories of up to three 1024-key
    splits: PAD == SPLIT == RAGGED bitwise and within 1e-2 of the oracle."""
    import torch
    from paper_2404_15778_b200 import attend_device
    rng = np.random.default_rng(q_max)
    H, dh = 8, 128
    q_lens = [q_max, 1, max(1, q_max // 2), 3, q_max]
    kv = [int(rng.integers(max(q, 1100), 3000)) for q in q_lens]
    qs = [rng.standard_normal((H, q, dh)) for q in q_lens]
    ks = [rng.standard_normal((H, n, dh)) for n in kv]
    vs = [rng.standard_normal((H, n, dh)) for n in kv]
    offs = [n - q for n, q in zip(kv, q_lens)]
    Q, K, Vv, cu = _workload_to_device(qs, ks, vs, torch.bfloat16)
    outs = [attend_device(ctx, Q, K, Vv, cu, offs, s) for s in ("pad", "split", "ragged")]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    r = lambda a: torch.tensor(a).bfloat16().double().numpy()
    want = OR.attend_split([r(q) for q in qs], [r(k) for k in ks], [r(v) for v in vs], offs)
    got = outs[2].double().cpu().numpy()
    for i in range(len(q_lens)):
        w = want[i].transpose(1, 0, 2)
        err = np.abs(got[cu[i]:cu[i + 1]] - w).max() / np.abs(w).max()
        assert err < 1e-2, err


def test_attention_decode_two_ctas_per_sm(ctx):
    """Single-row decode blocks with more (sequence, head) items than SMs and
    histories <= 512 run the one-stage ring at two CTAs per SM (RAGGED / PAD:
    8 x 36 = 288 items); SPLIT launches one sequence (36 items) at a time on
    the two-stage build — bitwise equal, and within 1e-2 of the oracle."""
    import torch
    from paper_2404_15778_b200 import attend_device
    rng = np.random.default_rng(11)
    H, dh = 36, 128
    q_lens = [1] * 8
    kv = [int(rng.integers(2, 512)) for _ in q_lens]
    kv[3] = 1   # a history of the new row alone
    qs = [rng.standard_normal((H, 1, dh)) for _ in q_lens]
    ks = [rng.standard_normal((H, n, dh)) for n in kv]
    vs = [rng.standard_normal((H, n, dh)) for n in kv]
    offs = [n - 1 for n in kv]
    Q, K, Vv, cu = _workload_to_device(qs, ks, vs, torch.bfloat16)
    outs = [attend_device(ctx, Q, K, Vv, cu, offs, s) for s in ("pad", "split", "ragged")]
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[1], outs[2])
    r = lambda a: torch.tensor(a).bfloat16().double().numpy()
    want = OR.attend_split([r(q) for q in qs], [r(k) for k in ks], [r(v) for v in vs], offs)
    got = outs[2].double().cpu().numpy()
    for i in range(len(q_lens)):
        w = want[i].transpose(1, 0, 2)
        err = np.abs(got[cu[i]:cu[i + 1]] - w).max() / np.abs(w).max()
        assert err < 1e-2, err
