"""Pin the CPU oracle against golden vectors produced by the reference itself.

The vectors come from tests/golden/make_golden.py (which imports the
reference package read-only).  If any of these fail, the oracle is not a
trustworthy checker for the CUDA path.
"""

import json
import os

import numpy as np
import pytest

import oracle
from oracle import engine as OE
from oracle import ragged as OR
from oracle import rng as ORNG
from oracle import sampling as OS
from oracle.control import AlgParams, alg1_update



def load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as fh:
        return json.load(fh)


def test_rng_restatement_matches_reference_stream(golden_dir):
    for seed, sid, role, ctr, u0, u1 in load(golden_dir, "rng.json"):
        assert ORNG.keyed_uniforms(seed, sid, role, ctr, 2) == [u0, u1]
        g = OS.KeyedStreams(seed).gen(sid, role, ctr)
        assert [g(), g()] == [u0, u1]


def test_rng_restatement_matches_numpy_broadly():
    rs = np.random.default_rng(3)
    for _ in range(300):
        key = (int(rs.integers(0, 2**63)) * int(rs.integers(1, 3)),
               int(rs.integers(0, 2**33)), int(rs.integers(0, 2)),
               int(rs.integers(0, 2**20)))
        g = np.random.default_rng(np.random.SeedSequence(entropy=key))
        assert ORNG.pcg64_uniforms(key, 3) == [g.random() for _ in range(3)]


def test_algorithm1_traces(golden_dir):
    for case in load(golden_dir, "control.json"):
        p = AlgParams(*case["params"])
        l, s = p.l0, 0
        for accs, l_ref, s_ref in case["trace"]:
            l, s = alg1_update(l, s, accs, p)
            assert (l, s) == (l_ref, s_ref)


def test_algorithm1_paper_trace():
    # ref tests/test_draft_control.py:35-55 hand cases
    p = AlgParams()
    assert alg1_update(7, 0, (7, 3), p) == (9, 0)
    assert alg1_update(9, 0, (3, 1), p) == (8, 1)
    assert alg1_update(8, 1, (2, 2), p) == (6, 1)
    assert alg1_update(1, 1, (0,), p) == (1, 1)
    assert alg1_update(31, 0, (31,), p) == (32, 0)
    with pytest.raises(ValueError):
        alg1_update(6, 1, (9, 2), p)


def _f(x):
    return float("-inf") if x == "-inf" else x


def test_shaping_and_inverse_cdf(golden_dir):
    cases = load(golden_dir, "sampling.json")["shape"]
    for c in cases:
        probs = OS.shape_probs(np.array([_f(x) for x in c["logits"]]), c["t"], c["top_p"])
        np.testing.assert_allclose(probs, c["probs"], rtol=0, atol=1e-15)
        assert OS.inverse_cdf(np.asarray(c["probs"]), c["u"]) == c["tok"]


def test_shaping_hand_cases():
    # ref tests/test_sampling.py:21-50
    np.testing.assert_array_equal(OS.shape_probs(np.array([1.0, 3.0, 2.0]), 0.0, 0.9),
                                  [0, 1, 0])
    np.testing.assert_allclose(OS.shape_probs(np.array([0.0, 0.0, np.log(2.0)]), 1.0, 0.5),
                               [0, 0, 1], atol=1e-12)
    np.testing.assert_allclose(OS.shape_probs(np.zeros(4), 1.0, 0.5), [.5, .5, 0, 0],
                               atol=1e-12)
    with pytest.raises(ValueError):
        OS.shape_probs(np.full(4, -np.inf), 1.0, 0.9)


def test_accept_decisions(golden_dir):
    for c in load(golden_dir, "sampling.json")["accept"]:
        q = OS.shape_probs(np.asarray(c["q_logits"]), c["t"], c["top_p"])
        p = OS.shape_probs(np.asarray(c["p_logits"]), c["t"], c["top_p"])
        ks = OS.KeyedStreams(c["seed"])
        tok = OS.inverse_cdf(p, ks.draft(c["sid"], c["ctr"])())
        assert tok == c["tok"]
        ok, fix = OS.accept_or_resample(q, p, tok, ks.verify(c["sid"], c["ctr"]))
        assert ok == c["accepted"] and fix == c["corrected"]


def test_attention_pad_split(golden_dir):
    z = np.load(os.path.join(golden_dir, "attention.npz"))
    for c in range(6):
        offs = z[f"c{c}_off"].tolist()
        qs = [z[f"c{c}_{i}_q"] for i in range(len(offs))]
        ks = [z[f"c{c}_{i}_k"] for i in range(len(offs))]
        vs = [z[f"c{c}_{i}_v"] for i in range(len(offs))]
        for fn, tag in ((OR.attend_pad, "pad"), (OR.attend_split, "split")):
            for i, o in enumerate(fn(qs, ks, vs, offs)):
                np.testing.assert_allclose(o, z[f"c{c}_{i}_{tag}"], rtol=0, atol=1e-12)


TINY = OR.Geometry(2, 4, 64, 16, 96, 256)


def test_init_draws_match_reference(golden_dir):
    z = np.load(os.path.join(golden_dir, "forward.npz"))
    w = OR.init_weights(TINY, 5)
    pick = {"tok_emb": w["tok_emb"], "pos_emb": w["pos_emb"], "head": w["head"],
            "wq0": w["layers"][0]["wq"], "w_fc1": w["layers"][1]["w_fc"],
            "w_proj1": w["layers"][1]["w_proj"]}
    for k, v in pick.items():
        np.testing.assert_array_equal(v.reshape(-1)[:64], z[f"init_{k}_head"])
        np.testing.assert_allclose([v.sum(), np.abs(v).sum()], z[f"init_{k}_sum"],
                                   rtol=1e-12)


def test_forward_ragged_matches_reference(golden_dir):
    z = np.load(os.path.join(golden_dir, "forward.npz"))
    meta = load(golden_dir, "forward.json")
    w = OR.init_weights(TINY, 5)
    for strat in ("pad", "split"):
        cache = OR.RaggedCache(2, 4, 4, 16)
        for s, p in enumerate(meta["prompts"]):
            pre = OR.forward_ragged(w, cache, [s], [p], strat)[0][-1]
            np.testing.assert_allclose(pre, z[f"{strat}_prefill_{s}"], rtol=0, atol=1e-12)
        outs = OR.forward_ragged(w, cache, [0, 1, 2, 3], meta["blocks"], strat)
        for s in range(4):
            np.testing.assert_allclose(outs[s], z[f"{strat}_block_{s}"], rtol=0, atol=1e-12)
        assert [cache.length(s) for s in range(4)] == [7, 8, 11, 4]


def _check_run(res, ref):
    assert res.tokens == ref["tokens"]
    assert res.finish_reason == ref["finish_reason"]
    assert res.completion_step == ref["completion_step"]
    assert res.main_calls == ref["main_calls"] and res.draft_calls == ref["draft_calls"]
    for a, b in zip(res.logprobs, ref["logprobs"]):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-9)
    assert len(res.steps) == len(ref["steps"])
    for s, r in zip(res.steps, ref["steps"]):
        assert s["draft_length"] == r["draft_length"]
        assert list(s["accepted"]) == r["accepted"]
        assert [list(e) for e in s["emitted"]] == r["emitted"]
        if "kv_lengths" in s:
            assert list(s["kv_lengths"]) == r["kv_lengths"]


C1_MAIN = OR.Geometry(2, 4, 128, 32, 512, 1024)
C1_DRAFT = OR.Geometry(1, 4, 128, 32, 512, 1024)


@pytest.mark.parametrize("strat", ["pad", "split"])
def test_c1_greedy_runs(golden_dir, strat):
    d = load(golden_dir, "decode.json")
    wm, wd = OR.init_weights(C1_MAIN, 0), OR.init_weights(C1_DRAFT, 1)
    req = OE.Request(d["c1_prompts"], 64, temperature=0.0, strategy=strat)
    _check_run(OE.run_regular(OE.OracleModel(wm, 4, strat), req),
               d["runs"][f"c1_regular_{strat}"])
    _check_run(OE.run_speculative(OE.OracleModel(wm, 4, strat), OE.OracleModel(wd, 4, strat),
                                  req, oracle.FixedLength(4)),
               d["runs"][f"c1_spec_{strat}"])


def test_c1_synthetic_aligned_draft(golden_dir):
    d = load(golden_dir, "decode.json")
    wm = OR.init_weights(C1_MAIN, 0)
    req = OE.Request(d["c1_prompts"], 64, temperature=0.0)
    _check_run(OE.run_speculative(OE.OracleModel(wm, 4), OE.OracleAlignedDraft(wm, 0.8, 17, 4),
                                  req, oracle.AdaptiveLength()),
               d["runs"]["c1_spec_synth08"])


def test_tiny_sampled_runs(golden_dir):
    d = load(golden_dir, "decode.json")
    tw = OR.init_weights(OR.Geometry(2, 4, 64, 16, 96, 256), 1234)
    req = OE.Request(d["tiny_prompts"], 12, temperature=0.7, top_p=0.9, seed=1234)
    res = OE.run_regular(OE.OracleModel(tw, 2), req)
    _check_run(res, d["runs"]["tiny_regular_sampled"])
    # the reference's own pinned golden (ref tests/test_bench.py:142-154)
    assert res.tokens == [[38, 32, 87, 74, 67, 27, 25, 29, 14, 19, 1, 62],
                          [76, 95, 58, 30, 94, 4, 73, 41, 86, 32, 41, 19]]
    req2 = OE.Request(d["tiny_prompts"], 40, temperature=0.7, top_p=0.9, seed=1234)
    _check_run(OE.run_speculative(OE.OracleModel(tw, 2),
                                  OE.OracleAlignedDraft(tw, 0.8, 1234 + 17, 2), req2,
                                  oracle.AdaptiveLength()),
               d["runs"]["tiny_spec_sampled"])


def test_tiny_sampled_realdraft_and_eos(golden_dir):
    d = load(golden_dir, "decode.json")
    tw = OR.init_weights(OR.Geometry(2, 4, 64, 16, 96, 256), 1234)
    dw = OR.init_weights(OR.Geometry(1, 4, 64, 16, 96, 256), 99)
    req = OE.Request(d["eos_prompts"], 30, temperature=1.0, top_p=0.95, seed=8,
                     eos_token=7, sequence_ids=[5, 0, 11])
    _check_run(OE.run_speculative(OE.OracleModel(tw, 3), OE.OracleModel(dw, 3), req,
                                  oracle.AdaptiveLength(AlgParams(3, 2, 10, 8))),
               d["runs"]["tiny_spec_sampled_realdraft"])
    _check_run(OE.run_regular(OE.OracleModel(tw, 3), req),
               d["runs"]["tiny_regular_sampled_eos"])
