"""The device-resident decode loop (north_star (4); ref:engine.py:237-362,
draft_control.py:49-69) against the per-step host loop, through the C ABI.

BASS_LOOP_DEVICE books every step on the GPU (committed tokens, EOS /
length, cache-length rollback, Algorithm 1, the step trace) and drives the
steps after the prompt step from one CUDA graph (WHILE over a SWITCH on the
draft length); BASS_LOOP_HOST plans each step on the host and reads it back.
Both must give bit-identical results — tokens, logprobs, finish reasons and
steps, the whole step trace, forward-call counters, the final Algorithm-1
state and the providers' cache lengths — with one host synchronisation per
generation on the device path.
"""

import numpy as np
import pytest

from oracle import ragged as OR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2404_15778_b200 as B
    return B


def _weights(B, g, seed):
    w = OR.init_weights(g, seed)
    return B.DeviceWeights.from_reference(w, "bf16")


MAIN = OR.Geometry(2, 4, 512, 128, 2048, 512)
DRAFT = OR.Geometry(1, 4, 256, 64, 2048, 512)


@pytest.fixture(scope="module")
def models(B):
    return _weights(B, MAIN, 3), _weights(B, DRAFT, 4)


def _run(B, wm, wd, req, ctl, mode, strategy="ragged", align=-1.0, align_tokens=None, cap=None):
    b = req.batch_size
    main = B.CudaModel(wm, b, strategy, capacity=cap)
    draft = B.CudaModel(wd, b, strategy, capacity=cap)
    eng = B.CudaEngine(main, draft)
    eng.set_strategy(strategy)
    eng.set_loop(mode)
    res, arr, raw = eng.run(req, ctl, speculative=True, align=align, align_seed=99, align_tokens=align_tokens)
    info = eng.loop_info()
    return res, raw, info, main.lengths(), draft.lengths(), eng


def _same(a, b):
    ra, rawa, ia, lma, lda, _ = a
    rb, rawb, ib, lmb, ldb, _ = b
    assert ra.tokens == rb.tokens
    assert ra.logprobs == rb.logprobs                       # bitwise
    assert ra.finish_reason == rb.finish_reason
    assert ra.completion_step == rb.completion_step
    assert ra.main_forward_calls == rb.main_forward_calls
    assert ra.draft_forward_calls == rb.draft_forward_calls
    assert len(ra.steps) == len(rb.steps)
    for x, y in zip(ra.steps, rb.steps):
        assert x.draft_length == y.draft_length
        assert list(x.accepted) == list(y.accepted)
        assert [list(e) for e in x.emitted] == [list(e) for e in y.emitted]
        assert list(x.kv_lengths) == list(y.kv_lengths)
        assert tuple(x.slots) == tuple(y.slots) and tuple(x.finished) == tuple(y.finished)
    assert (rawa.final_l_draft, rawa.final_s) == (rawb.final_l_draft, rawb.final_s)
    assert lma == lmb and lda == ldb


def _prompts(n, V, seed, lo=5, hi=40):
    rs = np.random.default_rng(seed)
    return [rs.integers(0, V, int(rs.integers(lo, hi))).tolist() for _ in range(n)]


@pytest.mark.parametrize("strategy", ["ragged", "split", "pad"])
def test_greedy_harness_device_equals_host(B, models, strategy):
    wm, wd = models
    prompts = _prompts(5, 2048, 1)
    req = B.GenerationRequest(prompts, 40, temperature=0.0, sequence_ids=[3, 1, 4, 1_000_000_007, 5])
    # main model's greedy trajectory -> keyed acceptance override (bench harness)
    eng = B.CudaEngine(B.CudaModel(wm, 5), B.CudaModel(wd, 5))
    traj = eng.run(req, None, speculative=False)[1]["tokens"]
    ctl = lambda: B.AdaptiveDraftController()   # noqa: E731
    host = _run(B, wm, wd, req, ctl(), "host", strategy, 0.7, traj)
    dev = _run(B, wm, wd, req, ctl(), "device", strategy, 0.7, traj)
    _same(host, dev)
    assert dev[2]["mode"] == "device" and dev[2]["syncs"] == 1
    assert host[2]["syncs"] == len(host[0].steps)
    assert host[0].tokens == [t[:40] for t in traj.tolist()]   # greedy spec == regular
    assert len({s.draft_length for s in dev[0].steps}) > 2          # Algorithm 1 moved l


def test_greedy_self_draft_grows_to_limit_and_eos(B, models):
    wm, _ = models
    prompts = _prompts(3, 2048, 2)
    eng = B.CudaEngine(B.CudaModel(wm, 3), B.CudaModel(wm, 3))
    free = eng.run(B.GenerationRequest(prompts, 48, temperature=0.0), None, speculative=False)[0]
    eos = free.tokens[1][20]   # a token the main model emits: some sequences stop early
    req = B.GenerationRequest(prompts, 48, temperature=0.0, eos_token=eos)
    p = B.DraftLengthParams(l0=3, incre=3, mod=4, limit=12)
    host = _run(B, wm, wm, req, B.AdaptiveDraftController(p), "host")
    dev = _run(B, wm, wm, req, B.AdaptiveDraftController(p), "device")
    _same(host, dev)
    assert "eos" in dev[0].finish_reason
    assert max(s.draft_length for s in dev[0].steps) == 12


@pytest.mark.parametrize("fixed", [None, 4])
def test_sampled_device_equals_host(B, models, fixed):
    wm, wd = models
    prompts = _prompts(4, 2048, 3)
    req = B.GenerationRequest(prompts, 32, temperature=0.7, top_p=0.9, seed=1234)
    mk = (lambda: B.FixedDraftController(fixed)) if fixed else (lambda: B.AdaptiveDraftController())
    # a draft with the main weights: high acceptance (bonus rows, resamples)
    host = _run(B, wm, wm, req, mk(), "host")
    dev = _run(B, wm, wm, req, mk(), "device")
    _same(host, dev)
    assert any(a > 0 for s in dev[0].steps for a in s.accepted)
    # an unrelated draft: rejections and corrections
    host = _run(B, wm, wd, req, mk(), "host")
    dev = _run(B, wm, wd, req, mk(), "device")
    _same(host, dev)


def test_graph_reused_across_generations_and_rebuilt_on_change(B, models):
    wm, wd = models
    prompts = _prompts(4, 2048, 5)
    req = B.GenerationRequest(prompts, 24, temperature=0.0)
    main, draft = B.CudaModel(wm, 4), B.CudaModel(wd, 4)
    eng = B.CudaEngine(main, draft)
    outs = []
    for _ in range(3):
        for m in (main, draft):
            for s in range(4):
                m.rollback(s, 0)
        outs.append(eng.run(req, B.AdaptiveDraftController(), speculative=True)[0].tokens)
    info = eng.loop_info()
    assert outs[0] == outs[1] == outs[2]
    assert info["syncs"] == 1 and info["graph_builds"] >= 1
    builds = info["graph_builds"]
    for m in (main, draft):
        for s in range(4):
            m.rollback(s, 0)
    eng.run(B.GenerationRequest(prompts, 24, temperature=0.0, eos_token=7), B.AdaptiveDraftController(),
            speculative=True)
    assert eng.loop_info()["graph_builds"] == builds + 1   # eos is baked into the finalize kernel


@pytest.mark.parametrize("temperature,strategy", [(0.0, "ragged"), (0.7, "ragged"), (0.7, "split"), (0.0, "pad")])
def test_int8_device_loop_equals_host(B, temperature, strategy):
    cfg = B.ModelConfig(2, 2, 256, 128, 1024, 256)
    wm = B.DeviceWeights.init_model(cfg, 6, "int8")
    prompts = _prompts(3, 1024, 6)
    req = B.GenerationRequest(prompts, 24, temperature=temperature, top_p=0.9, seed=5)
    host = _run(B, wm, wm, req, B.AdaptiveDraftController(), "host", strategy)
    dev = _run(B, wm, wm, req, B.AdaptiveDraftController(), "device", strategy)
    _same(host, dev)


def test_sampled_point_mass_harness_device_equals_host(B, models):
    """The sampled acceptance harness (point-mass draft rows on keyed
    override tokens from an independent-seed trajectory): accepted proposals,
    identical on both loop drivers, and the harness tokens really are what
    the draft rows propose."""
    wm, wd = models
    prompts = _prompts(4, 2048, 8)
    req = B.GenerationRequest(prompts, 32, temperature=0.7, top_p=0.9, seed=77)
    eng = B.CudaEngine(B.CudaModel(wm, 4), B.CudaModel(wd, 4))
    traj = eng.run(B.GenerationRequest(prompts, 32, temperature=0.7, top_p=0.9, seed=78), None,
                   speculative=False)[1]["tokens"]
    host = _run(B, wm, wd, req, B.AdaptiveDraftController(), "host", "ragged", 0.9, traj)
    dev = _run(B, wm, wd, req, B.AdaptiveDraftController(), "device", "ragged", 0.9, traj)
    _same(host, dev)
    acc = [a for s in dev[0].steps for a in s.accepted]
    assert sum(acc) > 0   # the random-init draft alone is never accepted


@pytest.mark.parametrize("b,new", [(1, 20), (40, 12), (3, 1), (3, 2)])
def test_device_loop_edge_batches_and_lengths(B, models, b, new):
    """b = 1 and b = 40 (several warps in the plan / book kernels), a
    generation that ends in the prompt step (the graph runs zero iterations)
    and one that ends right after it."""
    wm, wd = models
    prompts = _prompts(b, 2048, 11 + b)
    req = B.GenerationRequest(prompts, new, temperature=0.0)
    host = _run(B, wm, wd, req, B.AdaptiveDraftController(), "host")
    dev = _run(B, wm, wd, req, B.AdaptiveDraftController(), "device")
    _same(host, dev)
    assert all(len(t) == new for t in dev[0].tokens)


def test_fresh_weights_first_use_in_the_device_loop(B):
    """Weights whose lazily computed state (the folded-LayerNorm constants)
    has never been built: the device loop prepares it before capturing its
    graph (a capture would otherwise record the preparation instead of running
    it).  Each run gets its own fresh upload."""
    def fresh(seed):
        return B.DeviceWeights.from_reference(OR.init_weights(OR.Geometry(2, 4, 512, 128, 1000, 256), seed), "bf16")
    prompts = _prompts(6, 1000, 21)
    req = B.GenerationRequest(prompts, 16, temperature=0.0)
    host = _run(B, fresh(41), fresh(42), req, B.AdaptiveDraftController(), "host")
    dev = _run(B, fresh(41), fresh(42), req, B.AdaptiveDraftController(), "device")
    _same(host, dev)
    reg = B.decode_regular(B.CudaModel(fresh(41), 6), req)
    assert dev[0].tokens == reg.tokens


def test_sampled_with_eos_device_equals_host(B, models):
    """Sampled decoding that stops on an EOS token inside accepted blocks,
    corrections and bonus tokens (ref:engine.py:103-117 finalize rules)."""
    wm, _ = models
    prompts = _prompts(5, 2048, 31)
    base = B.GenerationRequest(prompts, 40, temperature=0.9, top_p=0.95, seed=3)
    free = _run(B, wm, wm, base, B.AdaptiveDraftController(), "host")[0]
    eos = free.tokens[0][5]
    req = B.GenerationRequest(prompts, 40, temperature=0.9, top_p=0.95, seed=3, eos_token=eos)
    host = _run(B, wm, wm, req, B.AdaptiveDraftController(), "host")
    dev = _run(B, wm, wm, req, B.AdaptiveDraftController(), "device")
    _same(host, dev)
    assert "eos" in dev[0].finish_reason
