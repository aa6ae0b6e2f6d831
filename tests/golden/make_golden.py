"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed, small) go next to this script.  They pin the oracle
(`oracle/`) and, through it, the CUDA path.  Nothing at test/bench time
reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from batchspec import attention as A          # noqa: E402
from batchspec import draft_control as DC     # noqa: E402
from batchspec import engine as E             # noqa: E402
from batchspec import model as M              # noqa: E402
from batchspec import sampling as S           # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def dump(name, obj):
    with open(os.path.join(OUT, name), "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))


def rng_vectors():
    rs = np.random.default_rng(0)
    out = []
    for seed in (0, 1, 1234, 2**40 + 7, 2**64 - 1):
        stream = S.RngStream(seed)
        for _ in range(40):
            sid = int(rs.integers(0, 100))
            role = S.ROLE_DRAFT if rs.integers(0, 2) == 0 else S.ROLE_VERIFY
            ctr = int(rs.integers(0, 5000))
            g = stream.generator(sid, role, ctr)
            out.append([seed, sid, S._ROLE_CODES[role], ctr, g.random(), g.random()])
    dump("rng.json", out)


def control_vectors():
    rs = np.random.default_rng(42)
    traces = []
    for params in (DC.DraftLengthParams(), DC.DraftLengthParams(l0=3, incre=1, mod=4, limit=9)):
        st = DC.init_state(params)
        tr = []
        for _ in range(300):
            b = int(rs.integers(1, 9))
            accs = [int(rs.integers(0, st.l_draft + 1)) for _ in range(b)]
            if rs.random() < 0.3:
                accs[0] = st.l_draft
            st = DC.update(st, accs)
            tr.append([accs, st.l_draft, st.s])
        traces.append({"params": [params.l0, params.incre, params.mod, params.limit],
                       "trace": tr})
    dump("control.json", traces)


def sampling_vectors():
    rs = np.random.default_rng(7)
    shape_cases, accept_cases = [], []
    for i in range(120):
        v = int(rs.choice([3, 8, 16, 50, 97]))
        logits = (rs.standard_normal(v) * rs.choice([0.5, 2.0, 8.0])).tolist()
        if i % 10 == 0:
            logits[int(rs.integers(0, v))] = float("-inf")
        t = float(rs.choice([0.0, 0.2, 0.7, 1.0, 1.5]))
        p = float(rs.choice([1.0, 0.95, 0.9, 0.5, 0.1]))
        d = S.to_distribution(np.asarray(logits), t, p)
        u = float(rs.random())
        shape_cases.append({"logits": [x if np.isfinite(x) else "-inf" for x in logits],
                            "t": t, "top_p": p, "probs": d.probs.tolist(),
                            "u": u, "tok": S._inverse_cdf(d.probs, u)})
    for i in range(120):
        v = int(rs.choice([4, 16, 64]))
        t = float(rs.choice([0.5, 1.0]))
        p = float(rs.choice([1.0, 0.9]))
        ql = rs.standard_normal(v) * 2
        pl = ql + rs.standard_normal(v) * float(rs.choice([0.1, 1.0, 3.0]))
        q = S.to_distribution(ql, t, p)
        pd = S.to_distribution(pl, t, p)
        stream = S.RngStream(int(rs.integers(0, 1000)))
        sid, ctr = int(rs.integers(0, 8)), int(rs.integers(0, 500))
        tok = S.sample(pd, stream.generator(sid, S.ROLE_DRAFT, ctr))
        dec = S.speculative_accept(q, pd, tok, stream.generator(sid, S.ROLE_VERIFY, ctr))
        accept_cases.append({"q_logits": ql.tolist(), "p_logits": pl.tolist(), "t": t,
                             "top_p": p, "seed": stream.seed, "sid": sid, "ctr": ctr,
                             "tok": tok, "accepted": dec.accepted,
                             "corrected": dec.corrected_token})
    dump("sampling.json", {"shape": shape_cases, "accept": accept_cases})


def attention_vectors():
    rs = np.random.default_rng(11)
    arrays = {}
    for c in range(6):
        b = int(rs.integers(1, 6))
        nh, dh = int(rs.choice([1, 2, 4])), int(rs.choice([8, 16, 32]))
        q_lens = rs.integers(1, 9, b).tolist()
        kv_lens = [int(q + rs.integers(0, 40)) for q in q_lens]
        w = A.AttentionWorkload(
            queries=[rs.standard_normal((nh, q, dh)) for q in q_lens],
            keys=[rs.standard_normal((nh, n, dh)) for n in kv_lens],
            values=[rs.standard_normal((nh, n, dh)) for n in kv_lens],
            offsets=[n - q for n, q in zip(kv_lens, q_lens)])
        pad = A.attend(w, A.AttentionStrategy.PAD)
        spl = A.attend(w, A.AttentionStrategy.SPLIT)
        for i in range(b):
            for nm, arr in (("q", w.queries[i]), ("k", w.keys[i]), ("v", w.values[i]),
                            ("pad", pad[i]), ("split", spl[i])):
                arrays[f"c{c}_{i}_{nm}"] = arr
        arrays[f"c{c}_off"] = np.asarray(w.offsets)
    np.savez_compressed(os.path.join(OUT, "attention.npz"), **arrays)


TINY = dict(n_layer=2, n_head=4, d_model=64, vocab_size=96, max_seq_len=256)


def forward_vectors():
    cfg = M.desk_config(**TINY)
    w = M.init_model(cfg, 5)
    rs = np.random.default_rng(0)
    prompts = [rs.integers(0, 96, n).tolist() for n in (4, 1, 6, 3)]
    blocks = [rs.integers(0, 96, n).tolist() for n in (3, 7, 5, 1)]
    out = {"prompts": prompts, "blocks": blocks}
    arrays = {}
    for strat in (A.AttentionStrategy.PAD, A.AttentionStrategy.SPLIT):
        cache = M.new_cache(cfg, 4)
        pre = [M.prefill(w, cache, s, p, strat) for s, p in enumerate(prompts)]
        logits = M.forward_block(w, cache, [0, 1, 2, 3], blocks, strat)
        for s in range(4):
            arrays[f"{strat.value}_prefill_{s}"] = pre[s]
            arrays[f"{strat.value}_block_{s}"] = logits[s]
    init = {"tok_emb": w.token_emb, "pos_emb": w.pos_emb, "head": w.head,
            "wq0": w.blocks[0].wq, "w_fc1": w.blocks[1].w_fc,
            "w_proj1": w.blocks[1].w_proj}
    for k, v in init.items():
        arrays[f"init_{k}_head"] = v.reshape(-1)[:64]
        arrays[f"init_{k}_sum"] = np.asarray([v.sum(), np.abs(v).sum()])
    np.savez_compressed(os.path.join(OUT, "forward.npz"), **arrays)
    dump("forward.json", out)


def _result(res):
    return {"tokens": res.tokens, "logprobs": res.logprobs,
            "finish_reason": res.finish_reason, "completion_step": res.completion_step,
            "main_calls": res.main_forward_calls, "draft_calls": res.draft_forward_calls,
            "steps": [{"draft_length": s.draft_length, "slots": list(s.slots),
                       "accepted": list(s.accepted),
                       "emitted": [list(e) for e in s.emitted],
                       "finished": list(s.finished), "kv_lengths": list(s.kv_lengths)}
                      for s in res.steps]}


def decode_vectors():
    runs = {}
    # C1: main 2L d128 seed 0; independent draft 1L seed 1.
    c1 = M.ModelConfig(n_layer=2, n_head=4, d_model=128, d_head=32,
                       vocab_size=512, max_seq_len=1024)
    c1d = M.ModelConfig(n_layer=1, n_head=4, d_model=128, d_head=32,
                        vocab_size=512, max_seq_len=1024)
    wm, wd = M.init_model(c1, 0), M.init_model(c1d, 1)
    rng = np.random.default_rng(0 + 1_000_003)
    prompts = [rng.integers(0, 512, 16).tolist() for _ in range(4)]
    for strat in (A.AttentionStrategy.PAD, A.AttentionStrategy.SPLIT):
        req = E.GenerationRequest(prompts=prompts, max_new_tokens=64, temperature=0.0,
                                  strategy=strat, seed=0)
        runs[f"c1_regular_{strat.value}"] = _result(E.decode_regular(M.MainModel(wm, 4, strat), req))
        runs[f"c1_spec_{strat.value}"] = _result(E.decode_speculative(
            M.MainModel(wm, 4, strat), M.MainModel(wd, 4, strat), req,
            DC.FixedDraftController(4)))
    req = E.GenerationRequest(prompts=prompts, max_new_tokens=64, temperature=0.0, seed=0)
    runs["c1_spec_synth08"] = _result(E.decode_speculative(
        M.MainModel(wm, 4), M.SyntheticAlignedDraft(wm, 0.8, 17, 4), req,
        DC.AdaptiveDraftController()))
    # tiny sampled (pins test_bench golden tokens, ref tests/test_bench.py:142-154)
    tcfg = M.desk_config(**TINY)
    tw = M.init_model(tcfg, 1234)
    trng = np.random.default_rng(1234 + 1_000_003)
    tprompts = [trng.integers(0, 96, 5).tolist() for _ in range(2)]
    treq = E.GenerationRequest(prompts=tprompts, max_new_tokens=12, temperature=0.7,
                               top_p=0.9, seed=1234)
    runs["tiny_regular_sampled"] = _result(E.decode_regular(M.MainModel(tw, 2), treq))
    treq2 = E.GenerationRequest(prompts=tprompts, max_new_tokens=40, temperature=0.7,
                                top_p=0.9, seed=1234)
    runs["tiny_spec_sampled"] = _result(E.decode_speculative(
        M.MainModel(tw, 2), M.SyntheticAlignedDraft(tw, 0.8, 1234 + 17, 2), treq2,
        DC.AdaptiveDraftController()))
    # sampled speculative with an independent (real-model) draft, 3 slots, EOS
    dcfg = M.desk_config(n_layer=1, n_head=4, d_model=64, vocab_size=96, max_seq_len=256)
    dw = M.init_model(dcfg, 99)
    sp = [[3, 14, 15, 9], [2, 71, 82], [81, 8, 28, 45, 90]]
    sreq = E.GenerationRequest(prompts=sp, max_new_tokens=30, temperature=1.0, top_p=0.95,
                               seed=8, eos_token=7, sequence_ids=[5, 0, 11])
    runs["tiny_spec_sampled_realdraft"] = _result(E.decode_speculative(
        M.MainModel(tw, 3), M.MainModel(dw, 3), sreq, DC.AdaptiveDraftController(
            DC.DraftLengthParams(l0=3, incre=2, mod=10, limit=8))))
    runs["tiny_regular_sampled_eos"] = _result(E.decode_regular(M.MainModel(tw, 3), sreq))
    dump("decode.json", {"c1_prompts": prompts, "tiny_prompts": tprompts,
                         "eos_prompts": sp, "runs": runs})


if __name__ == "__main__":
    rng_vectors()
    control_vectors()
    sampling_vectors()
    attention_vectors()
    forward_vectors()
    decode_vectors()
    print("golden vectors written to", OUT)
