"""Regular and batched speculative decoding loops, restated.

ref:engine.py:99-385.  Providers implement the reference's LogitsProvider
protocol (ref:model.py:263-285): ``vocab_size``, ``max_seq_len``,
``prefill``, ``forward``, ``rollback``, ``length``.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np
from scipy.special import logsumexp

from .ragged import RaggedCache, forward_ragged
from .sampling import KeyedStreams, accept_or_resample, inverse_cdf, shape_probs


@dataclass
class Request:
    """ref:engine.py:36-61 (validation kept)."""

    prompts: list
    max_new_tokens: int
    temperature: float = 1.0
    top_p: float = 1.0
    eos_token: int | None = None
    strategy: str = "pad"
    seed: int = 0
    sequence_ids: list | None = None

    def __post_init__(self):
        if len(self.prompts) < 1:
            raise ValueError("batch size must be >= 1")
        if self.max_new_tokens < 1:
            raise ValueError("max_new_tokens must be >= 1")
        if any(len(p) < 1 for p in self.prompts):
            raise ValueError("every prompt needs at least one token")
        if self.sequence_ids is None:
            self.sequence_ids = list(range(len(self.prompts)))
        elif len(self.sequence_ids) != len(self.prompts):
            raise ValueError("sequence_ids must match batch size")


@dataclass
class Outcome:
    mode: str
    tokens: list
    logprobs: list
    finish_reason: list
    completion_step: list
    steps: list = field(default_factory=list)
    main_calls: int = 0
    draft_calls: int = 0


class OracleModel:
    """MainModel equivalent (ref:model.py:288-332)."""

    def __init__(self, weights, n_slot, strategy="pad", quantized=False):
        g = weights["geometry"]
        self.w, self.strategy = weights, strategy
        self.cache = RaggedCache(g.n_layer, n_slot, g.n_head, g.d_head)
        self.vocab_size, self.max_seq_len = g.vocab_size, g.max_seq_len
        # INT8 W8A8 path (ref:model.py:296-302 `quantized=True`)
        self.qw = None
        if quantized:
            from .quant import prepare
            self.qw = prepare(weights)

    def _fwd(self, slots, blocks):
        if self.qw is not None:
            from .quant import forward_ragged_int8
            return forward_ragged_int8(self.w, self.qw, self.cache, slots, blocks, self.strategy)
        return forward_ragged(self.w, self.cache, slots, blocks, self.strategy)

    def prefill(self, slot, prompt):
        if len(prompt) == 0:
            raise ValueError("empty prompt: prefill needs at least one token")
        if self.cache.length(slot) != 0:
            raise ValueError(f"sequence {slot} already has cached context")
        return self._fwd([slot], [list(prompt)])[0][-1]

    def forward(self, slots, blocks):
        return self._fwd(slots, blocks)

    def rollback(self, slot, n):
        self.cache.truncate(slot, n)

    def length(self, slot):
        return self.cache.length(slot)


def blake_perturbation(seed: int, prefix, vocab: int) -> tuple[float, int]:
    """(u, y) from blake2b-128(seed i64 LE || prefix i64 LE) (ref:model.py:370-377)."""
    data = int(seed).to_bytes(8, "little", signed=True)
    data += np.asarray(prefix, dtype=np.int64).tobytes()
    dg = hashlib.blake2b(data, digest_size=16).digest()
    return int.from_bytes(dg[:8], "little") / 2.0 ** 64, \
        int.from_bytes(dg[8:], "little") % vocab


class OracleAlignedDraft:
    """SyntheticAlignedDraft equivalent (ref:model.py:335-415): the main
    weights on a private cache; a row becomes a point mass on y whenever the
    hash draw u >= alignment."""

    def __init__(self, weights, alignment, perturb_seed, n_slot, strategy="pad"):
        if not 0.0 <= alignment <= 1.0:
            raise ValueError(f"alignment must be in [0, 1], got {alignment}")
        self.inner = OracleModel(weights, n_slot, strategy)
        self.alignment, self.seed = float(alignment), int(perturb_seed)
        self.hist = [[] for _ in range(n_slot)]
        self.vocab_size, self.max_seq_len = self.inner.vocab_size, self.inner.max_seq_len

    def _mix(self, slot, raw, base):
        if self.alignment == 1.0:
            return raw
        out = raw.copy()
        for j in range(raw.shape[0]):
            u, y = blake_perturbation(self.seed, self.hist[slot][:base + j + 1],
                                      self.vocab_size)
            if u >= self.alignment:
                out[j] = -np.inf
                out[j, y] = 0.0
        return out

    def prefill(self, slot, prompt):
        base = len(self.hist[slot])
        raw = self.inner.prefill(slot, prompt)
        self.hist[slot] = list(prompt)
        return self._mix(slot, raw[None, :], base + len(prompt) - 1)[0]

    def forward(self, slots, blocks):
        outs = []
        for s, blk, raw in zip(slots, blocks, self.inner.forward(slots, blocks)):
            base = len(self.hist[s])
            self.hist[s].extend(blk)
            outs.append(self._mix(s, raw, base))
        return outs

    def rollback(self, slot, n):
        self.inner.rollback(slot, n)
        del self.hist[slot][n:]

    def length(self, slot):
        return self.inner.length(slot)


def _lp(raw, tok):
    """ref:engine.py:99-100 (unshaped logits)."""
    return float(raw[tok] - logsumexp(raw))


def _clip(emitted, n_done, budget, eos):
    """EOS cut then length clip (ref:engine.py:103-117)."""
    why = None
    if eos is not None and eos in emitted:
        emitted = emitted[:emitted.index(eos) + 1]
        why = "eos"
    room = budget - n_done
    if len(emitted) > room:
        emitted, why = emitted[:room], "length"
    elif len(emitted) == room and why is None:
        why = "length"
    return emitted, why


def run_regular(main, req: Request) -> Outcome:
    """One token per sequence per step (ref:engine.py:120-197)."""
    b = len(req.prompts)
    for p in req.prompts:
        if len(p) + req.max_new_tokens > main.max_seq_len:
            raise ValueError("prompt + max_new_tokens exceeds max_seq_len")
    greedy = req.temperature == 0.0
    rs = KeyedStreams(req.seed)
    cur = [main.prefill(s, req.prompts[s]) for s in range(b)]
    res = Outcome("regular", [[] for _ in range(b)], [[] for _ in range(b)],
                  [""] * b, [0] * b, main_calls=b)
    done = [False] * b
    step = 0
    while not all(done):
        step += 1
        live = [s for s in range(b) if not done[s]]
        em = []
        for s in live:
            raw = cur[s]
            pos = len(req.prompts[s]) + len(res.tokens[s])
            if greedy:
                tok = int(np.argmax(raw))
            else:
                tok = inverse_cdf(shape_probs(raw, req.temperature, req.top_p),
                                  rs.verify(req.sequence_ids[s], pos)())
            res.tokens[s].append(tok)
            res.logprobs[s].append(_lp(raw, tok))
            em.append((tok,))
            if req.eos_token is not None and tok == req.eos_token:
                done[s], res.finish_reason[s] = True, "eos"
            elif len(res.tokens[s]) >= req.max_new_tokens:
                done[s], res.finish_reason[s] = True, "length"
        go = [s for s in live if not done[s]]
        if go:
            outs = main.forward(go, [[res.tokens[s][-1]] for s in go])
            res.main_calls += len(go)
            for s, o in zip(go, outs):
                cur[s] = o[-1]
        for s in live:
            if done[s] and res.completion_step[s] == 0:
                res.completion_step[s] = step
        res.steps.append(dict(draft_length=0, slots=tuple(live),
                              accepted=tuple(0 for _ in live), emitted=tuple(em),
                              finished=tuple(done[s] for s in live)))
    return res


def run_speculative(main, draft, req: Request, ctl) -> Outcome:
    """Batched speculative decoding (ref:engine.py:200-385)."""
    b = len(req.prompts)
    if main.vocab_size != draft.vocab_size:
        raise ValueError("vocab mismatch")
    for p in req.prompts:
        if len(p) + req.max_new_tokens + ctl.max_length > main.max_seq_len:
            raise ValueError("context overflow")
    greedy = req.temperature == 0.0
    rs = KeyedStreams(req.seed)
    sid = req.sequence_ids
    shp = lambda raw: shape_probs(raw, req.temperature, req.top_p)
    com = [list(p) for p in req.prompts]
    res = Outcome("speculative", [[] for _ in range(b)], [[] for _ in range(b)],
                  [""] * b, [0] * b)
    done = [False] * b
    step = 0
    while not all(done):
        step += 1
        k = ctl.length
        live = [s for s in range(b) if not done[s]]
        prop = {s: [] for s in live}
        pd = {s: [] for s in live}
        feed = {s: com[s][draft.length(s):] for s in live}
        for j in range(k):                                   # draft phase
            outs = draft.forward(live, [feed[s] for s in live])
            res.draft_calls += len(live)
            for s, o in zip(live, outs):
                if greedy:
                    t = int(np.argmax(o[-1]))
                else:
                    dist = shp(o[-1])
                    t = inverse_cdf(dist, rs.draft(sid[s], len(com[s]) + j)())
                    pd[s].append(dist)
                prop[s].append(t)
                feed[s] = [t]
        outs = main.forward(live, [com[s][main.length(s):] + prop[s] for s in live])
        res.main_calls += len(live)
        ver = {s: o[-(k + 1):] for s, o in zip(live, outs)}
        acc, core = {}, {}
        for s in live:                                       # accept pass
            c0, x, em = len(com[s]), 0, []
            for j in range(k):
                t = prop[s][j]
                if greedy:
                    am = int(np.argmax(ver[s][j]))
                    ok, fix = t == am, am
                else:
                    ok, fix = accept_or_resample(shp(ver[s][j]), pd[s][j], t,
                                                 rs.verify(sid[s], c0 + j))
                if ok:
                    em.append(t)
                    x += 1
                else:
                    em.append(fix)
                    break
            acc[s], core[s] = x, em
        bonus = [s for s in live if acc[s] == k
                 and not (req.eos_token is not None and req.eos_token in core[s])
                 and req.max_new_tokens - len(res.tokens[s]) > k]
        bpd = {}
        if bonus and not greedy:
            outs = draft.forward(bonus, [[prop[s][-1]] for s in bonus])
            res.draft_calls += len(bonus)
            bpd = {s: shp(o[-1]) for s, o in zip(bonus, outs)}
        emitted_step = {}
        for s in live:
            em = core[s]
            if s in bpd or (greedy and s in bonus):
                pos = len(com[s]) + k
                if greedy:
                    em.append(int(np.argmax(ver[s][k])))
                else:
                    tb = inverse_cdf(bpd[s], rs.draft(sid[s], pos)())
                    ok, fix = accept_or_resample(shp(ver[s][k]), bpd[s], tb,
                                                 rs.verify(sid[s], pos))
                    em.append(tb if ok else fix)
            em, why = _clip(em, len(res.tokens[s]), req.max_new_tokens,
                            req.eos_token)
            for j, t in enumerate(em):
                res.logprobs[s].append(_lp(ver[s][j], t))
            res.tokens[s].extend(em)
            com[s].extend(em)
            emitted_step[s] = tuple(em)
            if why is not None:
                done[s], res.finish_reason[s] = True, why
            tgt = len(com[s]) - 1
            main.rollback(s, min(main.length(s), tgt))
            draft.rollback(s, min(draft.length(s), tgt))
        ctl.observe([acc[s] for s in live])
        for s in live:
            if done[s] and res.completion_step[s] == 0:
                res.completion_step[s] = step
        res.steps.append(dict(draft_length=k, slots=tuple(live),
                              accepted=tuple(acc[s] for s in live),
                              emitted=tuple(emitted_step[s] for s in live),
                              finished=tuple(done[s] for s in live),
                              kv_lengths=tuple(len(c) for c in com)))
    return res
