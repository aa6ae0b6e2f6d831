"""Regular and batched speculative decoding — the reference's decode API.

Same types and signatures as ref:engine.py:36-385.  Dispatch:

* both providers are `CudaModel`s on one context and the controller is one of
  ours -> the device-computed loop in libbass (`bass_spec_generate` /
  `bass_regular_generate`): forwards, draft picks, accept/resample, bonus,
  finalize and logprobs all run on the GPU, one small read-back per step;
* anything else (e.g. a reference provider, `CudaAlignedDraft`) -> the
  reference-style host loop over the LogitsProvider protocol, with the
  sampling decisions made by the device kernels of `sampling.py`.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .attention import AttentionStrategy
from .control import AdaptiveDraftController, DraftLengthState, FixedDraftController
from .model import CudaModel
from .sampling import ROLE_DRAFT, ROLE_VERIFY, device_accept, device_shape_sample, device_uniforms


@dataclass
class GenerationRequest:
    """ref:engine.py:36-61."""

    prompts: list
    max_new_tokens: int
    temperature: float = 1.0
    top_p: float = 1.0
    eos_token: int | None = None
    strategy: AttentionStrategy = AttentionStrategy.PAD
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

    @property
    def batch_size(self) -> int:
        return len(self.prompts)


@dataclass(frozen=True)
class SpecStepOutcome:
    """ref:engine.py:64-75."""

    step_index: int
    draft_length: int
    slots: tuple
    accepted: tuple
    emitted: tuple
    finished: tuple
    kv_lengths: tuple
    duration_s: float


@dataclass
class GenerationResult:
    """ref:engine.py:78-91."""

    mode: str
    prompts: list
    sequence_ids: list
    tokens: list
    logprobs: list
    finish_reason: list
    completion_step: list
    finish_wall_s: list
    steps: list
    wall_time_s: float
    main_forward_calls: int
    draft_forward_calls: int


def step_trace(result: GenerationResult) -> list:
    return result.steps


# ------------------------------------------------------------ device path
class CudaEngine:
    """libbass engine over two CudaModels' weights and caches."""

    def __init__(self, main: CudaModel, draft: CudaModel | None = None):
        self.main, self.draft, self.ctx = main, draft, main.ctx
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.bass_engine_create(
            main.weights.handle, main.kv, draft.weights.handle if draft else None,
            draft.kv if draft else None, C.byref(h)))
        self.handle = h

    def set_strategy(self, strategy):
        from .attention import strategy_code
        self.ctx.check(self.ctx.lib.bass_engine_set_strategy(self.handle, strategy_code(strategy)))

    def set_loop(self, mode: str):
        """"device" (default): every step after the prompt step runs from one
        CUDA graph with the step planning, bookkeeping and Algorithm 1 on the
        GPU (one host synchronisation per generation); "host": the host plans
        every step and reads its outcome back.  Identical results."""
        code = {"host": L.LOOP_HOST, "device": L.LOOP_DEVICE}[mode]
        self.ctx.check(self.ctx.lib.bass_engine_set_loop(self.handle, code))

    def loop_info(self) -> dict:
        """How the last speculative generation ran: loop mode, host
        synchronisations, loop-graph captures so far."""
        mode, syncs, builds = C.c_int32(), C.c_int32(), C.c_int64()
        self.ctx.check(self.ctx.lib.bass_engine_loop_info(self.handle, C.byref(mode), C.byref(syncs),
                                                          C.byref(builds)))
        return {"mode": "device" if mode.value == L.LOOP_DEVICE else "host", "syncs": syncs.value,
                "graph_builds": builds.value}

    def __del__(self):
        try:
            if getattr(self, "handle", None) and L.alive():
                self.ctx.lib.bass_engine_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def run(self, request: GenerationRequest, controller=None, speculative=True,
            align: float = -1.0, align_seed: int = 0, align_tokens=None, max_steps=None):
        """Run one generation; returns (GenerationResult, raw arrays dict)."""
        b, maxnew = request.batch_size, request.max_new_tokens
        flat = np.ascontiguousarray(np.concatenate([np.asarray(p, dtype=np.int32)
                                                    for p in request.prompts]))
        offs = np.zeros(b + 1, dtype=np.int32)
        offs[1:] = np.cumsum([len(p) for p in request.prompts])
        sids = np.ascontiguousarray(np.asarray(request.sequence_ids, dtype=np.int64))
        req = L.GenRequest()
        req.batch, req.prompt_tokens, req.prompt_offsets = b, L.ptr(flat, C.c_int32), \
            L.ptr(offs, C.c_int32)
        req.max_new_tokens = maxnew
        req.temperature, req.top_p = float(request.temperature), float(request.top_p)
        req.eos_token = -1 if request.eos_token is None else int(request.eos_token)
        req.seed = int(request.seed) & 0xFFFFFFFFFFFFFFFF
        req.sequence_ids = L.ptr(sids, C.c_int64)
        if isinstance(controller, FixedDraftController):
            req.ctl_fixed = controller.length
        elif isinstance(controller, AdaptiveDraftController):
            st = controller.state
            req.ctl_fixed, req.l0, req.s0 = 0, st.l_draft, st.s
            req.incre, req.mod, req.limit = st.params.incre, st.params.mod, st.params.limit
        req.align = float(align)
        req.align_seed = int(align_seed) & 0xFFFFFFFFFFFFFFFF
        if align_tokens is not None:
            at = np.ascontiguousarray(np.asarray(align_tokens, dtype=np.int32).reshape(b, maxnew))
            req.align_tokens = L.ptr(at, C.c_int32)
        steps_cap = max_steps or (maxnew + 8)
        arr = {
            "tokens": np.zeros((b, maxnew), np.int32), "logprobs": np.zeros((b, maxnew), np.float64),
            "n_tokens": np.zeros(b, np.int32), "finish_reason": np.zeros(b, np.int32),
            "completion_step": np.zeros(b, np.int32), "finish_wall_s": np.zeros(b, np.float64),
            "step_draft_len": np.zeros(steps_cap, np.int32),
            "step_accepted": np.zeros((steps_cap, b), np.int32),
            "step_emitted": np.zeros((steps_cap, b), np.int32),
            "step_kv_len": np.zeros((steps_cap, b), np.int32),
            "step_wall_s": np.zeros(steps_cap, np.float64),
        }
        res = L.GenResult()
        ct = {"tokens": C.c_int32, "logprobs": C.c_double, "n_tokens": C.c_int32,
              "finish_reason": C.c_int32, "completion_step": C.c_int32,
              "finish_wall_s": C.c_double, "step_draft_len": C.c_int32,
              "step_accepted": C.c_int32, "step_emitted": C.c_int32, "step_kv_len": C.c_int32,
              "step_wall_s": C.c_double}
        for k, t in ct.items():
            setattr(res, k, L.ptr(arr[k], t))
        res.max_steps = steps_cap
        fn = self.ctx.lib.bass_spec_generate if speculative else self.ctx.lib.bass_regular_generate
        self.ctx.check(fn(self.handle, C.byref(req), C.byref(res)))
        if isinstance(controller, AdaptiveDraftController) and speculative:
            controller.state = DraftLengthState(res.final_l_draft, res.final_s,
                                                controller.state.params)
        return _to_result(request, arr, res, "speculative" if speculative else "regular"), arr, res


def _to_result(request, arr, res, mode) -> GenerationResult:
    b = request.batch_size
    n = arr["n_tokens"]
    tokens = [arr["tokens"][s, :n[s]].tolist() for s in range(b)]
    logprobs = [arr["logprobs"][s, :n[s]].tolist() for s in range(b)]
    reason = ["eos" if r == 0 else "length" for r in arr["finish_reason"]]
    steps, cursor = [], [0] * b
    for i in range(min(res.n_steps, res.max_steps)):
        acc_row, em_row = arr["step_accepted"][i], arr["step_emitted"][i]
        slots = tuple(s for s in range(b) if acc_row[s] >= 0)
        emitted = []
        for s in slots:
            k = int(em_row[s])
            emitted.append(tuple(tokens[s][cursor[s]:cursor[s] + k]))
            cursor[s] += k
        steps.append(SpecStepOutcome(
            step_index=i + 1, draft_length=int(arr["step_draft_len"][i]), slots=slots,
            accepted=tuple(int(acc_row[s]) for s in slots), emitted=tuple(emitted),
            finished=tuple(bool(arr["completion_step"][s] and arr["completion_step"][s] <= i + 1)
                           for s in slots),
            kv_lengths=tuple(int(x) for x in arr["step_kv_len"][i]),
            duration_s=float(arr["step_wall_s"][i])))
    return GenerationResult(
        mode=mode, prompts=request.prompts, sequence_ids=list(request.sequence_ids),
        tokens=tokens, logprobs=logprobs, finish_reason=reason,
        completion_step=arr["completion_step"].tolist(),
        finish_wall_s=arr["finish_wall_s"].tolist(), steps=steps, wall_time_s=float(res.wall_s),
        main_forward_calls=int(res.main_forward_calls),
        draft_forward_calls=int(res.draft_forward_calls))


def _device_pair(main, draft, controller) -> bool:
    ok = isinstance(main, CudaModel) and (draft is None or (
        isinstance(draft, CudaModel) and draft.ctx is main.ctx))
    if controller is not None:
        ok = ok and isinstance(controller, (AdaptiveDraftController, FixedDraftController))
    return ok


def _engine_for(main, draft):
    """One engine per (main, draft) pair, owned by the main provider."""
    cache = main.__dict__.setdefault("_engines", {})
    eng = cache.get(id(draft))
    if eng is None or eng.draft is not draft:
        eng = CudaEngine(main, draft)
        cache[id(draft)] = eng
    return eng


def decode_regular(main, request: GenerationRequest) -> GenerationResult:
    """ref:engine.py:120-197."""
    if _device_pair(main, None, None):
        eng = _engine_for(main, None)
        eng.set_strategy(main.strategy)
        return eng.run(request, None, speculative=False)[0]
    return _host_regular(main, request)


def decode_speculative(main, draft, request: GenerationRequest, controller) -> GenerationResult:
    """ref:engine.py:200-385."""
    if main.vocab_size != draft.vocab_size:
        raise ValueError(f"vocab mismatch: main {main.vocab_size} vs draft {draft.vocab_size}")
    if _device_pair(main, draft, controller):
        eng = _engine_for(main, draft)
        eng.set_strategy(main.strategy)
        return eng.run(request, controller, speculative=True)[0]
    return _host_speculative(main, draft, request, controller)


# ------------------------------------------------------------- host loop
def _ctx_of(*providers):
    from .model import CudaContext
    for p in providers:
        for obj in (p, getattr(p, "inner", None)):
            if isinstance(obj, CudaModel):
                return obj.ctx
    return CudaContext.default()


class _Sampler:
    """Device sampling decisions for the host loop."""

    def __init__(self, ctx, request):
        self.ctx, self.req = ctx, request

    def draw(self, raw, sid, role, pos):
        u = device_uniforms(self.ctx, self.req.seed, [sid], [role], [pos])[0, 0]
        return int(device_shape_sample(self.ctx, raw[None, :], self.req.temperature,
                                       self.req.top_p, [u])[0])

    def accept(self, q_raw, p_raw, tok, sid, pos):
        acc, cor = device_accept(self.ctx, q_raw[None, :], p_raw[None, :], self.req.temperature,
                                 self.req.top_p, [tok], self.req.seed, [sid], [pos])
        return bool(acc[0]), (None if acc[0] else int(cor[0]))


def _lse(raw):
    m = np.max(raw)
    return float(m + np.log(np.sum(np.exp(raw - m))))


def _finalize(emitted, n_done, budget, eos):
    why = None
    if eos is not None and eos in emitted:
        emitted, why = emitted[:emitted.index(eos) + 1], "eos"
    room = budget - n_done
    if len(emitted) > room:
        emitted, why = emitted[:room], "length"
    elif len(emitted) == room and why is None:
        why = "length"
    return emitted, why


def _host_regular(main, request):
    b = request.batch_size
    for p in request.prompts:
        if len(p) + request.max_new_tokens > main.max_seq_len:
            raise ValueError(f"prompt ({len(p)}) + max_new_tokens ({request.max_new_tokens}) "
                             f"exceeds max_seq_len {main.max_seq_len}")
    greedy = request.temperature == 0.0
    smp = _Sampler(_ctx_of(main), request)
    t0 = time.perf_counter()
    cur = [main.prefill(s, request.prompts[s]) for s in range(b)]
    calls = b
    gen = [[] for _ in range(b)]
    lps = [[] for _ in range(b)]
    why = [""] * b
    cstep = [0] * b
    fin_t = [0.0] * b
    done = [False] * b
    steps = []
    k = 0
    while not all(done):
        k += 1
        ts = time.perf_counter()
        live = [s for s in range(b) if not done[s]]
        em = []
        for s in live:
            raw = cur[s]
            pos = len(request.prompts[s]) + len(gen[s])
            tok = int(np.argmax(raw)) if greedy else smp.draw(raw, request.sequence_ids[s],
                                                              ROLE_VERIFY, pos)
            gen[s].append(tok)
            lps[s].append(float(raw[tok]) - _lse(raw))
            em.append((tok,))
            if request.eos_token is not None and tok == request.eos_token:
                done[s], why[s] = True, "eos"
            elif len(gen[s]) >= request.max_new_tokens:
                done[s], why[s] = True, "length"
        go = [s for s in live if not done[s]]
        if go:
            for s, o in zip(go, main.forward(go, [[gen[s][-1]] for s in go])):
                cur[s] = o[-1]
            calls += len(go)
        now = time.perf_counter()
        for s in live:
            if done[s] and cstep[s] == 0:
                cstep[s], fin_t[s] = k, now - t0
        steps.append(SpecStepOutcome(k, 0, tuple(live), tuple(0 for _ in live), tuple(em),
                                     tuple(done[s] for s in live),
                                     tuple(len(request.prompts[s]) + len(gen[s]) for s in range(b)),
                                     now - ts))
    return GenerationResult("regular", request.prompts, list(request.sequence_ids), gen, lps, why,
                            cstep, fin_t, steps, time.perf_counter() - t0, calls, 0)


def _host_speculative(main, draft, request, controller):
    b = request.batch_size
    limit = controller.max_length
    for p in request.prompts:
        if len(p) + request.max_new_tokens + limit > main.max_seq_len:
            raise ValueError(f"context overflow: prompt ({len(p)}) + max_new_tokens "
                             f"({request.max_new_tokens}) + draft limit ({limit}) exceeds "
                             f"max_seq_len {main.max_seq_len}")
    greedy = request.temperature == 0.0
    smp = _Sampler(_ctx_of(main, draft), request)
    sid = request.sequence_ids
    com = [list(p) for p in request.prompts]
    gen = [[] for _ in range(b)]
    lps = [[] for _ in range(b)]
    why = [""] * b
    cstep = [0] * b
    fin_t = [0.0] * b
    done = [False] * b
    steps = []
    mcalls = dcalls = 0
    k = 0
    t0 = time.perf_counter()
    while not all(done):
        k += 1
        ts = time.perf_counter()
        l = controller.length
        live = [s for s in range(b) if not done[s]]
        prop = {s: [] for s in live}
        praw = {s: [] for s in live}
        feed = {s: com[s][draft.length(s):] for s in live}
        for j in range(l):
            outs = draft.forward(live, [feed[s] for s in live])
            dcalls += len(live)
            for s, o in zip(live, outs):
                raw = o[-1]
                t = int(np.argmax(raw)) if greedy else smp.draw(raw, sid[s], ROLE_DRAFT,
                                                                len(com[s]) + j)
                praw[s].append(raw)
                prop[s].append(t)
                feed[s] = [t]
        outs = main.forward(live, [com[s][main.length(s):] + prop[s] for s in live])
        mcalls += len(live)
        ver = {s: o[-(l + 1):] for s, o in zip(live, outs)}
        acc, core = {}, {}
        for s in live:
            c0, x, em = len(com[s]), 0, []
            for j in range(l):
                t = prop[s][j]
                if greedy:
                    am = int(np.argmax(ver[s][j]))
                    ok, fix = t == am, am
                else:
                    ok, fix = smp.accept(ver[s][j], praw[s][j], t, sid[s], c0 + j)
                if ok:
                    em.append(t)
                    x += 1
                else:
                    em.append(fix)
                    break
            acc[s], core[s] = x, em
        bonus = [s for s in live if acc[s] == l
                 and not (request.eos_token is not None and request.eos_token in core[s])
                 and request.max_new_tokens - len(gen[s]) > l]
        braw = {}
        if bonus and not greedy:
            outs = draft.forward(bonus, [[prop[s][-1]] for s in bonus])
            dcalls += len(bonus)
            braw = {s: o[-1] for s, o in zip(bonus, outs)}
        step_em = {}
        for s in live:
            em = core[s]
            if s in bonus:
                pos = len(com[s]) + l
                if greedy:
                    em.append(int(np.argmax(ver[s][l])))
                else:
                    tb = smp.draw(braw[s], sid[s], ROLE_DRAFT, pos)
                    ok, fix = smp.accept(ver[s][l], braw[s], tb, sid[s], pos)
                    em.append(tb if ok else fix)
            em, w = _finalize(em, len(gen[s]), request.max_new_tokens, request.eos_token)
            for j, t in enumerate(em):
                lps[s].append(float(ver[s][j][t]) - _lse(ver[s][j]))
            gen[s].extend(em)
            com[s].extend(em)
            step_em[s] = tuple(em)
            if w is not None:
                done[s], why[s] = True, w
            tgt = len(com[s]) - 1
            main.rollback(s, min(main.length(s), tgt))
            draft.rollback(s, min(draft.length(s), tgt))
        controller.observe([acc[s] for s in live])
        now = time.perf_counter()
        for s in live:
            if done[s] and cstep[s] == 0:
                cstep[s], fin_t[s] = k, now - t0
        steps.append(SpecStepOutcome(k, l, tuple(live), tuple(acc[s] for s in live),
                                     tuple(step_em[s] for s in live),
                                     tuple(done[s] for s in live),
                                     tuple(len(c) for c in com), now - ts))
    return GenerationResult("speculative", request.prompts, list(sid), gen, lps, why, cstep,
                            fin_t, steps, time.perf_counter() - t0, mcalls, dcalls)
