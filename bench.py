"""BASS on B200: per-sequence ms/token and tokens/s for batched speculative
decoding of a 7.8B-class random-init model (BASELINE.json configs[1]).

One bench *step* = one full generation through the public C-ABI engine
(`bass_spec_generate`): 8 synthetic 128-token prompts per GPU -> 128 new
tokens each, greedy, dynamic draft length (Algorithm 1), 310M-class draft.
Weights are random-init bf16 (no checkpoints offline) and are 17 GB per
replica, far larger than L2, so no L2 flush is needed between steps.

Draft proposals follow the benchmark harness of SURVEY 7.2(2): the draft runs
its full forward every draft token (cost-faithful), and its proposal is
overridden per (sequence id, position) by a keyed hash — the main model's
greedy token (from a greedy regular-decoding run of the same prompts) with
probability `--align` (default 0.874, the paper's measured acceptance,
PAPER.md:578), else a hash token.  Greedy outputs are unaffected (spec ==
regular) — the override only sets the acceptance regime.

    python bench.py [--gpus N --steps K --warmup W]            # our arm
    python bench.py --impl reference ...                       # CPU reference arm
Multi-GPU: torchrun, one rank per GPU, sequences sharded by rank (replica per
GPU, no collectives on the hot path; NCCL only for barriers and the final
max/sum reductions).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "per-seq ms/token + tokens/sec at batch 8 (7.8B-class); ragged-attn HBM GB/s"

CONFIGS = {
    # name: main (L, H, d, dh, V, S), draft (...), batch/GPU, prompt, new, T, top_p
    "c2": dict(main=(30, 36, 4608, 128, 50272, 2048), draft=(4, 16, 2048, 128, 50272, 2048),
               batch=8, prompt=128, new=128, temperature=0.0, top_p=1.0,
               workload="7.8B-class main (L30 d4608 H36 V50272) + 310M-class draft (L4 d2048 H16), "
                        "batch 8/GPU, bf16, greedy, dynamic draft length"),
    "c3": dict(main=(40, 40, 5120, 128, 50272, 2048), draft=(12, 12, 768, 64, 50272, 2048),
               batch=8, prompt=128, new=128, temperature=0.2, top_p=0.95,
               workload="OPT-13B-shape main + OPT-125M-shape draft, batch 8/GPU, bf16, sampled "
                        "T=0.2 top_p=0.95"),
    # BASELINE configs[4]: 64 global sequences sharded over the ranks (strong
    # scaling: total work fixed), ~256-token contexts
    "c5": dict(main=(30, 36, 4608, 128, 50272, 2048), draft=(4, 16, 2048, 128, 50272, 2048),
               batch=64, global_batch=64, prompt=128, new=128, temperature=0.0, top_p=1.0,
               workload="7.8B-class main + 310M-class draft, 64 sequences sharded over the GPUs (replica per "
                        "GPU), bf16, greedy, dynamic draft length"),
    "small": dict(main=(4, 8, 512, 64, 4096, 1024), draft=(1, 8, 512, 64, 4096, 1024),
                  batch=8, prompt=64, new=64, temperature=0.0, top_p=1.0,
                  workload="small smoke config"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.samples, self._stop = device, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------- trace analysis
TRACE_CLASSES = {1: "gemm", 2: "attn", 3: "norm", 4: "combine"}


def _union_ms(iv):
    """Total length (ms) of the union of [start, end] ns intervals."""
    if not len(iv):
        return 0.0
    o = np.argsort(iv[:, 0], kind="stable")
    s0, e0 = iv[o, 0], iv[o, 1]
    ce = np.maximum.accumulate(e0)
    new_blk = np.r_[True, s0[1:] > ce[:-1]]
    starts = s0[new_blk]
    ends = ce[np.r_[np.flatnonzero(new_blk)[1:] - 1, len(ce) - 1]]
    return float((ends - starts).sum()) / 1e6


def trace_summary(rec):
    """Per kernel class: union time, launches, median launch span, from the
    {t0, t1, smid, tag} records of bass_trace_read (tag = class | seq << 4)."""
    rec = rec[rec[:, 0] > 0]
    cls = rec[:, 3] & 15
    seq = rec[:, 3] >> 4
    out = {"classes": {}}
    for c, name in TRACE_CLASSES.items():
        r, sq = rec[cls == c], seq[cls == c]
        if not len(r):
            continue
        o = np.argsort(sq, kind="stable")
        r, sq = r[o], sq[o]
        cut = np.flatnonzero(np.diff(sq)) + 1
        spans = [(x[:, 1].max() - x[:, 0].min()) / 1e3 for x in np.split(r, cut)]
        out["classes"][name] = {"union_ms": _union_ms(r[:, :2]), "launches": len(spans),
                                "median_span_us": float(np.median(spans)), "ctas": int(len(r))}
    # critical-path attribution: walking the launches in issue order, the part
    # of launch i's [first CTA start, last CTA end] that lies past every
    # earlier launch's end belongs to launch i alone — the per-class sums
    # partition the traced timeline (their total is the busy time), unlike
    # the union above, which also counts CTAs launched early (PDL) that
    # wait on their predecessor
    if len(rec):
        o = np.argsort(seq, kind="stable")
        r, sq, cl = rec[o], seq[o], cls[o]
        cut = np.flatnonzero(np.diff(sq)) + 1
        frontier = 0
        exposed = {}
        for x, c in zip(np.split(r, cut), np.split(cl, cut)):
            s0, e1 = int(x[:, 0].min()), int(x[:, 1].max())
            exp = max(0, e1 - max(frontier, s0))
            frontier = max(frontier, e1)
            name = TRACE_CLASSES.get(int(c[0]), "other")
            exposed[name] = exposed.get(name, 0) + exp
        for name, ns in exposed.items():
            if name in out["classes"]:
                out["classes"][name]["exposed_ms"] = ns / 1e6
    out["untraced_ms"] = None
    if len(rec):
        busy = _union_ms(rec[:, :2])
        out["untraced_ms"] = (rec[:, 1].max() - rec[:, 0].min()) / 1e6 - busy   # no traced CTA resident (sampling, embed, host gaps)
    return out


# ------------------------------------------- ragged attention (metric part 3)
def ragged_attention_point(ctx, hbm, b=64, L=8192, q=17, H=36, dh=128, reps=10, seed=7):
    """The metric's "ragged-attn HBM GB/s": the RAGGED attention kernel alone
    at the C4 sweep's largest point (b = 64, L_i ~ U[L/2, L] seeded, q = k + 1
    = 17 new rows per sequence, H = 36, d_head = 128), device-timed
    (bass_attention_bench: back-to-back launches, CUDA events); bytes = real
    K/V rows + Q in + O out, K/V ~ 9.7 GB >> L2."""
    import ctypes as C
    import torch
    from paper_2404_15778_b200 import _lib as L_
    from paper_2404_15778_b200.attention import strategy_code
    rng = np.random.default_rng(seed)
    lens = rng.integers(L // 2, L + 1, b)
    stride = int(lens.max())
    K = torch.randn(b * H * stride * dh, device="cuda", dtype=torch.bfloat16)
    V = torch.randn_like(K)
    q_lens = np.full(b, q)
    cu = np.concatenate([[0], np.cumsum(q_lens)]).astype(np.int32)
    offs = (lens - q_lens).astype(np.int32)
    Q = torch.randn(int(cu[-1]), H, dh, device="cuda", dtype=torch.bfloat16)
    out = torch.empty_like(Q)
    ms = C.c_double()
    torch.cuda.synchronize()
    ctx.check(ctx.lib.bass_attention_bench(ctx.handle, strategy_code("ragged"), b, H, dh, L_.ptr(cu, C.c_int32),
                                           L_.ptr(offs, C.c_int32), C.c_void_p(Q.data_ptr()),
                                           C.c_void_p(K.data_ptr()), C.c_void_p(V.data_ptr()), stride, 1,
                                           C.c_void_p(out.data_ptr()), reps, C.byref(ms)))
    by = sum(2 * H * int(n) * dh * 2 + 2 * H * q * dh * 2 for n in lens)
    gbs = by / (ms.value / 1e3) / 1e9
    del K, V, Q, out
    torch.cuda.empty_cache()
    return {"kernel": "attn_stream_kernel (RAGGED)", "b": b, "L": f"U[{L // 2}, {L}]", "q": q, "H": H,
            "d_head": dh, "us_per_launch": ms.value * 1e3, "bytes_per_launch": by, "GB/s": gbs, "peak": hbm,
            "frac": gbs / hbm, "timing": "device (CUDA events), back-to-back launches, K/V >> L2"}


# ------------------------------------------------- acceptance-harness schedule
_M64 = (1 << 64) - 1


def _splitmix64(x):
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def harness_schedule(batch, prompt, new, align, align_seed=99, sids=None, params=(7, 2, 10, 32)):
    """Per-step draft lengths of a greedy generation under the keyed
    acceptance override (csrc/sampling_kernels.cuh aligned_override: the
    proposal at absolute position p is the main model's greedy token iff
    u(seed, sid, p) < align) driven by Algorithm 1 (ref:draft_control.py:49-69),
    with the engine's bonus / length rules (ref:engine.py:276-349).  No model
    is needed: it reproduces the GPU run's steps and draft lengths exactly
    (up to hash tokens that happen to equal the greedy token, p ~ 1/V).
    align < 0 (natural acceptance of a random-init draft ~ 0): nothing is
    accepted.  Returns (list of l per step, tokens per sequence)."""
    l0, incre, mod, limit = params
    sids = list(range(batch)) if sids is None else sids
    C, gen, done = [prompt] * batch, [0] * batch, [False] * batch
    l, s, ls = l0, 0, []
    while not all(done):
        accs = []
        for i in range(batch):
            if done[i]:
                continue
            x = 0
            while align >= 0 and x < l:
                h = _splitmix64(align_seed ^ _splitmix64((sids[i] * 0x100000001B3 + C[i] + x) & _M64))
                if (h >> 11) * 2.0 ** -53 >= align:
                    break
                x += 1
            rem = new - gen[i]
            n = min(x + (1 if x < l or rem > l else 0), rem)
            gen[i] += n
            C[i] += n
            done[i] = gen[i] >= new
            accs.append(x)
        ls.append(l)
        if max(accs) == l:
            l, s = min(l + incre, limit), 0
        else:
            l, s = max([1, l - math.ceil(l / mod) - s] + accs), 1
    return ls, new


# ------------------------------------------------------------ CPU reference
def cpu_reference(cfg, step_lengths, tokens_per_seq, batch):
    """Time the oracle port (numpy fp64, all host threads) on a bounded
    sample — one full-width layer (+ head) of each piece a generation is made
    of (ref:model.py:211-245 per-sequence cost structure) — and compose one
    generation from the per-step draft-length schedule:
    T = T_prefill + sum_steps (t_verify + l_step * t_draft_token).
    An extrapolated estimate (kind "port"), not a timed full run."""
    from oracle.cpu_timing import time_generation_pieces
    from oracle.ragged import Geometry
    gm, gd = Geometry(*cfg["main"]), Geometry(*cfg["draft"])
    ctx_len = cfg["prompt"] + cfg["new"] // 2
    k = max(1, int(round(statistics.mean(step_lengths))))
    # the reference runs its dense layers per sequence (ref:model.py:211-245),
    # so a piece's time is linear in the batch: sample at most 8 sequences
    sb = min(batch, 8)
    t0 = time.perf_counter()
    p = {n: t * batch / sb for n, t in time_generation_pieces(gm, gd, sb, cfg["prompt"], ctx_len, k).items()}
    wall = time.perf_counter() - t0
    t_gen = p["prefill_main"] + p["prefill_draft"] + sum(p["verify"] + l * p["draft_token"] for l in step_lengths)
    tps = batch * tokens_per_seq / t_gen
    return {"value": tps, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": (f"extrapolated: oracle numpy fp64, one full-width layer + head per piece (verify "
                       f"{sb}x{k + 1} rows at ctx {ctx_len}, x{batch / sb:g} sequences; one draft token; "
                       f"step-1 prompt blocks) x layer "
                       f"count, composed over a {len(step_lengths)}-step schedule (mean draft length "
                       f"{statistics.mean(step_lengths):.2f}, {tokens_per_seq * batch / len(step_lengths) / batch:.2f} "
                       f"tokens/step/seq); sample wall {wall:.1f}s"),
            "t_gen_s": t_gen, "pieces_s": p,
            "per_seq_ms_per_token": 1000 * t_gen / tokens_per_seq}


def run_reference_arm(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # the GPU arm's acceptance regime, replayed exactly: greedy configs use the
    # keyed override at --align (draft lengths and tokens/step identical to the
    # GPU run); sampled configs the natural acceptance of a random-init draft
    ls, per_seq = harness_schedule(cfg["batch"], cfg["prompt"], cfg["new"],
                                   args.align if cfg["temperature"] == 0.0 else -1.0)
    # each step is one bounded sample (~10-30 s of host work); no warm-up
    # is needed for the CPU port, W is accepted for the interface only
    vals = [cpu_reference(cfg, ls, per_seq, cfg["batch"]) for _ in range(max(1, args.steps))]
    v = statistics.median([x["value"] for x in vals])
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median([x["t_gen_s"] for x in vals]) * 1e3,
            "ms_per_step_kind": "extrapolated (one generation composed from per-layer samples)",
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["workload"], "batch_per_gpu": cfg["batch"],
                       "prompt_len": cfg["prompt"], "max_new_tokens": cfg["new"],
                       "align": args.align, "steps_per_generation": len(ls),
                       "mean_draft_len": statistics.mean(ls)},
            "per_seq_ms_per_token": statistics.median(x["per_seq_ms_per_token"] for x in vals),
            "cpu_baseline": {k_: vals[-1][k_] for k_ in ("kind", "cores", "sample")} | {"value": v,
                                                                                     "unit": "tokens/s"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--align", type=float, default=None,
                    help="keyed-override acceptance (greedy configs; default 0.874). Sampled configs run the "
                         "natural acceptance: an overridden proposal may have zero draft probability")
    ap.add_argument("--strategy", default="ragged", choices=["pad", "split", "ragged"])
    ap.add_argument("--gemm", default="auto", choices=["auto", "simt", "tc"])
    ap.add_argument("--loop", default="device", choices=["device", "host"],
                    help="decode-loop driver: one CUDA graph per generation (device) or per-step host planning")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "int8"],
                    help="int8: the W8A8 path (SURVEY 8(f1), ref:quant.py) for main and draft")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-attn-point", dest="attn_point", action="store_false",
                    help="skip the standalone ragged-attention point (the metric's GB/s part)")
    ap.add_argument("--profile-only", action="store_true", help="one profiled generation (ncu)")
    ap.add_argument("--save-traj", default=None, help="save the greedy trajectory (.npy)")
    ap.add_argument("--load-traj", default=None, help="reuse a saved trajectory (ncu runs)")
    ap.add_argument("--kernel-events", type=int, default=0,
                    help="extra generation with per-kernel CUDA events (diagnostics; breaks PDL overlap)")
    ap.add_argument("--trace", type=int, default=1, help="traced generation for the in-chain roofline (0: off)")
    ap.add_argument("--trace-records", type=int, default=6 << 20)
    ap.add_argument("--split", action="append", default=[],
                    help="split-K override NxK:S for a projection shape of either model (tuning)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.align is None:
        args.align = 0.874 if cfg["temperature"] == 0.0 else -1.0
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    import torch
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2404_15778_b200 as B
    from paper_2404_15778_b200 import _lib as L

    ctx = B.CudaContext(local)
    stream = torch.cuda.Stream(device=local)
    ctx.set_stream(stream.cuda_stream)
    mcfg, dcfg = B.ModelConfig(*cfg["main"]), B.ModelConfig(*cfg["draft"])
    wm = B.DeviceWeights.random(mcfg, seed=1000, dtype=args.dtype, ctx=ctx)
    wd = B.DeviceWeights.random(dcfg, seed=2000, dtype=args.dtype, ctx=ctx)
    gm = {"auto": L.GEMM_AUTO, "simt": L.GEMM_SIMT, "tc": L.GEMM_TC}[args.gemm]
    wm.set_gemm(gm)
    wd.set_gemm(gm)
    for ov in args.split:   # NxK:S — applied to whichever model has that projection shape
        nk, sp = ov.split(":")
        n_, k_ = nk.split("x")
        wm.set_split(int(n_), int(k_), int(sp))
        wd.set_split(int(n_), int(k_), int(sp))
    from paper_2404_15778_b200.shard import gather_tokens, global_sequence_ids, reduce_run
    # sequence-sharded: a rank owns a contiguous range of global sequences;
    # prompts and RNG keys derive from the global id, so outputs are
    # sharding-independent.  c2/c3: batch per GPU (weak scaling); c5: a fixed
    # global batch split over the ranks (strong scaling)
    n_total = cfg.get("global_batch", cfg["batch"] * world)
    scaling = "strong" if "global_batch" in cfg else "weak"
    sids = global_sequence_ids(n_total, world, rank)
    b, P, new = len(sids), cfg["prompt"], cfg["new"]
    ctl_params = B.DraftLengthParams()
    cap = P + new + ctl_params.limit + 8
    main_m = B.CudaModel(wm, b, args.strategy, capacity=cap)
    draft_m = B.CudaModel(wd, b, args.strategy, capacity=cap)
    eng = B.CudaEngine(main_m, draft_m)
    eng.set_strategy(args.strategy)
    eng.set_loop(args.loop)
    prompts = [np.random.default_rng(1_000_003 + sid).integers(0, mcfg.vocab_size, P).tolist()
               for sid in sids]
    req = B.GenerationRequest(prompts, new, temperature=cfg["temperature"], top_p=cfg["top_p"],
                              seed=1234, sequence_ids=sids)

    def reset():
        for m in (main_m, draft_m):
            for s in range(b):
                m.rollback(s, 0)

    # main model's greedy trajectory (regular decoding) -> harness override
    rd = None
    if args.load_traj:      # ncu capture: trajectory from an earlier run of the same config
        align_tokens = np.load(args.load_traj)
    elif args.profile_only:
        align_tokens = np.zeros((b, new), np.int32)
    else:
        reset()
        rd, rd_arr, _ = eng.run(req, None, speculative=False)
        align_tokens = rd_arr["tokens"]
        if cfg["temperature"] > 0.0 and args.align >= 0.0:
            # sampled harness: the draft rows become point masses on keyed
            # override tokens taken from an INDEPENDENT-seed main trajectory,
            # so proposals never depend on the verify draws and speculative
            # sampling stays exact (the output law is the main model's)
            reset()
            req_t = B.GenerationRequest(prompts, new, temperature=cfg["temperature"], top_p=cfg["top_p"],
                                        seed=req.seed + 7919, sequence_ids=sids)
            align_tokens = eng.run(req_t, None, speculative=False)[1]["tokens"]
        if args.save_traj:
            np.save(args.save_traj, align_tokens)

    def generate():
        reset()
        return eng.run(req, B.AdaptiveDraftController(ctl_params), speculative=True,
                       align=args.align, align_seed=99, align_tokens=align_tokens)

    for _ in range(max(args.warmup, 0)):
        generate()
    if args.profile_only:
        generate()
        torch.cuda.synchronize()
        return

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # warm regular-decoding reference point (same engine, same prompts)
    rd_warm = None
    if rd is not None:
        reset()
        rd_warm = eng.run(req, None, speculative=False)[0]

    launches0 = ctx.launches
    h2d0, d2h0 = ctx.transfer_bytes()
    algo0 = ctx.algo_read()
    results = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # pass A (headline): K generations, no instrumentation
    with ClockSampler(local) as clocks:
        barrier()
        t_host0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(generate())
        ev1.record(stream)
        barrier()
        t_host1 = time.perf_counter()
    loop_info = eng.loop_info()
    launches = ctx.launches - launches0
    h2d1, d2h1 = ctx.transfer_bytes()
    algo1 = ctx.algo_read()
    dev_s = ev0.elapsed_time(ev1) / 1e3
    host_s = t_host1 - t_host0
    # pass T (roofline): one more generation with the per-CTA timeline trace
    # on (a globaltimer read at CTA start and one 32-byte record at its end;
    # the PDL chain is untouched).  A kernel class's in-chain time is the
    # union of its CTAs' [start, end] intervals: overlapping launches
    # (the next GEMM's weight prefetch during its predecessor) are counted
    # once, so it can never exceed the generation's device time.
    trace = None
    if args.trace:
        ctx.trace(args.trace_records)
        evt0, evt1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evt0.record(stream)
        generate()
        evt1.record(stream)
        torch.cuda.synchronize()
        trace = trace_summary(ctx.trace_read(args.trace_records))
        trace["generation_ms"] = evt0.elapsed_time(evt1)
        ctx.trace(0)
    # optional pass B: per-launch CUDA events (break PDL overlap; diagnostics only)
    prof = None
    if args.kernel_events:
        ctx.profile(True)
        generate()
        torch.cuda.synchronize()
        prof = ctx.profile_read()
        ctx.profile(False)

    tokens = sum(sum(len(t) for t in r[0].tokens) for r in results)
    if rd is not None and cfg["temperature"] == 0.0:
        assert all(r[0].tokens == rd.tokens for r in results), "greedy speculative != regular"
    if world > 1:
        dev_s, host_s, tokens = reduce_run(torch.distributed, "cuda", dev_s, host_s, tokens)
        gathered = gather_tokens(torch.distributed, world, sids, results[-1][0].tokens)   # final gather
        assert sorted(gathered) == list(range(n_total))
    if rank != 0:
        torch.distributed.destroy_process_group()
        return

    per_tok = []
    for r, arr, raw in results:
        per_tok.append([w / max(len(t), 1) for w, t in zip(r.finish_wall_s, r.tokens)])
    first = statistics.mean(min(p) for p in per_tok) * 1e3
    last = statistics.mean(max(p) for p in per_tok) * 1e3
    allm = statistics.mean(statistics.mean(p) for p in per_tok) * 1e3
    steps_per_gen = statistics.mean(len(r[0].steps) for r in results)
    acc = [x for r in results for s in r[0].steps for x in s.accepted]
    dl = [s.draft_length for r in results for s in r[0].steps]
    tok_per_step = sum(len(t) for t in results[0][0].tokens) / b / len(results[0][0].steps)
    rd_per_tok = (statistics.mean(w / len(t) for w, t in zip(rd_warm.finish_wall_s, rd_warm.tokens)) * 1e3
                  if rd_warm is not None else None)

    hbm, tfl, peak_kind = peaks()
    step_ms = dev_s / args.steps * 1e3
    # algorithmic work per generation (SURVEY 8(d) per-launch formulas, summed
    # over every launch of the timed generations)
    algo = {k: {f: (algo1[k][f] - algo0[k][f]) / args.steps for f in ("launches", "bytes", "flops")}
            for k in algo1}
    all_bytes = sum(v["bytes"] for v in algo.values())

    def roof(cls, tcls, kernel):
        g = algo[cls]
        out = {"bound": "hbm", "kernel": kernel, "peak": hbm, "unit": "GB/s", "peak_kind": peak_kind,
               "bytes_per_generation": g["bytes"], "launches_per_generation": g["launches"]}
        if trace and trace["classes"].get(tcls):
            t = trace["classes"][tcls]
            ach = g["bytes"] / (t["union_ms"] / 1e3) / 1e9
            out.update({"achieved": ach, "frac": ach / hbm, "in_chain_ms_per_generation": t["union_ms"],
                        "share_of_generation": t["union_ms"] / trace["generation_ms"],
                        "median_launch_span_us": t["median_span_us"],
                        "tflops": g["flops"] / (t["union_ms"] / 1e3) / 1e12})
            if t.get("exposed_ms"):
                ex = g["bytes"] / (t["exposed_ms"] / 1e3) / 1e9
                out.update({"exposed_ms_per_generation": t["exposed_ms"], "achieved_exposed": ex,
                            "frac_exposed": ex / hbm})
        return out

    traffic = None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    traffic_src = None
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            traffic, traffic_src = tj.get("dram_bytes_per_launch"), tj.get("shape")
        except Exception:
            traffic = None
    roofline = roof("gemm", "gemm", "gemm_tc_kernel (tcgen05 weight streaming)")
    roofline.update({"traffic": traffic, "traffic_launch": traffic_src,
                     "step_frac": all_bytes / (step_ms / 1e3) / 1e9 / hbm,
                     "method": "achieved = algorithmic GEMM bytes per generation / in-chain GEMM time (union of "
                               "the GEMM CTAs' globaltimer intervals in a traced generation); step_frac = all "
                               "algorithmic bytes per generation / ms_per_step / peak; frac_exposed = bytes / "
                               "the class's critical-path share (each launch owns the part of its span past "
                               "every earlier launch's end; the classes partition the traced timeline)"})
    line = {
        "metric": METRIC,
        "value": tokens / dev_s,
        "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (random-init weights, uniform prompt ids)",
        "config": {"workload": cfg["workload"] + (", INT8 W8A8 (int8 x int8 -> s32 tcgen05 GEMMs; "
                                                  "bf16 attention / KV)" if args.dtype == "int8" else ""),
                   "batch_per_gpu": b, "global_batch": n_total,
                   "prompt_len": P, "max_new_tokens": new, "step": "one full generation",
                   "draft_harness": (f"keyed override, align={args.align}" + (
                                         " (sampled: point-mass draft rows on an independent-seed main "
                                         "trajectory)" if cfg["temperature"] > 0.0 else "") if args.align >= 0
                                     else "natural acceptance (draft samples its own proposals)"),
                   "strategy": args.strategy, "gemm": args.gemm,
                   "l2": "weights (17 GB/replica) >> L2; no flush needed",
                   "parallelism": f"seq-sharded replicas x{world}"},
        "per_seq_ms_per_token": {"first": first, "last": last, "all": allm},
        "regular_decode_ms_per_token": rd_per_tok,
        "tokens_per_step_per_seq": tok_per_step,
        "mean_accepted": statistics.mean(acc) if acc else 0.0,
        "mean_draft_len": statistics.mean(dl) if dl else 0.0,
        "steps_per_generation": steps_per_gen,
        "host_ms_per_generation": {
            "enqueue": statistics.mean(r[2].host_enqueue_s for r in results) * 1e3,
            "sync_wait": statistics.mean(r[2].sync_wait_s for r in results) * 1e3},
        "e2e": {"value": tokens / host_s, "unit": "tokens/s",
                "h2d_bytes_per_step": (h2d1 - h2d0) // max(args.steps, 1),
                "d2h_bytes_per_step": (d2h1 - d2h0) // max(args.steps, 1)},
        "gpu_launches": launches,
        "loop": loop_info,
        "roofline": roofline,
        "attention_roofline": roof("attention", "attn", "attn_stream_kernel (persistent TMA + tcgen05)"),
        "algorithmic_bytes_per_generation": {k: v["bytes"] for k, v in algo.items()},
        "trace": ({"generation_ms": trace["generation_ms"], "untraced_ms": trace["untraced_ms"],
                   "classes": trace["classes"]} if trace else None),
        "kernel_event_ms_per_generation": ({k: v["ms"] for k, v in prof.items()} if prof else None),
        "clocks": clocks.summary(),
    }
    if rank == 0 and args.attn_point:
        line["ragged_attention"] = ragged_attention_point(ctx, hbm)
    if world == 1 and not args.no_cpu_baseline:
        # the GPU run's own per-step draft lengths (first timed generation)
        cb = cpu_reference(cfg, [s_.draft_length for s_ in results[0][0].steps],
                           sum(len(t) for t in results[0][0].tokens) / b, b)
        line["cpu_baseline"] = {k_: cb[k_] for k_ in ("value", "unit", "cores", "kind", "sample")}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
