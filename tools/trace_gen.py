"""Per-CTA timeline of one C2 speculative generation (bass_trace_enable):
every GEMM / attention / LayerNorm CTA records {start, end, SM} with the
globaltimer.  Prints per-class totals, the launch-to-launch gaps (negative =
overlap via PDL) and one main-model layer's timeline.

    python tools/trace_gen.py [out.npy]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_15778_b200 as B  # noqa: E402

CLS = {1: "gemm", 2: "attn", 3: "norm", 4: "combine", 5: "mega"}


def main():
    cfg = bench.CONFIGS["c2"]
    ctx = B.CudaContext(0)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    wm = B.DeviceWeights.random(B.ModelConfig(*cfg["main"]), seed=1000, ctx=ctx)
    wd = B.DeviceWeights.random(B.ModelConfig(*cfg["draft"]), seed=2000, ctx=ctx)
    b, P, new = cfg["batch"], cfg["prompt"], cfg["new"]
    cap = P + new + 40
    main_m, draft_m = B.CudaModel(wm, b, "ragged", capacity=cap), B.CudaModel(wd, b, "ragged", capacity=cap)
    eng = B.CudaEngine(main_m, draft_m)
    prompts = [np.random.default_rng(1_000_003 + i).integers(0, 50272, P).tolist() for i in range(b)]
    req = B.GenerationRequest(prompts, new, temperature=0.0, seed=1234, sequence_ids=list(range(b)))

    def reset():
        for m in (main_m, draft_m):
            for s in range(b):
                m.rollback(s, 0)

    reset()
    _, rd_arr, _ = eng.run(req, None, speculative=False)
    for it in range(2):
        reset()
        if it == 1:
            ctx.check(ctx.lib.bass_trace_enable(ctx.handle, 8 << 20))
        res = eng.run(req, B.AdaptiveDraftController(B.DraftLengthParams()), speculative=True, align=0.874,
                      align_seed=99, align_tokens=rd_arr["tokens"])
    buf = np.zeros((8 << 20) * 4, np.uint64)
    n = C.c_int64()
    ctx.check(ctx.lib.bass_trace_read(ctx.handle, buf.ctypes.data_as(C.POINTER(C.c_uint64)), 8 << 20, C.byref(n)))
    ctx.check(ctx.lib.bass_trace_enable(ctx.handle, 0))
    rec = buf[: 4 * n.value].reshape(-1, 4).astype(np.int64)
    if len(sys.argv) > 1:
        np.save(sys.argv[1], rec)
    analyse(rec)


def analyse_mega(rec, t0):
    """Per-phase view of the layer megakernels: producer X-ready, epilogue done,
    barrier release (us from the launch's first CTA start)."""
    tag = rec[:, 3]
    kern = rec[(tag & 15) == 5]
    second = (tag >> 62) & 1
    ph = rec[((tag & 15) == 13) & (second == 0)]
    ph2 = rec[((tag & 15) == 13) & (second == 1)]
    p2seq = (ph2[:, 3] >> 4) & ((1 << 36) - 1)
    if not len(kern):
        return
    kseq = kern[:, 3] >> 4
    pseq = (ph[:, 3] >> 4) & ((1 << 36) - 1)
    pidx = ph[:, 3] >> 40
    seqs = np.unique(kseq)
    rows = []
    for sq in seqs:
        k = kern[kseq == sq]
        s0 = k[:, 0].min()
        P = ph[pseq == sq]
        P2 = ph2[p2seq == sq]
        phases = []
        for p in np.unique(P[:, 3] >> 40):
            r = P[(P[:, 3] >> 40) == p]
            r2 = P2[((P2[:, 3] >> 40) & 0x3fffff) == p]
            rdy = r[:, 2][r[:, 2] > 0]
            wt = r2[:, 0][r2[:, 0] > 0] if len(r2) else np.array([])
            phases.append(((r[:, 0].min() - s0) / 1e3, (r[:, 0].max() - s0) / 1e3, (r[:, 1].max() - s0) / 1e3,
                           ((rdy.min() - s0) / 1e3) if len(rdy) else -1, ((rdy.max() - s0) / 1e3) if len(rdy) else -1,
                           ((wt.min() - s0) / 1e3) if len(wt) else -1, ((wt.max() - s0) / 1e3) if len(wt) else -1))
        rows.append(((k[:, 0].max() - s0) / 1e3, (k[:, 1].max() - s0) / 1e3, phases))
    by = {}
    for r in rows:
        by.setdefault(len(r[2]), []).append(r)
    for n, rs in sorted(by.items()):
        print(f"\nmega launches with {n} phases: {len(rs)}; median span {np.median([r[1] for r in rs]):.1f} us")
        mid = rs[len(rs) // 2]
        print(f"  example: CTA starts spread {mid[0]:.1f} us, end {mid[1]:.1f} us")
        for i, (d0, d1, rel, r0, r1, w0, w1) in enumerate(mid[2]):
            print(f"  phase {i}: prod-wait {w0:7.1f}..{w1:7.1f}  x-ready {r0:7.1f}..{r1:7.1f}  "
                  f"done {d0:7.1f}..{d1:7.1f}  released {rel:7.1f}")


def analyse(rec):
    rec = rec[rec[:, 0] > 0]
    analyse_mega(rec, rec[:, 0].min())
    rec = rec[(rec[:, 3] & 15) != 13]
    rec = rec[(rec[:, 3] >> 62) == 0]
    t0 = rec[:, 0].min()
    seq = rec[:, 3] >> 4
    order = np.argsort(seq, kind="stable")
    rec, seq = rec[order], seq[order]
    bounds = np.flatnonzero(np.diff(seq)) + 1
    launches = []
    for r in np.split(rec, bounds):
        launches.append(dict(cls=CLS.get(int(r[0, 3] & 15), "?"), grid=len(r), s0=(r[:, 0].min() - t0) / 1e3,
                             s1=(r[:, 0].max() - t0) / 1e3, e0=(r[:, 1].min() - t0) / 1e3,
                             e1=(r[:, 1].max() - t0) / 1e3, sms=len(np.unique(r[:, 2])),
                             maxper=int(np.bincount(r[:, 2]).max())))
    if os.environ.get("TRACE_CSV"):
        with open(os.environ["TRACE_CSV"], "w") as fh:
            fh.write("cls,grid,s0,s1,e0,e1,sms,maxper\n")
            for l in launches:
                fh.write(f"{l['cls']},{l['grid']},{l['s0']:.2f},{l['s1']:.2f},{l['e0']:.2f},{l['e1']:.2f},{l['sms']},{l['maxper']}\n")
    total = launches[-1]["e1"] - launches[0]["s0"]
    print(f"launches {len(launches)}  span {total / 1e3:.2f} ms")
    by = {}
    for i, l in enumerate(launches):
        d = by.setdefault(l["cls"], [0, 0.0, 0.0, 0.0])
        d[0] += 1
        d[1] += l["e1"] - l["s0"]                      # launch span
        d[2] += l["e1"] - l["s1"]                      # from last CTA start to last end
        if i + 1 < len(launches):
            d[3] += launches[i + 1]["s0"] - l["e1"]    # gap to next launch (negative = overlap)
    for k, (cnt, span, tail, gap) in by.items():
        print(f"{k:8s} n={cnt:6d} span={span / 1e3:8.2f} ms  avg={span / cnt:7.2f} us  avg_gap_after={gap / cnt:6.2f} us")
    # layer periods: attention launches of the main (largest grid) and draft models
    att = [l for l in launches if l["cls"] == "attn"]
    if not att:
        return
    gmax = max(l["grid"] for l in att)
    for name, sel in (("main", [l for l in att if l["grid"] == gmax]), ("draft", [l for l in att if l["grid"] != gmax])):
        d = np.diff([l["s0"] for l in sel])
        d = d[d < 200]   # consecutive layers of one forward
        if len(d):
            print(f"{name} layer period: median {np.median(d):.1f} us  (n={len(d)})")
    # a main-model layer in the middle
    mid = next(i for i in range(len(launches) // 2, len(launches)) if launches[i]["cls"] == "attn" and launches[i]["grid"] == gmax)
    print("\ntimeline around the middle (us, relative):")
    base = launches[mid]["s0"]
    for l in launches[mid: mid + 24]:
        print(f"{l['cls']:8s} grid={l['grid']:4d} sms={l['sms']:3d} max/SM={l['maxper']}  start {l['s0'] - base:8.2f}..{l['s1'] - base:8.2f}"
              f"  end {l['e0'] - base:8.2f}..{l['e1'] - base:8.2f}  span {l['e1'] - l['s0']:7.2f}")
    # a draft-model token in the middle (its attention launches have the smaller grid)
    dmid = next((i for i in range(len(launches) // 2, len(launches))
                 if launches[i]["cls"] == "attn" and launches[i]["grid"] != gmax), None)
    if dmid is not None:
        print("\ndraft timeline (us, relative):")
        base = launches[dmid]["s0"]
        for l in launches[dmid: dmid + 22]:
            print(f"{l['cls']:8s} grid={l['grid']:4d} sms={l['sms']:3d} max/SM={l['maxper']}  start {l['s0'] - base:8.2f}..{l['s1'] - base:8.2f}"
                  f"  end {l['e0'] - base:8.2f}..{l['e1'] - base:8.2f}  span {l['e1'] - l['s0']:7.2f}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--load":
        analyse(np.load(sys.argv[2]))
    else:
        main()
