"""Per-CTA detail of a traced C2 generation (the records `tools/trace_gen.py
out.npy` saves: {start_ns, end_ns, smid, class | launch_seq << 4} per CTA).

For one draft token in the middle of the generation (located by its LM head,
the GEMM launch with one CTA per 128-row vocabulary tile) and one main-model
verify layer (located by its attention launch, one CTA per SM), prints each
launch's CTA start / end spread in microseconds from a common origin, the
number of SMs it used and how many CTAs each SM ran — the view behind the
DESIGN §9 table (which kernel's CTAs start before their predecessor ends,
i.e. prefetch under PDL, and which wait for free SMs).

    python tools/trace_gen.py /tmp/t.npy && python tools/cta_detail.py /tmp/t.npy
"""
import sys

import numpy as np

GEMM, ATTN = 1, 2
HEAD_TILES = (50272 + 127) // 128   # C2 vocabulary / 128-row weight tiles
SMS = 148


def launches(path):
    rec = np.load(path)
    rec = rec[rec[:, 0] > 0]
    rec = rec[((rec[:, 3] & 15) != 13) & ((rec[:, 3] >> 62) == 0)]
    seq = rec[:, 3] >> 4
    o = np.argsort(seq, kind="stable")
    rec, seq = rec[o], seq[o]
    return np.split(rec, np.flatnonzero(np.diff(seq)) + 1)


def row(tag, r, base):
    st, en = (r[:, 0] - base) / 1e3, (r[:, 1] - base) / 1e3
    per_sm = np.bincount(np.bincount(r[:, 2], minlength=SMS))
    print(f"{tag:+3d} cls={r[0, 3] & 15} grid={len(r):4d} sms={len(np.unique(r[:, 2])):3d}  "
          f"start {st.min():7.1f} {np.median(st):7.1f} {st.max():7.1f}  "
          f"end {en.min():7.1f} {np.median(en):7.1f} {en.max():7.1f}  "
          f"dur med {np.median(en - st):6.1f}  CTAs/SM hist {per_sm.tolist()}")


def main():
    L = launches(sys.argv[1])
    cls = [int(r[0, 3] & 15) for r in L]
    heads = [i for i, r in enumerate(L) if cls[i] == GEMM and len(r) == HEAD_TILES]
    if heads:
        h = heads[len(heads) // 2]
        base = L[max(0, h - 9)][:, 0].min()
        print("draft token around its LM head (us): launch, grid, SMs, start[min,med,max], end[min,med,max]")
        for j in range(max(0, h - 9), min(len(L), h + 8)):
            row(j - h, L[j], base)
    atts = [i for i, r in enumerate(L) if cls[i] == ATTN and len(r) == SMS]
    if atts:
        a = atts[len(atts) // 2]
        base = L[a][:, 0].min()
        print("\nmain verify layer from its attention (us)")
        for j in range(max(0, a - 1), min(len(L), a + 7)):
            row(j - a, L[j], base)


if __name__ == "__main__":
    main()
