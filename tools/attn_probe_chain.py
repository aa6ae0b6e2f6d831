"""Debug build only (-DBASS_ATTN_PROBE): pipeline stamps of the LAST attention
launch of a C2 speculative generation (the verify's last layer), relative
to each CTA's start, in ns.  Columns as in attn_stream.cu's APROBE ids."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_15778_b200 as B  # noqa: E402


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
    req = B.GenerationRequest(prompts, new // 2, temperature=0.0, seed=1234, sequence_ids=list(range(b)))
    lib = ctx.lib
    lib.bass_attn_probe.argtypes = [C.c_int, C.POINTER(C.c_uint64)]
    buf = np.zeros(16 * 32, np.uint64)
    for it in range(2):
        for m in (main_m, draft_m):
            for s in range(b):
                m.rollback(s, 0)
        if it == 1:
            lib.bass_attn_probe(1, buf.ctypes.data_as(C.POINTER(C.c_uint64)))
        eng.run(req, B.AdaptiveDraftController(B.DraftLengthParams()), speculative=True)
    lib.bass_attn_probe(0, buf.ctypes.data_as(C.POINTER(C.c_uint64)))
    st = buf.reshape(16, 32).astype(np.int64)
    for r in range(16):
        rel = [(st[r, i] - st[r, 0]) / 1.965 if st[r, i] else -1 for i in range(1, 27)]
        print(f"cta {r:2d}: " + " ".join(f"{v:6.0f}" for v in rel))


if __name__ == "__main__":
    main()
