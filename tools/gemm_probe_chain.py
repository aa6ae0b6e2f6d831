"""Debug build only (-DBASS_GEMM_PROBE): globaltimer stamps of the first 16
CTAs of the last GEMM launch of each projection shape in a C2 speculative
generation (the verify's last layer), in ns relative to the producer's
dependency-wait return (stamp 1).  Stamps: 0 start, 1 producer past
griddepcontrol.wait, 2 first stage ready, 3 last MMA issued, 4 epilogue past
wait, 5 accumulator ready, 6 partial parked, 7 cluster barrier, 8 reduced,
9 stats flushed, 10 final cluster barrier, 11 exit."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2404_15778_b200 as B  # noqa: E402

SHAPES = {"qkv": (13824, 4608), "o": (4608, 4608), "fc": (18432, 4608), "proj": (4608, 18432),
          "d_qkv": (6144, 2048), "d_o": (2048, 2048), "d_fc": (8192, 2048), "d_proj": (2048, 8192)}


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
    req = B.GenerationRequest(prompts, 48, temperature=0.0, seed=1234, sequence_ids=list(range(b)))
    lib = ctx.lib
    lib.bass_gemm_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
    buf = np.zeros(16 * 16, np.uint64)
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(SHAPES)
    for name in names:
        n, k = SHAPES[name]
        for it in range(2):
            for m in (main_m, draft_m):
                for s in range(b):
                    m.rollback(s, 0)
            if it == 1:
                lib.bass_gemm_probe(1, n, k, buf.ctypes.data_as(C.POINTER(C.c_uint64)))
            eng.run(req, B.AdaptiveDraftController(B.DraftLengthParams()), speculative=True)
        lib.bass_gemm_probe(0, n, k, buf.ctypes.data_as(C.POINTER(C.c_uint64)))
        st = buf.reshape(16, 16).astype(np.int64)
        print(f"== {name} N={n} K={k}  (ns from stamp 1; -1 = not reached)")
        ref = st[:, 1][st[:, 1] > 0].min()
        for r in range(16):
            print(f"cta {r:2d}: " + " ".join(f"{(v - ref) if v else -1:7d}" for v in st[r, :12]))


if __name__ == "__main__":
    main()
