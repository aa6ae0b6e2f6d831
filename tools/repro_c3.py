"""Small C3-shaped repro (sampled, draft d_head=64) for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_15778_b200 as B
main = tuple(int(x) for x in os.environ.get("MAIN", "2,5,640,128,50272,512").split(","))
draft = tuple(int(x) for x in os.environ.get("DRAFT", "2,12,768,64,50272,512").split(","))
ctx = B.CudaContext.default()
wm = B.DeviceWeights.random(B.ModelConfig(*main), seed=1, ctx=ctx)
wd = B.DeviceWeights.random(B.ModelConfig(*draft), seed=2, ctx=ctx)
b = 8
mm, dm = B.CudaModel(wm, b, "ragged", capacity=300), B.CudaModel(wd, b, "ragged", capacity=300)
eng = B.CudaEngine(mm, dm)
prompts = [np.random.default_rng(i).integers(0, 50272, int(os.environ.get("PROMPT", "64"))).tolist() for i in range(b)]
req = B.GenerationRequest(prompts, int(os.environ.get("NEW", "24")), temperature=0.2, top_p=0.95, seed=1234, sequence_ids=list(range(b)))
res, _, _ = eng.run(req, B.AdaptiveDraftController(B.DraftLengthParams()), speculative=True)
print("ok", [len(t) for t in res.tokens])
