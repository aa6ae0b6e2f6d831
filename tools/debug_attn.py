import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2404_15778_b200 as B
from oracle import ragged as OR
ctx = B.CudaContext.default()
z = np.load("tests/golden/attention.npz")
for c in (1, 3, 4):
    offs = z[f"c{c}_off"].tolist()
    n = len(offs)
    qs = [z[f"c{c}_{i}_q"] for i in range(n)]; ks = [z[f"c{c}_{i}_k"] for i in range(n)]; vs = [z[f"c{c}_{i}_v"] for i in range(n)]
    H, dh = qs[0].shape[0], qs[0].shape[2]
    stride = max(k.shape[1] for k in ks)
    K = np.zeros((n, H, stride, dh)); V = np.zeros_like(K)
    for i in range(n):
        K[i, :, :ks[i].shape[1]] = ks[i]; V[i, :, :vs[i].shape[1]] = vs[i]
    Q = np.concatenate([q.transpose(1, 0, 2) for q in qs], 0)
    cu = np.concatenate([[0], np.cumsum([q.shape[1] for q in qs])])
    d = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda")
    out = B.attend_device(ctx, d(Q), d(K), d(V), cu, offs, "ragged").cpu().numpy()
    for i in range(n):
        want = z[f"c{c}_{i}_pad"].transpose(1, 0, 2)
        got = out[cu[i]:cu[i+1]]
        err = np.abs(got - want).max(axis=2)
        print("case", c, "seq", i, "off", offs[i], "q", qs[i].shape[1], "H", H, "dh", dh)
        print(np.array2string(err, precision=2))
        # is got equal to attention with a different layout guess?
        alt = OR.attend_split([Q[cu[i]:cu[i+1]].reshape(-1, H, dh).transpose(1,0,2)], [ks[i]], [vs[i]], [offs[i]])[0].transpose(1,0,2)
        print(" alt err", np.abs(got - alt).max())
