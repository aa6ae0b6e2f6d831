import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2404_15778_b200 as B
from oracle import ragged as OR
for dtype in ("fp32", "bf16"):
    for gemm in (1,):
        g = OR.Geometry(2, 4, 256, 64, 1000, 256)
        dw = B.DeviceWeights.from_reference(OR.init_weights(g, 3), dtype)
        a, b = B.CudaModel(dw, 3), B.CudaModel(dw, 3)
        for m in (a, b):
            m.prefill(0, [1, 2, 3]); m.prefill(1, [4, 5]); m.prefill(2, [9, 9, 9, 9])
        together = a.forward([0, 1, 2], [[7, 8, 9], [11], [3, 4]])
        alone = [b.forward([s], [t])[0] for s, t in ((0, [7, 8, 9]), (1, [11]), (2, [3, 4]))]
        print(dtype, [float(np.abs(x - y).max()) for x, y in zip(together, alone)])
        # repeat determinism
        c = B.CudaModel(dw, 3)
        c.prefill(0, [1, 2, 3]); c.prefill(1, [4, 5]); c.prefill(2, [9, 9, 9, 9])
        t2 = c.forward([0, 1, 2], [[7, 8, 9], [11], [3, 4]])
        print(" repeat", [float(np.abs(x - y).max()) for x, y in zip(together, t2)])
