"""Golden BASSCKPT file + logits, written by the REFERENCE package itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ckpt.py

tiny.ckpt: ref save_checkpoint(init_model(ModelConfig(1, 2, 32, 16, 50, 64), 3))
ckpt.json: the reference's prefill logits of that model for one prompt.
"""

import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from batchspec import checkpoint as CK   # noqa: E402
from batchspec import model as M         # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

cfg = M.ModelConfig(n_layer=1, n_head=2, d_model=32, d_head=16, vocab_size=50, max_seq_len=64)
w = M.init_model(cfg, 3)
CK.save_checkpoint(w, os.path.join(OUT, "tiny.ckpt"))
back = CK.load_checkpoint(os.path.join(OUT, "tiny.ckpt"), cfg)
prompt = [1, 7, 3, 49, 0, 12]
main = M.MainModel(back, 1)
logits = main.prefill(0, prompt)
with open(os.path.join(OUT, "ckpt.json"), "w") as fh:
    json.dump({"config": [1, 2, 32, 16, 50, 64], "seed": 3, "prompt": prompt,
               "prefill_logits": [float(x) for x in logits]}, fh)
print("wrote tiny.ckpt, ckpt.json")
