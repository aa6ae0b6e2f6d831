"""CPU oracle for the BASS hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithm that the
B200 build replaces (`/root/reference/pkg/src/batchspec/*.py`, cited per
function as ``ref:<file>:<line>``).  It exists to *check* the CUDA path:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2404_15778_b200`` never imports it and never
  falls back to it.

Parity pinning: every module here is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the reference package
read-only in the build container (``tests/test_oracle_golden.py``).  The
reference is pure Python, so the vectors are outputs of the reference itself,
not of this restatement.
"""

from .control import AlgParams, alg1_update, AdaptiveLength, FixedLength
from .rng import seedseq_state, pcg64_uniforms, keyed_uniforms
from .sampling import (shape_probs, inverse_cdf, accept_or_resample,
                       KeyedStreams)
from .ragged import (Geometry, init_weights, RaggedCache, forward_ragged,
                     attend_pad, attend_split, layer_norm, gelu_erf)
from .engine import (Request, OracleModel, OracleAlignedDraft,
                     run_regular, run_speculative)

__all__ = [n for n in dir() if not n.startswith("_")]
