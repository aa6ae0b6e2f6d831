"""CPU-side checks of the C ABI boundary: the in-tree libbass.so loads, exports
every symbol include/bass.h declares, and the Python mirror validates the
reference's error contracts before touching the device."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bass.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(bass_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("bass_ctx_create", "bass_model_create", "bass_kv_create", "bass_kv_truncate",
                 "bass_forward_ragged", "bass_attention", "bass_accept", "bass_spec_generate",
                 "bass_regular_generate", "bass_rng_uniforms"):
        assert need in syms


def test_library_loads_and_exports_every_symbol():
    from paper_2404_15778_b200 import _lib
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    assert L.bass_version() == 1


def test_library_is_sm100a():
    import subprocess
    from paper_2404_15778_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_request_validation_matches_reference_messages():
    from paper_2404_15778_b200 import GenerationRequest
    with pytest.raises(ValueError):
        GenerationRequest(prompts=[], max_new_tokens=4)
    with pytest.raises(ValueError):
        GenerationRequest(prompts=[[]], max_new_tokens=4)
    with pytest.raises(ValueError):
        GenerationRequest(prompts=[[1]], max_new_tokens=0)
    with pytest.raises(ValueError):
        GenerationRequest(prompts=[[1], [2]], max_new_tokens=2, sequence_ids=[0])
    r = GenerationRequest(prompts=[[1], [2]], max_new_tokens=2)
    assert r.sequence_ids == [0, 1] and r.batch_size == 2


def test_model_config_validation():
    from paper_2404_15778_b200 import ModelConfig
    with pytest.raises(ValueError):
        ModelConfig(1, 3, 8, 2, 16, 32)
    with pytest.raises(ValueError):
        ModelConfig(1, 2, 8, 3, 16, 32)
    with pytest.raises(ValueError):
        ModelConfig(0, 2, 8, 4, 16, 32)


def test_controllers_follow_algorithm1():
    import oracle
    from paper_2404_15778_b200 import (AdaptiveDraftController, DraftLengthParams,
                                       FixedDraftController, init_state, update)
    import numpy as np
    rng = np.random.default_rng(5)
    st = init_state()
    l, s = 7, 0
    for _ in range(1000):
        acc = [int(rng.integers(0, st.l_draft + 1)) for _ in range(int(rng.integers(1, 9)))]
        st = update(st, acc)
        l, s = oracle.alg1_update(l, s, acc, oracle.AlgParams())
        assert (st.l_draft, st.s) == (l, s)
    c = AdaptiveDraftController()
    c.observe([7, 3])
    assert c.length == 9 and c.max_length == 32
    f = FixedDraftController(6)
    f.observe([6])
    assert f.length == 6 == f.max_length
    with pytest.raises(ValueError):
        DraftLengthParams(l0=0)
    with pytest.raises(ValueError):
        FixedDraftController(0)
