"""Host-side logic of the checkpoint container (ref:checkpoint.py) and the
run configuration of the report layer (ref:bench.py:47-149) — CPU only.

The golden file tests/golden/tiny.ckpt was written by the reference's own
`save_checkpoint` (tests/golden/make_golden_ckpt.py)."""

import json
import os
import struct

import numpy as np
import pytest

from oracle import ragged as OR
from paper_2404_15778_b200 import checkpoint as CK
from paper_2404_15778_b200 import report as R
from paper_2404_15778_b200.model import ModelConfig

CFG = ModelConfig(1, 2, 32, 16, 50, 64)


@pytest.fixture
def golden(golden_dir):
    return os.path.join(golden_dir, "tiny.ckpt")


def test_golden_file_parses_to_reference_init(golden):
    w = OR.init_weights(OR.Geometry(1, 2, 32, 16, 50, 64), 3)
    arrays = {name: np.array(a) for name, a, _, _ in CK.iter_checkpoint(golden, CFG)}
    assert list(arrays) == list(CK.manifest(CFG))
    assert np.array_equal(arrays["token_embedding"], w["tok_emb"].astype(np.float32))
    assert np.array_equal(arrays["layer0.w_fc"], w["layers"][0]["w_fc"].astype(np.float32))
    assert np.array_equal(arrays["output_head"], w["head"].astype(np.float32))
    assert np.array_equal(arrays["layer0.ffn_norm.gain"], np.ones(32, np.float32))


def test_save_matches_reference_bytes(golden, tmp_path):
    w = OR.init_weights(OR.Geometry(1, 2, 32, 16, 50, 64), 3)
    out = tmp_path / "x.ckpt"
    CK.save_checkpoint(w, out)
    assert out.read_bytes() == open(golden, "rb").read()


def _rewrite(golden, tmp_path, edit):
    raw = bytearray(open(golden, "rb").read())
    edit(raw)
    p = tmp_path / "bad.ckpt"
    p.write_bytes(bytes(raw))
    return p


def test_error_contracts(golden, tmp_path):
    """ref tests/test_checkpoint.py:49-86 (same error classes / texts)."""
    def magic(raw):
        raw[0:8] = b"NOTACKPT"

    def version(raw):
        raw[8:12] = struct.pack("<I", 2)

    def tag(raw):   # first array's dtype tag: after magic, header, name, rank, dims
        nlen = struct.unpack("<I", raw[16:20])[0]
        off = 20 + nlen + 4 + 8
        raw[off:off + 4] = struct.pack("<I", 7)

    with pytest.raises(CK.CheckpointError, match="magic"):
        list(CK.iter_checkpoint(_rewrite(golden, tmp_path, magic), CFG))
    with pytest.raises(CK.CheckpointError, match="version"):
        list(CK.iter_checkpoint(_rewrite(golden, tmp_path, version), CFG))
    with pytest.raises(CK.CheckpointError, match="dtype tag"):
        list(CK.iter_checkpoint(_rewrite(golden, tmp_path, tag), CFG))
    with pytest.raises(CK.CheckpointError, match="truncated"):
        list(CK.iter_checkpoint(_rewrite(golden, tmp_path, lambda r: r.__delitem__(slice(-100, None))), CFG))
    with pytest.raises(CK.CheckpointError, match="shape|missing|unexpected"):
        list(CK.iter_checkpoint(golden, ModelConfig(1, 2, 32, 16, 51, 64)))
    with pytest.raises(CK.CheckpointError, match="unexpected|missing"):
        list(CK.iter_checkpoint(golden, ModelConfig(2, 2, 32, 16, 50, 64)))
    empty = tmp_path / "empty.ckpt"
    empty.write_bytes(b"")
    with pytest.raises(CK.CheckpointError, match="truncated"):
        list(CK.iter_checkpoint(empty, CFG))
    assert issubclass(CK.CheckpointError, ValueError)


TINY_MAIN = {"n_layer": 2, "n_head": 4, "d_model": 64, "vocab_size": 96, "max_seq_len": 256}


def tiny_config(**over):
    base = {"seed": 1234, "batch_size": 2, "max_new_tokens": 12, "temperature": 0.7, "top_p": 0.9,
            "main": dict(TINY_MAIN), "draft": {"alignment": 0.8}, "prompt_len": 5}
    base.update(over)
    return R.RunConfig.from_dict(base)


def test_run_config_validation():
    """ref tests/test_bench.py:36-78."""
    with pytest.raises(R.ConfigError):
        tiny_config(draft={})
    with pytest.raises(R.ConfigError):
        tiny_config(draft={"alignment": 0.5, "checkpoint": "x"})
    with pytest.raises(R.ConfigError):
        tiny_config(fixed_draft=4, draft_params={"l0": 3})
    with pytest.raises(R.ConfigError):
        tiny_config(draft={"alignment": 1.5})
    with pytest.raises(R.ConfigError):
        tiny_config(main={"n_layer": 2, "bogus": 1}).main_config()
    with pytest.raises(R.ConfigError):
        tiny_config(quant_enabled=True, dtype="fp32")
    assert tiny_config(quant_enabled=True).device_dtype == "int8"


def test_run_config_file_round_trip_and_prompts(tmp_path):
    p = tmp_path / "run.json"
    p.write_text(json.dumps({"strategy": "split", "fixed_draft": 6, "draft": {"alignment": 0.5},
                             "main": dict(TINY_MAIN)}))
    conf = R.RunConfig.from_file(p)
    assert conf.strategy.value == "split" and conf.fixed_draft == 6
    assert R.make_controller(conf).length == 6
    assert tiny_config().resolve_prompts() == [[41, 71, 42, 0, 78], [62, 24, 43, 42, 76]]
    shared = tiny_config(batch_size=3, shared_prompt=True).resolve_prompts()
    assert shared[0] == shared[1] == shared[2]


def test_roofline_clock_orders_first_all_last():
    """The roofline-priced clock of a synthetic step trace (no GPU)."""
    from types import SimpleNamespace as NS
    steps = [NS(slots=(0, 1), draft_length=3, emitted=((1, 2, 3, 4), (5,)), finished=(False, False)),
             NS(slots=(0, 1), draft_length=3, emitted=((6,), (7, 8, 9, 10)), finished=(True, False)),
             NS(slots=(1,), draft_length=2, emitted=((11, 12),), finished=(True,))]
    res = NS(prompts=[[1] * 8, [2] * 8], tokens=[[0] * 5, [0] * 7], steps=steps)
    cfg = ModelConfig(2, 4, 64, 16, 96, 256)
    sim = R.simulate_from_trace(res, cfg, cfg, 2, hbm_gbs=1000.0)
    assert 0 < sim.finish_time_s[0] < sim.finish_time_s[1]
    assert sim.first_latency <= sim.all_latency <= sim.last_latency
