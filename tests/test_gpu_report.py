"""Device-side checkpoint loading (ref:checkpoint.py:91-143) and the report
layer (ref:bench.py:214-424) end to end on the GPU, mirroring the reference's
tests/test_checkpoint.py and tests/test_bench.py."""

import json
import os

import numpy as np
import pytest

from oracle import ragged as OR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2404_15778_b200 as B
    return B


def _bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    u = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return u.view(np.float32)


def test_checkpoint_to_device_matches_reference_logits(B, golden_dir, tmp_path):
    from paper_2404_15778_b200 import checkpoint as CK
    from paper_2404_15778_b200 import _lib as L
    meta = json.load(open(os.path.join(golden_dir, "ckpt.json")))
    cfg = B.ModelConfig(*meta["config"])
    path = os.path.join(golden_dir, "tiny.ckpt")
    dw = CK.load_checkpoint(path, cfg, "fp32")
    got = B.CudaModel(dw, 1).prefill(0, meta["prompt"])
    want = np.asarray(meta["prefill_logits"])
    assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
    # read-back is bit-exact (fp32) and saving reproduces the reference's bytes
    for name, arr, tid, layer in CK.iter_checkpoint(path, cfg):
        assert np.array_equal(dw.get(tid, layer), arr), name
    CK.save_checkpoint(dw, tmp_path / "back.ckpt")
    assert (tmp_path / "back.ckpt").read_bytes() == open(path, "rb").read()
    # bf16 models store the RNE-rounded values
    db = CK.load_checkpoint(path, cfg, "bf16")
    w = OR.init_weights(OR.Geometry(*meta["config"]), meta["seed"])
    assert np.array_equal(db.get(L.W_WQ, 0), _bf16(w["layers"][0]["wq"]))
    assert np.array_equal(db.get(L.W_HEAD, 0), _bf16(w["head"]))


def test_init_model_is_the_reference_init(B):
    from paper_2404_15778_b200 import _lib as L
    g = OR.Geometry(2, 4, 64, 16, 96, 256)
    w = OR.init_weights(g, 1234)
    dw = B.DeviceWeights.init_model(B.ModelConfig(2, 4, 64, 16, 96, 256), 1234, "fp32")
    assert np.array_equal(dw.get(L.W_TOK_EMB), w["tok_emb"].astype(np.float32))
    assert np.array_equal(dw.get(L.W_PROJ, 1), w["layers"][1]["w_proj"].astype(np.float32))
    assert np.array_equal(dw.get(L.W_HEAD), w["head"].astype(np.float32))


TINY_MAIN = {"n_layer": 2, "n_head": 4, "d_model": 64, "vocab_size": 96, "max_seq_len": 256}


def tiny_config(**over):
    from paper_2404_15778_b200 import report as R
    base = {"seed": 1234, "batch_size": 2, "max_new_tokens": 12, "temperature": 0.7, "top_p": 0.9,
            "main": dict(TINY_MAIN), "draft": {"alignment": 0.8}, "prompt_len": 5, "dtype": "fp32"}
    base.update(over)
    return R.RunConfig.from_dict(base)


def test_golden_tokens_for_pinned_seed(B):
    """ref tests/test_bench.py:142-154: the same tokens on the device (fp32)."""
    from paper_2404_15778_b200 import report as R
    conf = tiny_config()
    weights = R.build_main_weights(conf)
    req = B.GenerationRequest(prompts=conf.resolve_prompts(), max_new_tokens=12, temperature=0.7, top_p=0.9,
                              seed=1234)
    base = B.decode_regular(B.CudaModel(weights, 2), req)
    assert base.tokens == [[38, 32, 87, 74, 67, 27, 25, 29, 14, 19, 1, 62],
                           [76, 95, 58, 30, 94, 4, 73, 41, 86, 32, 41, 19]]


def test_report_schema_and_ordering(B, tmp_path):
    """ref tests/test_bench.py:92-140."""
    from paper_2404_15778_b200 import report as R
    report = R.run_generate(tiny_config(batch_size=4, out_dir=str(tmp_path / "a")))
    for key in ("schema_version", "baseline", "speculative", "acceptance_rate", "tokens_per_main_invocation",
                "speedup_simulated_all", "speedup_measured_all"):
        assert key in report
    for blk in (report["baseline"], report["speculative"]):
        for key in ("measured_first_s", "measured_last_s", "measured_all_s", "simulated_first_s",
                    "simulated_last_s", "simulated_all_s"):
            assert isinstance(blk[key], float)
        assert blk["measured_first_s"] <= blk["measured_all_s"] <= blk["measured_last_s"]
        assert blk["simulated_first_s"] <= blk["simulated_all_s"] <= blk["simulated_last_s"]
    seq = [r for r in report["records"] if r["record"] == "sequence"]
    assert len(seq) == 2 * 4
    spec = [r for r in seq if r["run"] == "speculative"]
    assert report["speculative"]["measured_all_s"] == pytest.approx(
        np.mean([r["measured_finish_s"] / r["tokens_generated"] for r in spec]))
    lines = (tmp_path / "a" / "report.jsonl").read_text().splitlines()
    assert json.loads(lines[0])["record"] == "summary" and len(lines) == 1 + 8
    R.run_generate(tiny_config(batch_size=4, out_dir=str(tmp_path / "b")))
    assert (tmp_path / "a" / "generations.jsonl").read_bytes() == (tmp_path / "b" / "generations.jsonl").read_bytes()


def test_greedy_run_reports_exact_match(B):
    from paper_2404_15778_b200 import report as R
    for dtype in ("fp32", "bf16"):
        report = R.run_generate(tiny_config(temperature=0.0, draft={"alignment": 1.0}, dtype=dtype), write=False)
        assert report["greedy_exact_match"] is True
        assert report["acceptance_rate"] == 1.0


def test_quality_under_budget(B, tmp_path):
    """ref tests/test_bench.py:164-205."""
    from paper_2404_15778_b200 import report as R
    conf = tiny_config(batch_size=2)
    weights = R.build_main_weights(conf)
    rng = np.random.default_rng(7)
    tasks = []
    for i in range(3):
        prompt = rng.integers(0, 96, 4).tolist()
        req = B.GenerationRequest(prompts=[prompt], max_new_tokens=6, temperature=0.0)
        greedy = B.decode_regular(B.CudaModel(weights, 1), req).tokens[0]
        tasks.append({"id": f"t{i}", "prompt": prompt, "max_new_tokens": 6, "accepted": [greedy]})
    path = tmp_path / "tasks.json"
    path.write_text(json.dumps({"tasks": [dict(t, accept_any=True) for t in tasks]}))
    rep = R.run_quality(conf, path, write=False)
    assert rep["pass_at_first"] == 1.0 and rep["pass_at_finished"] == 1.0
    path.write_text(json.dumps({"tasks": tasks}))
    rep = R.run_quality(tiny_config(batch_size=4, temperature=0.4), path, write=False)
    assert rep["pass_at_first"] <= rep["pass_at_finished"]
    rep = R.run_quality(tiny_config(batch_size=2, time_budget_s=0.0), path, write=False)
    assert rep["pass_at_first"] == rep["pass_at_finished"] == 0.0   # nothing finishes in zero time


def test_cli_generate_writes_report(B, tmp_path):
    from paper_2404_15778_b200 import cli
    cfgp = tmp_path / "run.json"
    cfgp.write_text(json.dumps({"main": TINY_MAIN, "batch_size": 2, "max_new_tokens": 8, "prompt_len": 4,
                                "temperature": 0.0, "draft": {"alignment": 0.9}}))
    assert cli.main(["generate", "--config", str(cfgp), "--out", str(tmp_path / "o"), "--dtype", "fp32"]) == 0
    rec = json.loads((tmp_path / "o" / "report.jsonl").read_text().splitlines()[0])
    assert rec["greedy_exact_match"] is True


def test_quant_enabled_run_is_the_int8_path(B):
    """ref:bench.py:85, 162-173 (`quant_enabled`): both providers on the INT8
    W8A8 path; greedy speculative == greedy regular in the report."""
    from paper_2404_15778_b200 import report as R
    main = dict(TINY_MAIN, d_model=128, vocab_size=256)
    conf = tiny_config(temperature=0.0, draft={"alignment": 1.0}, dtype="bf16", quant_enabled=True, main=main)
    assert conf.device_dtype == "int8"
    report = R.run_generate(conf, write=False)
    assert report["greedy_exact_match"] is True
    assert report["quant_enabled"] is True and report["dtype"] == "int8"
