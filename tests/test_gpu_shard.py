"""Sequence sharding on the device path (BASELINE configs[4]):
two processes on one GPU, each with its own libbass context, model replica
and controller, decode their halves of 64 global sequences; the final gather
(paper_2404_15778_b200.shard over torch.distributed, gloo) must equal the
one-process b = 64 run token for token — greedy and sampled
(ref tests/test_acceptance.py:130-151: outputs are independent of the batch
composition and of the draft-length schedule)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_TOTAL, NEW = 64, 20


def _models():
    import paper_2404_15778_b200 as B
    from oracle import ragged as OR
    wm = B.DeviceWeights.from_reference(OR.init_weights(OR.Geometry(2, 4, 512, 128, 1000, 256), 31), "bf16")
    wd = B.DeviceWeights.from_reference(OR.init_weights(OR.Geometry(1, 4, 512, 128, 1000, 256), 32), "bf16")
    return B, wm, wd


def _decode(sids, temperature):
    B, wm, wd = _models()
    prompts = [np.random.default_rng(1_000_003 + s).integers(0, 1000, 6 + s % 11).tolist() for s in sids]
    req = B.GenerationRequest(prompts, NEW, temperature=temperature, top_p=0.9, seed=5, sequence_ids=list(sids))
    res = B.decode_speculative(B.CudaModel(wm, len(sids)), B.CudaModel(wd, len(sids)), req,
                               B.AdaptiveDraftController())
    return res.tokens


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2404_15778_b200.shard import gather_tokens, global_sequence_ids
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sids = global_sequence_ids(N_TOTAL, world, rank)
    out = {}
    for temp in (0.0, 0.8):
        out[temp] = gather_tokens(dist, world, sids, _decode(sids, temp))
    if rank == 0:
        q.put(out)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_process_shards_gather_to_the_single_process_run():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for temp in (0.0, 0.8):
        whole = _decode(list(range(N_TOTAL)), temp)
        assert sorted(gathered[temp]) == list(range(N_TOTAL))
        assert [gathered[temp][s] for s in range(N_TOTAL)] == whole, temp
