"""Multi-process (gloo, world size 2, CPU) checks of the sequence-sharding host
logic used by bench.py under torchrun: disjoint covering shards, global
sequence ids, max/sum reductions and the final token gather."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2404_15778_b200.shard import global_sequence_ids, shard_range


def test_shards_partition_the_batch():
    for n in (1, 7, 8, 64, 65):
        for world in (1, 2, 4, 8):
            seen = []
            for r in range(world):
                a, b = shard_range(n, world, r)
                assert 0 <= a <= b <= n
                seen.extend(range(a, b))
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2404_15778_b200.shard import gather_tokens, reduce_run
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sids = global_sequence_ids(64, world, rank)
    toks = [[sid, sid + 1] for sid in sids]   # stand-in generations
    dev, host, n = reduce_run(dist, "cpu", 1.0 + rank, 2.0 + rank, sum(len(t) for t in toks))
    merged = gather_tokens(dist, world, sids, toks)
    q.put((rank, dev, host, n, sorted(merged)))
    dist.destroy_process_group()


def test_gloo_world2_reductions_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, dev, host, n, keys in res:
        assert dev == 2.0 and host == 3.0          # max over ranks
        assert n == 128                            # sum over ranks (64 seqs x 2 tokens)
        assert keys == list(range(64))             # every global sequence gathered
