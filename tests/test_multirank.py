"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): max-over-ranks timing,
weak-scaling unit accounting (replicas), and the sharded mode's rebase / merge of the
parts' CSRs (paper_2212_07679_b200/shard.py)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    w, r, lr = bench.dist_env()
    assert (w, r, lr) == (world, rank, rank)
    t = bench.max_over_ranks(10.0 + rank, world)          # each rank's own timing
    units = bench.weak_units(1000, world)
    dist.barrier()
    out[rank] = (t, units)
    dist.destroy_process_group()


def test_gloo_world2_max_and_weak_units():
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1] == (11.0, 2000)


def test_reference_arm_only_rank0_prints(monkeypatch, capsys):
    import bench
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")

    class A:
        config, steps, warmup, gpus = "c1", 1, 3, 2
    bench.run_reference(A())
    assert capsys.readouterr().out == ""


def _shard_worker(rank, world, port, out):
    """Each rank holds the rows of one part (disjoint row sets of one query set, as
    snn_query_*_part returns them: a CSR over all m rows, other parts' rows empty)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import numpy as np
    import oracle
    from paper_2212_07679_b200 import shard
    rng = np.random.default_rng(7)
    X = rng.random((3000, 2)).astype(np.float32)
    full = oracle.radius_query(X, X, 0.03, band_rel=0.0)
    off = torch.from_numpy(full["offsets"])
    ids = torch.from_numpy(full["indices"].astype(np.int32))
    m = len(off) - 1
    owner = torch.from_numpy(rng.integers(0, world, m))          # any disjoint row split
    counts = (off[1:] - off[:-1]) * (owner == rank)
    loff = torch.zeros(m + 1, dtype=torch.int64)
    torch.cumsum(counts, 0, out=loff[1:])
    lids = torch.zeros(int(loff[-1]), dtype=torch.int32)
    keep = torch.repeat_interleave(owner == rank, off[1:] - off[:-1])
    lids[:] = ids[keep]
    base, total, sizes = shard.part_bases(int(loff[-1]))
    goff = shard.global_offsets(loff.clone())
    gids = torch.full((total,), -1, dtype=torch.int32)
    shard.scatter_rows(loff, lids, goff, gids)
    # merge: every rank contributes its rows; -1 marks slots another rank fills
    gathered = [torch.zeros_like(gids) for _ in range(world)]
    dist.all_gather(gathered, gids)
    res = torch.stack(gathered).max(dim=0).values
    out[rank] = (base, total, sizes, bool(torch.equal(goff, off)), bool(torch.equal(res, ids)))
    dist.destroy_process_group()


def test_gloo_world2_shard_rebase_and_merge():
    """bench.py's sharded mode on 2 ranks: the all-gather of per-part nnz gives each part's
    base entry (rank order), the all-reduce of row counts gives the global offsets, and the
    parts' rows placed at those offsets reproduce the full CSR exactly."""
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_shard_worker, args=(2, port, out), nprocs=2, join=True)
    b0, t0, s0, ok_off0, ok_ids0 = out[0]
    b1, t1, s1, ok_off1, ok_ids1 = out[1]
    assert s0 == s1 and t0 == t1 == sum(s0)
    assert b0 == 0 and b1 == s0[0]
    assert ok_off0 and ok_off1 and ok_ids0 and ok_ids1
