"""Multi-rank host logic of bench.py on CPU (gloo, world size 2): max-over-ranks timing
and weak-scaling unit accounting (every rank runs an independent replica)."""
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
