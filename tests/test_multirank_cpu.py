"""N>1 host protocol on CPU with torch.distributed/gloo, world_size 2:
the 128-byte NCCL-id broadcast used by graphmd.init_rank_comm, and the
exchange-plan invariant every rank relies on (its FROM_r[j] span receives
exactly rank j's TO_j[r] rows), computed per rank from the partition
structure of that rank's slab (the C oracle stands in for the GPU build)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Oracle
        from paper_2506_02023_b200 import graphmd as G
        from tests import systems as S

        uid = bytes(range(128)) if rank == 0 else None
        got = G.broadcast_bytes(uid, 0)
        s = S.quartz((4, 3, 3))
        d = Oracle("c").create(*S.as_args(s), 4.0, p=world, allow_narrow=True)
        mk = d.layout(rank)["markers"]
        scnt = [int(mk[2 + j] - mk[1 + j]) for j in range(world)]
        rcnt = [int(mk[2 + world + j] - mk[1 + world + j]) for j in range(world)]
        import torch
        allt = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allt, torch.tensor(scnt, dtype=torch.int64))
        ok = G.exchange_plan_consistent(scnt, rcnt, rank, [t.tolist() for t in allt])
        q.put((rank, got == bytes(range(128)), ok, sum(rcnt)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_protocol():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), "uid broadcast mismatch"
    assert all(r[2] for r in res), "exchange plans inconsistent"
    assert all(r[3] > 0 for r in res), "no halo rows"

