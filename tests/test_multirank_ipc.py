"""One PROCESS per rank with the CUDA-IPC peer transport: W
processes (torch.multiprocessing, gloo for the 64-byte handle all-gather)
each own one slab, build only their rows and exchange halo rows by storing
straight into the peers' IPC windows.  On this box the processes share one
GPU; on an NVLink node the same stores are P2P writes.  Owned atoms' energies
and forces are bitwise equal to the single-handle p = W result, as for the
in-process rank groups (tests/test_gpu_multirank.py)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _system(which):
    from tests import systems as S

    return {"quartz": lambda: S.quartz((4, 4, 4)), "liquid": lambda: S.liquid(1200),
            "slab": lambda: S.quartz((8, 4, 4))}[which]()


def _worker(rank, world, port, which, r3, F, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_02023_b200 import graphmd as G
        s = _system(which)
        prm = G.ToyPotentialParams.init(7, F, 8, 3, 5.0, r3)
        h = G._Handle(0)
        G.init_rank_comm_ipc(h, rank, world, slot_rows=4 * s.size())
        d = G.Distributed.create_distributed(s, 5.0, r3 if r3 > 0 else None, world, 1, True,
                                             handle=h)
        out = G.forward_distributed(d, prm)
        ids = G.owned_ids(d)
        # a second evaluation reuses the windows (exchange epochs > 2)
        out2 = G.forward_distributed(d, prm)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), ids=ids, nint=G.num_interior(d), pa=out.per_atom[ids],
                 f=out.forces[ids], e=out.energy, st=out.stress, pa2=out2.per_atom[ids])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("which,r3,F", [("quartz", 0.0, 16), ("liquid", 3.0, 16), ("slab", 0.0, 16),
                                        ("slab", 3.0, 16), ("slab", 3.0, 64)])
def test_ipc_rank_processes_equal_single_handle(tmp_path, world, which, r3, F):
    """("slab": thick slabs with interior atoms, whose layer updates run
    between the send and the receive kernel of each exchange.)"""
    from paper_2506_02023_b200 import graphmd as G

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.environ["PYTHONPATH"] = root + os.pathsep + os.environ.get("PYTHONPATH", "")
    mp.start_processes(_worker, args=(world, _free_port(), which, r3, F, str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    s = _system(which)
    prm = G.ToyPotentialParams.init(7, F, 8, 3, 5.0, r3)
    ref = G.forward_distributed(
        G.Distributed.create_distributed(s, 5.0, r3 if r3 > 0 else None, world, 1, True), prm)
    seen = np.zeros(s.size(), bool)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        ids = z["ids"]
        assert not seen[ids].any()
        seen[ids] = True
        if which == "slab":
            assert 0 < int(z["nint"]) < len(ids)
        np.testing.assert_array_equal(z["pa"], ref.per_atom[ids])
        np.testing.assert_array_equal(z["pa2"], ref.per_atom[ids])
        np.testing.assert_array_equal(z["f"], ref.forces[ids])
        assert abs(float(z["e"]) - ref.energy) <= 1e-9 * abs(ref.energy)
        np.testing.assert_allclose(z["st"], ref.stress, atol=1e-12, rtol=1e-9)
    assert seen.all()
