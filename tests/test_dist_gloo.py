"""Multi-process host logic of the NCCL slab path, run on CPU with gloo
(world_size 2): slab extraction from gmt_slab_layout, reassembly, the
unique-id broadcast pattern and max-over-ranks timing.  The device-side
exchange itself is covered on one GPU by tests/test_gpu_slabs.py
(gmt_create_slabs runs the same partitioned algorithm with device-copy
halos)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import synth
        from paper_2604_26518_b200 import dist as gd
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n, L = 32, 4
        full = synth.tpms(n, "gyroid", 0.3)
        lay = gd.slab_layout(n, L, world, rank)
        assert lay == {"z0": rank * n // world, "nz": n // world, "Ld": 3, "L": 4}, lay
        mine = gd.slab_of(full, L, world, rank)
        assert mine.shape == (n // world, n, n) and mine.flags.c_contiguous
        assert np.array_equal(gd.gather_slabs(mine), full)
        vec = np.arange(6 * 3 * n ** 3, dtype=np.float32).reshape(6, 3, n, n, n)
        assert np.array_equal(gd.gather_slabs(gd.slab_of(vec, L, world, rank)), vec)
        # unique-id broadcast pattern (bytes stand in for ncclGetUniqueId here)
        obj = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(i == ids[0] and len(i) == 128 for i in ids)
        assert gd.max_over_ranks(1.5 + rank) == 1.5 + world - 1
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, f"{e!r}\n{traceback.format_exc()}"))


def test_slab_host_logic_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res


def test_slab_layout_errors_and_geometry():
    from paper_2604_26518_b200 import GmtError, gmt
    assert gmt.gmt_slab_layout(512, 0, 8, 7) == {"z0": 448, "nz": 64, "Ld": 6, "L": 8}
    assert gmt.gmt_slab_layout(64, 5, 1, 0)["Ld"] == 5
    with pytest.raises(GmtError):
        gmt.gmt_slab_layout(16, 3, 4, 0)      # 4 planes per slab: only 2 partitioned levels
    with pytest.raises(GmtError):
        gmt.gmt_slab_layout(30, 2, 4, 0)      # not divisible
    # 12 planes per slab: level 2 would hold 3 planes per slab and the first
    # replicated level 1.5 -- rejected instead of silently leaving planes unwritten
    with pytest.raises(GmtError):
        gmt.gmt_slab_layout(48, 4, 4, 0)
    assert gmt.gmt_slab_layout(48, 4, 2, 1) == {"z0": 24, "nz": 24, "Ld": 3, "L": 4}


def test_gather_level_knob(monkeypatch):
    """GMT_SLAB_MIN_PLANES: levels stay partitioned while a slab keeps that
    many planes (512^3 on 8 ranks: 64, 32, 16, 8 planes -> 4 partitioned
    levels instead of 6); below 3 partitioned levels the default 2 applies."""
    from paper_2604_26518_b200 import gmt
    monkeypatch.setenv("GMT_SLAB_MIN_PLANES", "8")
    assert gmt.gmt_slab_layout(512, 0, 8, 3)["Ld"] == 4
    assert gmt.gmt_slab_layout(256, 0, 8, 3)["Ld"] == 3
    assert gmt.gmt_slab_layout(32, 4, 4, 0)["Ld"] == 3      # falls back to >= 2 planes
    monkeypatch.delenv("GMT_SLAB_MIN_PLANES")
    assert gmt.gmt_slab_layout(512, 0, 8, 3)["Ld"] == 6
