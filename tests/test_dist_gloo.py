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


def _halo_worker(rank, world, port, q, lo, hi):
    """Run gmt_halo_schedule's list with gloo isend/irecv on CPU buffers (the
    NCCL transport issues the same list in one group) and check every ghost
    plane against the neighbour part's boundary plane."""
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2604_26518_b200 import gmt
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        nz, ncomp, plane = 5, 3, 12
        gl, gh = 2, 2                                   # allocated ghost planes per side
        cstride = (gl + nz + gh) * plane
        base = gl * plane                               # view base: plane 0 of component 0
        buf = torch.full((ncomp * cstride,), -1.0, dtype=torch.float64)

        def value(owner, c, z, i):                      # global plane owner * nz + z
            return 1e6 * owner + 1e4 * c + 100 * z + i

        for c in range(ncomp):
            for z in range(nz):
                s0 = base + c * cstride + z * plane
                buf[s0:s0 + plane] = torch.tensor([value(rank, c, z, i) for i in range(plane)],
                                                  dtype=torch.float64)
        ops = gmt.gmt_halo_schedule(world, rank, nz, ncomp, cstride, plane, lo, hi)
        assert len(ops) == 2 * ncomp * (lo + hi), ops
        reqs = []
        for peer, snd, off, cnt in ops:
            view = buf[base + off:base + off + cnt]     # contiguous plane slices of buf
            reqs.append(dist.isend(view.clone(), dst=peer) if snd else None)
            if not snd:
                recv = torch.empty(cnt, dtype=torch.float64)
                reqs[-1] = (dist.irecv(recv, src=peer), view, recv)
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                r[1].copy_(r[2])
            else:
                r.wait()
        dn, up = (rank - 1) % world, (rank + 1) % world
        for c in range(ncomp):
            for g in range(1, lo + 1):                  # lower ghosts = lower part's top planes
                s0 = base + c * cstride - g * plane
                want = [value(dn, c, nz - g, i) for i in range(plane)]
                assert buf[s0:s0 + plane].tolist() == want, ("lo", c, g)
            for g in range(hi):                         # upper ghosts = upper part's bottom planes
                s0 = base + c * cstride + (nz + g) * plane
                want = [value(up, c, g, i) for i in range(plane)]
                assert buf[s0:s0 + plane].tolist() == want, ("hi", c, g)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, f"{e!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("world,lo,hi", [(2, 1, 1), (3, 1, 1), (2, 1, 0), (3, 0, 1), (2, 2, 2)])
def test_halo_schedule_gloo(world, lo, hi):
    """The slab halo schedule (gmt_halo_schedule: the list the NCCL transport
    issues) executed by `world` processes over gloo: sends and receives pair up
    in issue order and every ghost plane ends with the neighbour part's
    boundary plane (periodic ring; world 2 has the same part below and above)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, q, lo, hi)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(60)
    assert res == {r: "ok" for r in range(world)}, res
