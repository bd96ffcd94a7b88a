"""bench.py -- GMG V-cycle throughput of libgmt on B200 (driver contract).

Metric (BASELINE.json "512^3 elasticity GMG V-cycles/s & DOF/s at 1/2/4/8
B200; % HBM roofline"), reported as throughput of the homogenisation step in
active DOF-load-cases per second: one step = one pass of the whole hot path
 on the 512^3 gyroid TPMS (configs[4]'s problem, which
fits one B200; configs[1] 64^3 is a parity case):
    Galerkin coarse-operator build from the (device-resident) material
  + the given initial guess (Alg. 2 line 1)
  + one V-cycle (damped-Jacobi smoothing, residual, restriction,
    prolongation, coarse levels, coarsest solve) for all 6 load cases
  + C^H reduction (App. F1) read back to the host.
value = DPN * (active nodes) * NRHS / step time.  V-cycles/s (= steps/s) and
the V-cycle time on its own are separate keys.  Both arms print the same
metric, unit and config; the reference arm is the FP64 oracle (there is no
reference implementation to install) timed on the host cores on a bounded
sample of the same workload (the 64^3 cell of the same generator, whose
throughput in the same unit it reports); our arm adds a like-for-like GPU
line at that sample size.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--res 512] [--physics elastic]
  python bench.py --impl reference ...   (the FP64 oracle on host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the batch-screening graph runs one branch per lattice: let more of them run
# concurrently than the default 8 hardware work queues (set before CUDA init)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

SCREEN_TOL = 1e-4   # Sec. 5.2: "a target r <= 1e-4 is used as an engineering-grade stability threshold"
SAMPLE_N = 64   # the reference arm's bounded sample: configs[1]'s size (~10 s of oracle work per step)


def physics_dims(physics: str):
    return (3, 6) if physics == "elastic" else (1, 3)   # (DPN, NRHS)


def metric_name(args) -> str:
    return (f"{args.res}^3 {args.physics} GMG homogenisation throughput: active DOF x load case x V-cycle "
            f"per second (step = Galerkin build + 1 V-cycle + C^H)")


def workload_config(args) -> dict:
    dpn, nr = physics_dims(args.physics)
    return {"workload": f"{args.res}^3 {args.physics} {args.geometry} v_f={args.vf}, {nr} load cases, "
                        f"one V-cycle from a given initial guess + C^H",
            "smoother": "damped Jacobi (2 pre, 2 post, 16 coarsest sweeps)",
            "l2": "inputs larger than L2 (level-0 vectors 9.7 GB at 512^3)"}


# --------------------------------------------------------------------------- activity model

def level_activity(s: np.ndarray, levels: int):
    """Per level l: (n_l, active nodes, interface nodes) of the homogeneity
    pyramid: level-l elements carry the common scale of their
    2^l x 2^l x 2^l voxels (or -1 if mixed); a node is active if one of its 8
    incident elements is non-void and an interface node if they differ."""
    out = []
    e = s.astype(np.float32)
    for l in range(levels):
        n = e.shape[0]
        if l > 0:
            v = e.reshape(n // 2, 2, n // 2, 2, n // 2, 2).transpose(0, 2, 4, 1, 3, 5).reshape(n // 2, n // 2, n // 2, 8)
            same = np.all(v == v[..., :1], axis=-1)
            e = np.where(same, v[..., 0], np.float32(-1))
            n //= 2
        # node (z, y, x) has incident elements (z-1..z, y-1..y, x-1..x)
        nz_any = np.zeros(e.shape, bool)
        mixed = e < 0
        for dz in (0, 1):
            for dy in (0, 1):
                for dx in (0, 1):
                    r = np.roll(e, shift=(dz, dy, dx), axis=(0, 1, 2))
                    nz_any |= r != 0
                    mixed |= (r != e) | (r < 0)
        out.append((n, int(nz_any.sum()), int((nz_any & mixed).sum())))
    return out


def vcycle_bytes(act, dpn: int, nr: int, pre=2, post=2, coarse=16) -> tuple[float, float]:
    """Algorithmic HBM bytes of one V-cycle, every level:
    per active node and sweep read u, write u (4V each), read f (levels >= 1,
    4V) and the node code (4 B); interface nodes of coarse levels also read
    their 27-point stencil (27 DPN^2 x 4 B); the residual pass as a sweep;
    restriction reads the fine residual and writes the coarse rhs; the coarse
    error is zeroed; prolongation reads the coarse error and updates the fine
    solution.  Returns (total, level-0 share)."""
    V = 4 * dpn * nr
    L = len(act)
    tot = 0.0
    lvl0 = 0.0
    for l, (n, A, I) in enumerate(act):
        f_read = V if l > 0 else 0
        sweep = (2 * V + f_read + 4) * A + (27 * dpn * dpn * 4 * I if l > 0 else 0)
        if l == L - 1:
            b = coarse * sweep
        else:
            A1 = act[l + 1][1]
            b = (pre + post + 1) * sweep                      # smoothing + residual
            b += V * A + V * A1                               # restriction
            b += V * A1                                       # zero coarse error
            b += V * A1 + 2 * V * A + 4 * A                   # prolongation + correction
        tot += b
        if l == 0:
            lvl0 = b
    return tot, lvl0


def active_nodes(s: np.ndarray, z0: int = 0, nz: int | None = None) -> int:
    """Nodes of planes [z0, z0+nz) touching at least one non-void voxel."""
    n = s.shape[0]
    nz = n - z0 if nz is None else nz
    occ = np.take(s != 0, np.arange(z0 - 1, z0 + nz) % n, axis=0)
    act = np.zeros((nz, n, n), dtype=bool)
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                act |= np.roll(occ, shift=(dy, dx), axis=(1, 2))[1 - dz:1 - dz + nz]
    return int(act.sum())


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--res", type=int, default=512)
    ap.add_argument("--physics", choices=["elastic", "thermal"], default="elastic")
    ap.add_argument("--geometry", default="gyroid")
    ap.add_argument("--vf", type=float, default=0.3)
    ap.add_argument("--levels", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l0-kernel", type=int, default=0, choices=[0, 1],
                    help="level-0 sweep: 0 CUDA-core sum-factorised stencil (k_l0), 1 tcgen05 element contractions")
    ap.add_argument("--no-like", action="store_true", help="skip the like-for-like GPU line at the sample size")
    ap.add_argument("--no-batch", action="store_true", help="skip the configs[2] batch-screening line")
    ap.add_argument("--batch-count", type=int, default=64)
    ap.add_argument("--batch-res", type=int, default=128)
    ap.add_argument("--breakdown", action="store_true", help="extra pass with per-class event timing")
    ap.add_argument("--no-solve", action="store_true", help="skip the (untimed) full solve to 1e-5")
    return ap.parse_args()


def make_material(geometry: str, n: int, vf: float):
    import synth
    if geometry == "gyroid":
        return synth.tpms(n, "gyroid", vf)
    if geometry == "gyroid_sheet":
        return synth.tpms(n, "gyroid", vf, sheet=True)
    if geometry == "truss":
        return synth.truss(n, "octet", 0.05)
    if geometry == "stochastic":
        return synth.stochastic(n, vf, seed=0)
    if geometry == "solid":
        return synth.solid(n)
    raise ValueError(geometry)


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(args, world: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the roofline
    kernel from the committed `ncu --set full` capture (profiles/r2/traffic.json),
    when it was taken on this exact single-GPU workload; else None."""
    p = os.path.join(ROOT, "profiles", "r2", "traffic.json")
    if world != 1 or not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    same = (d.get("res") == args.res and d.get("physics") == args.physics and d.get("geometry") == args.geometry
            and abs(float(d.get("vf", -1)) - args.vf) < 1e-9 and args.levels in (0, 8))
    return (float(d["dram_bytes_per_launch"]), d["source"]) if same else (None, None)


# --------------------------------------------------------------------------- oracle leg

def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        return max([int(d.get("num_threads", 1)) for d in threadpool_info()] or [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_step(physics: str, geometry: str, n: int, vf: float):
    """One step of the workload run by the FP64 oracle at resolution n (same
    generator and settings): assembly + Galerkin hierarchy, one V-cycle from
    zero, C^H.  Returns (seconds, active DOF-load-cases)."""
    from oracle import fem, gmg
    s = make_material(geometry, n, vf)
    ph = fem.Physics(physics)
    om = 0.45 if physics == "elastic" else 0.6
    L = gmg.default_levels(n)
    t0 = time.perf_counter()
    H = gmg.Hierarchy(s, ph, L)
    u = gmg.vcycle(H, np.zeros_like(H.f), omega=om, pre=2, post=2, coarse=16)
    fem.effective_tensor(s, ph, u)
    dt = time.perf_counter() - t0
    return dt, int(H.active[0].sum()) * ph.nrhs


def sample_desc(args, n, L_note=""):
    return (f"{n}^3 cell of the same workload ({args.geometry}, v_f={args.vf}, {args.physics}): "
            f"assembly + Galerkin hierarchy + 1 V-cycle + C^H by the FP64 oracle (scipy.sparse kernels "
            f"single-threaded, numpy BLAS on {blas_threads()} threads){L_note}")


def cpu_baseline(args, reps: int = 1):
    ts, dofs = [], 0
    for _ in range(reps):
        dt, dofs = oracle_step(args.physics, args.geometry, SAMPLE_N, args.vf)
        ts.append(dt)
    dt = float(np.mean(ts))
    return {"value": dofs / dt, "unit": "DOF/s", "cores": blas_threads(), "kind": "oracle",
            "sample": sample_desc(args, SAMPLE_N) + f"; {dt:.2f} s per step, mean of {reps}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    for _ in range(args.warmup):
        oracle_step(args.physics, args.geometry, SAMPLE_N, args.vf)
    ts, dofs = [], 0
    for _ in range(args.steps):
        dt, dofs = oracle_step(args.physics, args.geometry, SAMPLE_N, args.vf)
        ts.append(dt)
    ms = float(np.mean(ts)) * 1e3
    val = dofs / (ms * 1e-3)
    out = {"impl": "reference", "metric": metric_name(args), "value": val, "unit": "DOF/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(args), "sample_res": SAMPLE_N,
           "cpu_baseline": {"value": val, "unit": "DOF/s", "cores": blas_threads(), "kind": "oracle",
                            "sample": sample_desc(args, SAMPLE_N) + f"; {ms:.0f} ms per step"},
           "e2e": {"value": val, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# --------------------------------------------------------------------------- our leg

def maybe_spawn(args):
    """--gpus N without a torchrun environment: re-launch as N ranks."""
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)


def time_steps(fn, steps, stream, sync):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
    sync()
    return e0.elapsed_time(e1) / steps


def like_for_like(args, steps: int, warmup: int):
    """The same step on the GPU at the reference arm's sample size."""
    import torch
    from paper_2604_26518_b200 import Problem
    s = make_material(args.geometry, SAMPLE_N, args.vf)
    dpn, nr = physics_dims(args.physics)
    import synth
    u0 = torch.from_numpy(synth.initial_guess(SAMPLE_N, nr, dpn, seed=1, material=s)).cuda()
    s_dev = torch.from_numpy(np.ascontiguousarray(s)).cuda()
    with Problem(s_dev, physics=args.physics, levels=0) as P:
        st = torch.cuda.ExternalStream(P.stream)

        def step():
            P.gmt_set_material(s_dev)
            P.gmt_set_initial_guess(u0)
            P.gmt_vcycle(1)
            return P.gmt_homogenize()

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        ms = time_steps(step, steps, st, torch.cuda.synchronize)
    dofs = dpn * active_nodes(s) * nr
    return {"res": SAMPLE_N, "value": dofs / (ms * 1e-3), "unit": "DOF/s", "ms_per_step": ms,
            "note": "same step on the GPU at the reference arm's sample size"}


def batch_screening(args):
    """BASELINE configs[2]: high-throughput screening of a batch of 128^3
    truss / shell lattices (Sec. 7.1, App. C) on one GPU through gmt_batch_*:
    every V-cycle of the whole batch is one CUDA-graph launch.
      * cycle: one V-cycle of all lattices (graph) -> lattice V-cycles/s and
        DOF/s in the main metric's unit;
      * screening: new materials for all lattices (Galerkin builds), zero
        guess, batch V-cycles until every load case of every lattice reaches
        Sec. 5.2's engineering-grade r <= 1e-4 (residuals checked every 2
        cycles), C^H of all -> lattices/s."""
    import torch

    import synth
    from paper_2604_26518_b200 import Batch, Problem
    n, cnt = args.batch_res, args.batch_count
    mats = synth.batch_truss_psl(n, cnt, seed=0)
    dpn, nr = physics_dims("elastic")
    devs = [torch.from_numpy(np.ascontiguousarray(m)).cuda() for m in mats]
    probs = [Problem(d, physics="elastic") for d in devs]
    dofs = sum(dpn * active_nodes(m) * nr for m in mats)
    out = {"workload": f"{cnt} x {n}^3 elastic truss / shell lattices (synth.batch_truss_psl, seed 0), 6 load cases",
           "lattices": cnt}
    try:
        with Batch(probs) as bt:
            st = torch.cuda.ExternalStream(probs[0].stream)
            for _ in range(3):
                bt.gmt_batch_vcycle(1)
            torch.cuda.synchronize()
            reps = max(args.steps, 5)
            ms = time_steps(lambda: bt.gmt_batch_vcycle(1), reps, st, torch.cuda.synchronize)
            out["cycle"] = {"ms": ms, "lattice_vcycles_per_s": cnt * 1e3 / ms, "dof_per_s": dofs / (ms * 1e-3),
                            "unit_note": "DOF/s = active DOF x load case x V-cycle per second (main metric's unit)"}

            def screen():
                for P, d in zip(probs, devs):
                    P.gmt_set_material(d)
                    P.gmt_set_initial_guess(None)
                cyc = 0
                while cyc < 200:
                    bt.gmt_batch_vcycle(2)
                    cyc += 2
                    if bt.gmt_batch_residual_norms().max() <= SCREEN_TOL:
                        break
                return cyc, bt.gmt_batch_homogenize(), bt.gmt_batch_residual_norms().max()

            screen()                                      # warm-up (graph capture)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            cyc, CH, worst = screen()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            out["screening"] = {"s": dt, "lattices_per_s": cnt / dt, "cycles": cyc, "rel_tol": SCREEN_TOL,
                                "worst_final_rel": float(worst),
                                "C_H11_range": [float(CH[:, 0, 0].min()), float(CH[:, 0, 0].max())],
                                "note": "wall clock: Galerkin builds of all lattices + batched V-cycles to r <= 1e-4 "
                                        "(residual checks every 2 cycles) + batched C^H"}
    finally:
        for P in probs:
            P.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    maybe_spawn(args)
    import torch

    import synth
    from paper_2604_26518_b200 import Problem, build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = world > 1
    # multi-GPU: agglomerate coarse levels once a slab would hold < 8 planes
    os.environ.setdefault("GMT_SLAB_MIN_PLANES", "8")
    if dist:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    build.build()

    s = make_material(args.geometry, args.res, args.vf)
    n = args.res
    dpn, nr = physics_dims(args.physics)
    if dist:
        # one z-slab per rank (gmt_create_dist): halos by ncclSend/Recv,
        # replicated coarse levels by ncclAllGather, dot products by ncclAllReduce
        from paper_2604_26518_b200 import dist as gd
        lay = gd.slab_layout(n, args.levels, world, rank)
        z0, nz = lay["z0"], lay["nz"]
        nid = gd.share_unique_id()
    else:
        z0, nz = 0, n
    s_loc = np.ascontiguousarray(s[z0:z0 + nz])
    s_dev = torch.from_numpy(s_loc).cuda()
    u0 = synth.initial_guess(n, nr, dpn, seed=1, material=s, z0=z0, nz=nz)
    u0_dev = torch.from_numpy(u0).cuda()
    del u0
    if dist:
        P = Problem(s_dev, physics=args.physics, levels=args.levels, device=local, dist=(rank, world, nid))
    else:
        P = Problem(s_dev, physics=args.physics, levels=args.levels, device=local)
    P.gmt_set_level0_kernel(args.l0_kernel)
    P.gmt_profile_enable(1)   # bracket the dominant kernel (level-0 Jacobi sweep) live
    st = torch.cuda.ExternalStream(P.stream)

    def step():
        P.gmt_set_material(s_dev)           # Galerkin coarse-operator build
        P.gmt_set_initial_guess(u0_dev)     # Alg. 2 line 1 (given initial guess)
        P.gmt_vcycle(1)                     # one V-cycle, all load cases
        return P.gmt_homogenize()           # C^H -> host (synchronises)

    for _ in range(args.warmup):
        step()
    P.gmt_profile_collect()
    P.gmt_profile_read(0, reset=True)

    clocks = Clocks(local)
    if dist:
        td.barrier()
    torch.cuda.synchronize()
    launches0 = P.gmt_kernel_launches()
    clocks.start()
    out_CH = [None]

    def timed_step():
        out_CH[0] = step()
        P.gmt_profile_collect()

    ms = time_steps(timed_step, args.steps, st, torch.cuda.synchronize)
    clk = clocks.stop()
    CH = out_CH[0]
    if dist:
        td.barrier()
    launches = P.gmt_kernel_launches() - launches0
    if dist:
        ms = gd.max_over_ranks(ms, device="cuda")
    k_ms, k_cnt = P.gmt_profile_read(0)
    rel, _, _ = P.gmt_residual_norms()

    # the V-cycle alone (same state as a step: material built, guess set)
    P.gmt_set_material(s_dev)
    P.gmt_set_initial_guess(u0_dev)
    P.gmt_vcycle(1)
    torch.cuda.synchronize()
    if dist:
        td.barrier()
    vc_ms = time_steps(lambda: P.gmt_vcycle(1), args.steps, st, torch.cuda.synchronize)
    if dist:
        vc_ms = gd.max_over_ranks(vc_ms, device="cuda")

    # ---- e2e through the public API with host buffers: the u8 occupancy and
    # the given initial guess on the active nodes (compact layout, Sec. 4.1.1)
    # come from pinned host memory every step, C^H goes back to the host.
    binary = bool(np.all((s_loc == 0) | (s_loc == 1)))
    s_host = torch.from_numpy((s_loc > 0).astype(np.uint8) if binary else s_loc).pin_memory().numpy()
    e2e = None
    if not dist:
        P.gmt_set_material(s_dev)
        P.gmt_set_initial_guess(u0_dev)
        uc_host = torch.from_numpy(P.gmt_get_solution_compact()).pin_memory().numpy()

        def e2e_step():
            P.gmt_set_material(s_host)
            P.gmt_set_initial_guess_compact(uc_host)
            P.gmt_vcycle(1)
            return P.gmt_homogenize()

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e = {"ms_per_step": e2e_ms, "h2d": int(s_host.nbytes + uc_host.nbytes)}
        del uc_host

    # north star's second half: full GMG solve to 1e-5 relative residual from
    # a zero initial guess (informational, outside the timed steps)
    solve = None
    if not args.no_solve:
        P.gmt_set_material(s_dev)
        P.gmt_set_initial_guess(None)
        P.gmt_solve(1e-5, 200)            # warm-up: allocates the refinement buffers
        P.gmt_set_initial_guess(None)
        if dist:
            td.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        k, fr, hist = P.gmt_solve(1e-5, 200)
        CHs = P.gmt_homogenize()
        torch.cuda.synchronize()
        t_solve = (time.perf_counter() - t0) * 1e3
        if dist:
            t_solve = gd.max_over_ranks(t_solve, device="cuda")
        solve = {"rel_tol": 1e-5, "cycles": int(k), "final_rel": float(fr), "ms": t_solve,
                 "refinement": bool(P.gmt_refinement_active()) if not dist else False,
                 "C_H_diag": [float(CHs[i, i]) for i in range(nr)],
                 "note": "zero initial guess; residual norms every cycle; wall clock incl. the final C^H; "
                         "second solve (the first allocates the refinement buffers)"}

    breakdown = None
    if args.breakdown:
        P.gmt_profile_enable(0xFF)
        for _ in range(2):
            step(); P.gmt_profile_collect()
        P.gmt_profile_enable(0xFF)
        reps = 3
        for _ in range(reps):
            step(); P.gmt_profile_collect()
        breakdown = {}
        for c, name in enumerate(Problem.PROFILE_CLASSES):
            t, cnt = P.gmt_profile_read(c)
            breakdown[name] = {"ms_per_step": t / reps, "launches_per_step": cnt / reps}

    levels = P.levels
    P.close()
    n_act = active_nodes(s, z0, nz)
    bytes_launch = (2 * 4 * dpn * nr + 4) * n_act      # level-0 sweep: read u, write u, node code
    avg_ms = k_ms / max(k_cnt, 1)
    if dist:   # aggregate over ranks: all bytes / slowest rank's launch
        tb = torch.tensor([float(bytes_launch), float(n_act), float(launches)], dtype=torch.float64, device="cuda")
        td.all_reduce(tb)
        bytes_launch, n_act, launches = float(tb[0]), int(tb[1]), int(tb[2])
        avg_ms = gd.max_over_ranks(avg_ms, device="cuda")
        k_ms = gd.max_over_ranks(k_ms, device="cuda")
        td.destroy_process_group()
    if rank != 0:
        return

    hbm, hbm_src = measured_peaks()
    hbm_agg = hbm * world
    achieved = bytes_launch / (avg_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args, world)
    act = level_activity(s, levels)
    vb, vb0 = vcycle_bytes(act, dpn, nr)
    dofs = dpn * n_act * nr
    value = dofs / (ms * 1e-3)
    out = {
        "metric": metric_name(args),
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**workload_config(args), "levels": levels,
                   "parallelism": f"slab{world} (z-slabs, NCCL halos)" if dist else "single GPU"},
        "vcycles_per_s": 1e3 / ms, "vcycle_ms": vc_ms, "active_nodes": n_act, "active_dof_x_cases": dofs,
        "roofline": {"bound": "hbm",
                     "kernel": "level-0 damped-Jacobi sweep (" + ("k_l0_tc, tcgen05" if args.l0_kernel else "k_l0") + ")",
                     "achieved": achieved, "peak": hbm_agg, "unit": "GB/s", "frac": achieved / hbm_agg,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": hbm_src,
                     "bytes_per_launch": bytes_launch,
                     "bytes_rule": f"(2 x 4 x {dpn * nr} + 4) B x active nodes (read u, write u, node code)",
                     "avg_launch_ms": avg_ms, "launches_timed": k_cnt, "share_of_step": k_ms / args.steps / ms},
        "roofline_vcycle": {"bound": "hbm", "achieved": vb / (vc_ms * 1e-3) / 1e9, "peak": hbm_agg, "unit": "GB/s",
                            "frac": vb / (vc_ms * 1e-3) / 1e9 / hbm_agg, "bytes_per_vcycle": vb,
                            "level0_bytes": vb0, "vcycle_ms": vc_ms,
                            "levels": [{"n": a[0], "active": a[1], "interface": a[2]} for a in act],
                            "rule": "bench.vcycle_bytes (DESIGN.md Sec. 8(d))"},
        "clocks": clk,
        "gpu_launches": int(launches),
        "residual_after_cycle": float(np.max(rel)),
        "solve": solve,
        "C_H_diag": [float(CH[i, i]) for i in range(nr)],
    }
    if e2e:
        out["e2e"] = {"value": dofs / (e2e["ms_per_step"] * 1e-3), "unit": "DOF/s", "ms_per_step": e2e["ms_per_step"],
                      "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": nr * nr * 8,
                      "note": "pinned host u8 occupancy (gmt_set_material) + pinned host initial guess on the "
                              "active nodes (gmt_set_initial_guess_compact) + gmt_vcycle + C^H to host "
                              "(gmt_homogenize), wall clock"}
    else:
        out["e2e"] = {"value": None, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                      "note": "not measured for slab-partitioned runs"}
    if breakdown:
        out["breakdown"] = breakdown
    del s_dev, u0_dev
    if not dist and not args.no_like:
        out["like_for_like"] = like_for_like(args, max(args.steps, 5), max(args.warmup, 3))
    if not dist and not args.no_batch and args.physics == "elastic":
        torch.cuda.empty_cache()
        out["batch"] = batch_screening(args)
    if not args.no_cpu_baseline and not dist:
        out["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
