"""bench.py -- GMG V-cycle throughput of libgmt on B200 (driver contract).

Metric (BASELINE.json): "512^3 elasticity GMG V-cycles/s & DOF/s at 1/2/4/8 B200;
% HBM roofline".  Workload at N=1: configs[4]'s problem -- 512^3 linear
elasticity on a gyroid TPMS lattice, all 6 load cases, one V-cycle from a
given initial guess -- which fits one B200 (configs[1] 64^3 is a parity
case).  One step = one pass of the whole hot path:
  Galerkin coarse-operator build from the (device-resident) material
  + set the given initial guess (Alg. 2 line 1)
  + one V-cycle (damped-Jacobi smoothing, residual, restriction,
    prolongation, coarse levels, coarsest solve) for all 6 load cases
  + C^H reduction (App. F1) read back to the host.
value = steps/s ("V-cycles/s" as single-cycle homogenisations per second);
DOF/s = 3 N^3 * 6 load cases * value.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--res 512] [--physics elastic]
  python bench.py --impl reference ...   (the FP64 oracle on host cores)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_L0_JACOBI = {"elastic": 2 * 18 * 4 + 4, "thermal": 2 * 3 * 4 + 4}  # per active node, DESIGN.md Sec. 8(d)


def active_nodes(s: np.ndarray, z0: int = 0, nz: int | None = None) -> int:
    """Nodes of planes [z0, z0+nz) touching at least one non-void voxel (the
    sparse active set)."""
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
    ap.add_argument("--breakdown", action="store_true", help="extra pass with per-class event timing")
    ap.add_argument("--no-solve", action="store_true", help="skip the (untimed) full solve to 1e-5")
    return ap.parse_args()


def make_material(args):
    import synth
    n = args.res
    if args.geometry == "gyroid":
        return synth.tpms(n, "gyroid", args.vf)
    if args.geometry == "gyroid_sheet":
        return synth.tpms(n, "gyroid", args.vf, sheet=True)
    if args.geometry == "truss":
        return synth.truss(n, "octet", 0.05)
    if args.geometry == "stochastic":
        return synth.stochastic(n, args.vf, seed=0)
    if args.geometry == "solid":
        return synth.solid(n)
    raise ValueError(args.geometry)


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
    kernel from the committed `ncu --set full` capture (profiles/r1/traffic.json),
    when it was taken on this exact single-GPU workload; else None."""
    p = os.path.join(ROOT, "profiles", "r1", "traffic.json")
    if world != 1 or not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    same = (d.get("res") == args.res and d.get("physics") == args.physics and d.get("geometry") == args.geometry
            and abs(float(d.get("vf", -1)) - args.vf) < 1e-9 and args.levels in (0, 8))
    return (float(d["dram_bytes_per_launch"]), d["source"]) if same else (None, None)


# --------------------------------------------------------------------------- oracle leg

ORACLE_SAMPLE_N = 64   # configs[1]'s size: ~8 s of single-thread oracle work


def oracle_sample(physics: str, n_sample: int = ORACLE_SAMPLE_N, vf: float = 0.3):
    """One step of the same workload run by the FP64 oracle on a bounded
    sample (an n_sample^3 gyroid, same generator and settings), single
    threaded.  Returns (seconds, sample description)."""
    from threadpoolctl import threadpool_limits

    import synth
    from oracle import fem, gmg
    s = synth.tpms(n_sample, "gyroid", vf)
    ph = fem.Physics(physics)
    om = 0.45 if physics == "elastic" else 0.6
    L = gmg.default_levels(n_sample)
    with threadpool_limits(1):
        t0 = time.perf_counter()
        H = gmg.Hierarchy(s, ph, L)                     # assembly + Galerkin build
        u0 = np.zeros_like(H.f)
        u = gmg.vcycle(H, u0, omega=om, pre=2, post=2, coarse=16)
        fem.effective_tensor(s, ph, u)
        dt = time.perf_counter() - t0
    return dt, f"{n_sample}^3 gyroid v_f={vf}, L={L}: assembly+Galerkin+1 V-cycle+C^H, 1 thread"


def cpu_baseline(args):
    n_s = ORACLE_SAMPLE_N
    dt, desc = oracle_sample(args.physics, n_s, args.vf)
    scale = (args.res / n_s) ** 3          # oracle cost is linear in the node count
    return {"value": 1.0 / (dt * scale), "unit": "V-cycles/s", "cores": 1, "kind": "oracle",
            "sample": desc + f"; {dt:.2f} s, scaled by (N/{n_s})^3 = {scale:.0f} to the {args.res}^3 workload"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = []
    n_s = ORACLE_SAMPLE_N
    for _ in range(args.warmup):
        oracle_sample(args.physics, n_s, args.vf)
    for _ in range(args.steps):
        dt, desc = oracle_sample(args.physics, n_s, args.vf)
        steps.append(dt)
    scale = (args.res / n_s) ** 3
    ms = float(np.mean(steps)) * scale * 1e3
    val = 1e3 / ms
    out = {"impl": "reference", "metric": "512^3 elasticity GMG V-cycles/s (single-cycle homogenisation)",
           "value": val, "unit": "V-cycles/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.res}^3 {args.physics} gyroid TPMS v_f={args.vf}, 6 load cases"},
           "cpu_baseline": {"value": val, "unit": "V-cycles/s", "cores": 1, "kind": "oracle",
                            "sample": desc + f"; per-step time scaled by (N/{n_s})^3={scale:.0f}"},
           "e2e": {"value": val, "unit": "V-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# --------------------------------------------------------------------------- our leg

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import synth
    from paper_2604_26518_b200 import Problem, build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        world = max(world, 1)
    dist = world > 1
    if dist:
        import torch.distributed as td
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    build.build()

    s = make_material(args)
    n = args.res
    nr, dpn = (6, 3) if args.physics == "elastic" else (3, 1)
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
    P.gmt_profile_enable(1)   # bracket the dominant kernel (level-0 Jacobi) live
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
    rel_before = None

    clocks = Clocks(local)
    if dist:
        td.barrier()
    torch.cuda.synchronize()
    launches0 = P.gmt_kernel_launches()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    clocks.start()
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(args.steps):
            CH = step()
            P.gmt_profile_collect()
        e1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist:
        td.barrier()
    launches = P.gmt_kernel_launches() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        td.all_reduce(t, op=td.ReduceOp.MAX)
        ms = float(t.item())
    k_ms, k_cnt = P.gmt_profile_read(0)
    rel, _, _ = P.gmt_residual_norms()

    # ---- e2e: public API with host buffers: the step's inputs (u8 occupancy
    # and the given initial guess, both in pinned host memory) are copied to
    # the device inside the timed region every step, C^H is read back.
    s_u8 = torch.from_numpy((s_loc > 0).astype(np.uint8)).pin_memory().numpy()
    if not np.all((s_loc == 0) | (s_loc == 1)):
        s_u8 = None
    s_host = np.ascontiguousarray(s_loc) if s_u8 is None else s_u8
    u0_host = u0_dev.cpu().pin_memory().numpy()

    def e2e_step():
        P.gmt_set_material(s_host)
        P.gmt_set_initial_guess(u0_host)
        P.gmt_vcycle(1)
        return P.gmt_homogenize()

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if dist:
        td.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    if dist:
        e2e_ms = gd.max_over_ranks(e2e_ms, device="cuda")
    u0_bytes = int(u0_host.nbytes)
    del u0_host

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
    bytes_launch = BYTES_L0_JACOBI[args.physics] * n_act
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

    nodes = n ** 3
    hbm, hbm_src = measured_peaks()
    achieved = bytes_launch / (avg_ms * 1e-3) / 1e9
    hbm_agg = hbm * world
    traffic, traffic_src = ncu_traffic(args, world)
    value = 1e3 / ms
    dofs = dpn * nodes * nr
    out = {
        "metric": "512^3 elasticity GMG V-cycles/s (single-cycle homogenisation: Galerkin build + 1 V-cycle + C^H)",
        "value": value, "unit": "V-cycles/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{n}^3 {args.physics} {args.geometry} TPMS v_f={args.vf}, {nr} load cases, "
                               f"one V-cycle from a given initial guess",
                   "levels": levels, "smoother": "damped Jacobi (2 pre, 2 post, 16 coarsest)",
                   "l2": "inputs larger than L2 (9.7 GB level-0 vectors)",
                   "parallelism": f"slab{world} (z-slabs, NCCL halos)" if dist else "single GPU"},
        "dof_per_s": dofs * value,
        "roofline": {"bound": "hbm", "kernel": "level-0 damped-Jacobi sweep (k_fine_tiled + k_iface)",
                     "achieved": achieved, "peak": hbm_agg, "unit": "GB/s", "frac": achieved / hbm_agg,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": hbm_src,
                     "bytes_per_launch": bytes_launch, "bytes_rule": "148 B (elastic) x active nodes",
                     "active_nodes": n_act, "avg_launch_ms": avg_ms, "launches_timed": k_cnt,
                     "share_of_step": k_ms / args.steps / ms},
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": {"value": 1e3 / e2e_ms, "unit": "V-cycles/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(s_host.nbytes + u0_bytes), "d2h_bytes_per_step": nr * nr * 8,
                "note": "pinned host material (uint8 occupancy) + pinned host initial guess through "
                        "gmt_set_material/gmt_set_initial_guess/gmt_vcycle/gmt_homogenize"},
        "residual_after_cycle": float(np.max(rel)),
        "solve": solve,
        "C_H_diag": [float(CH[i, i]) for i in range(nr)],
    }
    if breakdown:
        out["breakdown"] = breakdown
    if not args.no_cpu_baseline and not dist:
        out["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
