"""Summaries of an ncu --set full capture of one level-0 sweep (k_l0 interior +
ring launches): raw metrics -> profiles/r2/ncu_full_512_k_l0.txt, SASS opcode
histogram -> profiles/r2/sass_hist_512_k_l0.txt, per-sweep DRAM bytes ->
profiles/r2/traffic.json.  Usage: ncu_l0_summary.py <rep> <tag>"""
import collections
import csv
import io
import json
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h = rows[0]
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
out = ["# k_l0 (CUDA-core sum-factorised stencil), 512^3 gyroid elastic, one Jacobi sweep = two launches:",
       "# interior tiles (TL=1, TMA staging: UTMALDG + mbarrier) and the ring of boundary tiles (TL=2, cp.async);",
       "# live they run as parallel graph branches (bench avg_launch_ms is the sweep).",
       f"# source: gpurun_out/{tag}/l0.ncu-rep (ncu --set full --clock-control none -k regex:k_l0 -s 8 -c 2; cold, serialised)"]
tot = 0.0
for v in rows[2:]:
    out += ["", f"{'Kernel Name':70s} {v[h.index('Kernel Name')]}", f"{'Grid Size':70s} {v[h.index('Grid Size')]}"]
    out += [f"{k:70s} {v[h.index(k)]}" for k in keys if k in h]
    tot += float(v[h.index("dram__bytes_read.sum")]) + float(v[h.index("dram__bytes_write.sum")])
    st = []
    for i, k in enumerate(h):
        if "average_warps_issue_stalled_" in k and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v[i]), k.replace("smsp__average_warps_issue_stalled_", "")
                           .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    out.append("# top stall reasons (warps per issue-active cycle)")
    out += [f"  {k:30s} {x:.3f}" for x, k in sorted(st, reverse=True)[:8]]
out += ["", f"# DRAM per sweep (both launches): {tot:.3f} GB read+write vs 6.046 GB algorithmic "
        "(148 B x 40.85 M active nodes)"]
open("profiles/r2/ncu_full_512_k_l0.txt", "w").write("\n".join(out) + "\n")
json.dump({"res": 512, "physics": "elastic", "geometry": "gyroid", "vf": 0.3,
           "kernel": "k_l0<3, M_JACOBI, false> interior (TMA) + ring (cp.async) launches of one sweep",
           "dram_bytes_per_launch": tot * 1e9,
           "source": "profiles/r2/ncu_full_512_k_l0.txt (dram__bytes_read.sum + dram__bytes_write.sum of the "
                     "two launches of one sweep)"}, open("profiles/r2/traffic.json", "w"), indent=1)

txt = ncu("--page", "source", "--csv", "--print-source", "sass")
res, seen = [], set()
for b in txt.split('"Kernel Name"')[1:]:
    lines = ('"Kernel Name"' + b).split("\n")
    name = next(csv.reader([lines[0]]))[1]
    if name in seen:
        continue
    seen.add(name)
    r = list(csv.reader(lines[1:]))
    hh = r[0]
    ia, isrc = hh.index("Instructions Executed"), hh.index("Source")
    cnt, t = collections.Counter(), 0
    for x in r[1:]:
        if len(x) <= ia or not x[ia].isdigit():
            continue
        op = x[isrc].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        o = o.split(".")[0]
        cnt[o] += int(x[ia])
        t += int(x[ia])
    res.append(f"== {name[:100]}\n   total warp instructions executed: {t}")
    res += [f"   {o:12s} {c:12d} {100 * c / t:6.2f}%" for o, c in cnt.most_common(30)]
    res += [f"   [{o}] {cnt.get(o, 0)}" for o in ("UTMALDG", "SYNCS", "LDGSTS", "LDGDEPBAR", "FFMA2", "FADD2", "FMUL2")]
open("profiles/r2/sass_hist_512_k_l0.txt", "w").write(
    f"# SASS opcode histogram (warp instructions executed, ncu source page) of one level-0 Jacobi sweep at 512^3\n"
    f"# (gpurun_out/{tag}/l0.ncu-rep): interior launch with TMA (UTMALDG, SYNCS = mbarrier), ring launch with cp.async (LDGSTS)\n"
    + "\n".join(res) + "\n")
print(f"DRAM per sweep {tot:.3f} GB")
