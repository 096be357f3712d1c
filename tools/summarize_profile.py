"""Summarise a round's ncu captures (gpurun_out/) into profiles/ (tracked).

usage: python tools/summarize_profile.py TAG WORKLOAD
writes profiles/ncu_<TAG>.md (launch list shares, per-launch DRAM traffic vs algorithmic
bytes, key counters of the full captures) and merges profiles/traffic.json.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def read_csv(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    return list(csv.DictReader(io.StringIO(txt[i:])))


def kclass(name):
    for k, c in (("dense_fwd_tc", "dense (tcgen05)"), ("dense_fwd", "dense"),
                 ("dense_bwd", "dense_backward"), ("dense_mat", "materialize"),
                 ("dense_grad", "finalize"), ("dense_rsum", "finalize"),
                 ("tcx_jit_bwd", "backward"), ("tcx_jit_fwd", "forward"), ("tcx_jit_mega", "fused"),
                 ("pass_kernel", "pass_kernel (generic)"), ("materialize", "materialize"),
                 ("finalize", "finalize")):
        if k in name:
            return c
    return "other"


def main():
    tag, workload = sys.argv[1], sys.argv[2]
    lines = [f"# ncu summary {tag} ({workload})", ""]
    # launch list: last step = last N launches (one bench step after warm-up)
    lp = os.path.join(OUT, f"launches_{tag}.csv")
    launches = read_csv(lp) if os.path.exists(lp) else []
    per = defaultdict(float)
    for r in launches:
        if r["Metric Name"] == "gpu__time_duration.sum":
            per[(int(r["ID"]), r["Kernel Name"])] = float(r["Metric Value"])
    ids = sorted(per) or [(0, "materialize")]
    # one step = launches after the last materialize kernel
    firsts = [i for i, (k, n) in enumerate(ids) if "materialize" in n or "dense_mat" in n]
    # a step starts at its first materialize launch (dense plans may launch two)
    last_mat = max(i for i in firsts if i == 0 or i - 1 not in firsts) if firsts else 0
    step = ids[last_mat:]
    tot = sum(per.get(k, 0.0) for k in step) or 1.0
    by = defaultdict(float)
    for k in step:
        by[kclass(k[1])] += per.get(k, 0.0)
    lines += ["## Launch list (one step; ncu per-launch times are cold-cache and serialised)", "",
              "| class | ms | share |", "|---|---|---|"]
    for c, v in sorted(by.items(), key=lambda x: -x[1]):
        lines.append(f"| {c} | {v / 1e6:.2f} | {v / tot:.3f} |")
    # traffic
    tp = os.path.join(OUT, f"traffic_{tag}.csv")
    tr = read_csv(tp) if os.path.exists(tp) else []
    m = defaultdict(dict)
    for r in tr:
        m[(int(r["ID"]), r["Kernel Name"])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        m[(int(r["ID"]), r["Kernel Name"])]["unit_" + r["Metric Name"]] = r["Metric Unit"]
    cls = defaultdict(list)
    for (i, n), d in sorted(m.items()):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = d.get("dram__bytes_read.sum", 0) * scale.get(d.get("unit_dram__bytes_read.sum", "byte"), 1)
        wr = d.get("dram__bytes_write.sum", 0) * scale.get(d.get("unit_dram__bytes_write.sum", "byte"), 1)
        cls[kclass(n)].append(rd + wr)
    # take the last step's launches per class (the captured bench runs 3 warm-up + 1 step)
    lines += ["", "## DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum)", "",
              "| class | launches captured | mean GB / launch |", "|---|---|---|"]
    traffic = {}
    if not cls:
        lines.append("| (no traffic pass this round; see the full captures below) | | |")
    for c, v in cls.items():
        lines.append(f"| {c} | {len(v)} | {sum(v) / len(v) / 1e9:.3f} |")
        traffic[c] = sum(v) / len(v)
    # full captures
    import glob
    reps = sorted(glob.glob(os.path.join(OUT, f"prof_*_{tag}.ncu-rep")))
    for rep in reps:
        kind = os.path.basename(rep)[len("prof_"):-len(f"_{tag}.ncu-rep")]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        keys = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed",
                "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
        lines += ["", f"## `ncu --set full` capture: {kind} kernel", "", "| metric | value |", "|---|---|"]
        for k in keys:
            if k in d:
                lines.append(f"| {k} | {d[k]} {u.get(k, '')} |")
        st = [(float(d[h].replace(",", "")), h) for h in hdr
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")
              and d[h].replace(",", "").replace(".", "").isdigit()]
        tot_s = sum(x for x, _ in st) or 1
        lines.append("| top stall reasons | " + ", ".join(
            f"{h[len('smsp__pcsamp_warps_issue_stalled_'):]} {x / tot_s:.1%}" for x, h in sorted(st, reverse=True)[:6]) + " |")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tj = os.path.join(PROF, "traffic.json")
    allt = json.load(open(tj)) if os.path.exists(tj) else {}
    if traffic:
        allt[workload] = {k: v for k, v in traffic.items()}
        allt[workload]["source"] = f"profiles/ncu_{tag}.md"
    json.dump(allt, open(tj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
