"""Summarise ncu --set full captures (.ncu-rep) into markdown: key raw metrics, top stall reasons
(from the source page) and the SASS opcode mix.  python tools/r2/ncu_summary.py OUT.md TITLE REP..."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    out, title, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    lines = [f"# {title}", ""]
    for rep in reps:
        rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
        h, units, v = rows[0], rows[1], rows[2]
        lines += [f"## `{rep.split('/')[-1]}`", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"| {k} | {v[i]} {units[i]} |")
        src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
        if len(src) > 2:
            sh = src[1]
            iS, iE = sh.index("Source"), sh.index("Instructions Executed")
            iW = sh.index("Warp Stall Sampling (All Samples)")
            ops, st = collections.Counter(), collections.Counter()
            for r in src[2:]:
                try:
                    n, w = int(r[iE]), int(r[iW] or 0)
                except (ValueError, IndexError):
                    continue
                t = r[iS].split()
                if not t:
                    continue
                op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
                ops[op] += n
                st[op] += w
            tot, totw = max(sum(ops.values()), 1), max(sum(st.values()), 1)
            lines += ["", "SASS opcode mix (share of executed warp instructions / of stall samples):", ""]
            lines.append(", ".join(f"{op} {n / tot:.1%}/{st[op] / totw:.1%}" for op, n in ops.most_common(12)))
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


main()
