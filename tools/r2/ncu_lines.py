"""Attribute ncu per-instruction stall samples and executed instructions to lines of the
generated JIT source: python tools/r2/ncu_lines.py REP CUBIN SRC [N]
(CUBIN / SRC: the TCX_JIT_DUMP files of the same kernel; nvdisasm -g maps SASS offsets to
source lines, ncu's source page gives per-address counts)."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, cubin, src = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr]
ia, isrc = h.index("Address"), h.index("Source")
ist = h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
recs = []
for r in rows[hdr + 1:]:
    if len(r) <= iex:
        continue
    try:
        recs.append((int(r[ia], 16), float(r[ist] or 0), float(r[iex] or 0), r[isrc].strip()))
    except ValueError:
        pass
base = min(a for a, _, _, _ in recs)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
for ln in dis.splitlines():
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
srclines = open(src).read().splitlines()
agg = collections.defaultdict(lambda: [0.0, 0.0])
miss = 0
for a, s, ex, _ in recs:
    key = line_of.get(a - base)
    if key is None:
        miss += 1
        key = ("?", 0)
    agg[key][0] += s
    agg[key][1] += ex
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"{rep}: {len(recs)} instructions, unmapped {miss}")
for (f, ln), (s, ex) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    text = srclines[ln - 1].strip()[:90] if f.startswith("tcx_jit") and 0 < ln <= len(srclines) else ""
    print(f"{100 * s / ts:5.2f}% stall {100 * ex / te:5.2f}% exec  {f}:{ln}  {text}")
