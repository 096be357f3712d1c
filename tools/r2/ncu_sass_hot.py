"""Top stalled SASS instructions of an ncu report (source page, SASS view):
python tools/r2/ncu_sass_hot.py REP [N] -> opcode-level stall share and the N hottest lines."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and any("Warp Stall Sampling" in c for c in r):
        hdr = i
        break
if hdr is None:
    print("no source table", rows[:3])
    sys.exit(0)
h = rows[hdr]
isrc = h.index("Source")
ist = [i for i, c in enumerate(h) if c.startswith("Warp Stall Sampling (All")][0]
iex = [i for i, c in enumerate(h) if c.startswith("Instructions Executed")]
iex = iex[0] if iex else None
data = []
for r in rows[hdr + 1:]:
    if len(r) <= ist:
        continue
    try:
        s = float(r[ist] or 0)
    except ValueError:
        continue
    ex = float(r[iex] or 0) if iex is not None and r[iex] not in ("", None) else 0.0
    data.append((s, ex, r[isrc].strip()))
tot = sum(d[0] for d in data) or 1.0
byop = collections.Counter()
exop = collections.Counter()
for s, ex, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    byop[op] += s
    exop[op] += ex
print(f"{rep}: stall samples {tot:.0f}")
tex = sum(exop.values()) or 1.0
for op, s in byop.most_common(15):
    print(f"  {op:10s} stall {100 * s / tot:5.1f}%  executed {100 * exop[op] / tex:5.1f}%")
print("hottest:")
for s, ex, src in sorted(data, reverse=True)[:N]:
    print(f"  {100 * s / tot:5.2f}%  {src[:110]}")
