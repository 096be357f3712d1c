"""Collect the bench JSON lines (last line of each gpurun_out log) into a profiles/*.jsonl file:
python tools/r2/collect.py OUT.jsonl LOG..."""
import json
import os
import sys

out = sys.argv[1]
with open(out, "a") as f:
    for path in sys.argv[2:]:
        try:
            last = [ln for ln in open(path).read().splitlines() if ln.startswith("{")][-1]
            d = json.loads(last)
        except Exception as ex:  # a failed run: record why
            d = {"error": repr(ex)}
        d["source_log"] = os.path.basename(path)
        f.write(json.dumps(d) + "\n")
