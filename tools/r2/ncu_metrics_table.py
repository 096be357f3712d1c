"""Per-kernel table from an `ncu --metrics ... --csv` launch list (one row per launch):
python tools/r2/ncu_metrics_table.py FILE.csv [algorithmic GB per launch for bwd / fwd, optional]

Prints kernel name, duration, DRAM read / write GB, L2 read / write GB (32-byte sectors) and the
achieved DRAM GB/s, so excess traffic over the algorithmic bytes shows per pass."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        key = (r["ID"], r["Kernel Name"])
        d = rows.setdefault(key, {})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                 "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        d[r["Metric Name"]] = v * scale
    return rows


def main():
    rows = load(sys.argv[1])
    print(f"{'kernel':28s} {'ms':>8s} {'dramR GB':>9s} {'dramW GB':>9s} {'L2R GB':>8s} {'L2W GB':>8s} {'GB/s':>7s}")
    for (i, name), d in rows.items():
        t = d.get("gpu__time_duration.sum", 0.0)
        rd = d.get("dram__bytes_read.sum", 0.0) / 1e9
        wr = d.get("dram__bytes_write.sum", 0.0) / 1e9
        l2r = d.get("lts__t_sectors_op_read.sum", 0.0) * 32 / 1e9
        l2w = d.get("lts__t_sectors_op_write.sum", 0.0) * 32 / 1e9
        gbs = (rd + wr) / t if t else 0.0
        print(f"{name[:28]:28s} {t * 1e3:8.2f} {rd:9.2f} {wr:9.2f} {l2r:8.2f} {l2w:8.2f} {gbs:7.0f}")


if __name__ == "__main__":
    main()
