"""Per-launch table of the LAST generator forward in an ncu launch list
(`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file X.csv python tools/gen_forward.py B reps prec`):

    python tools/layer_table.py X.csv N     (N = launches per forward)

Columns: launch, kernel (template args abbreviated), us, DRAM MB; totals."""
import csv
import sys
from collections import OrderedDict


def main():
    path, n = sys.argv[1], int(sys.argv[2])
    rows = OrderedDict()
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        k = rows.setdefault(r["ID"], {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            k["us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]
        elif r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[unit]
            k["dram"] = k.get("dram", 0.0) + v * scale
    last = list(rows.values())[-n:]
    tot_us = tot_mb = 0.0
    for i, k in enumerate(last):
        name = k["name"].replace("(lsg::gen::", "(").split("(")[0][:44]
        us, mb = k.get("us", 0.0), k.get("dram", 0.0) / 1e6
        tot_us += us
        tot_mb += mb
        print(f"{i:3d}  {name:44s} {us:8.1f} us {mb:9.1f} MB")
    print(f"total {tot_us:.1f} us, {tot_mb:.1f} MB DRAM over {len(last)} launches")


if __name__ == "__main__":
    main()
