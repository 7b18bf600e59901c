"""Summarise an ncu --csv launch list: per-kernel time, DRAM bytes, and
(for a generator forward) per-layer FLOP efficiency vs the measured peak."""
import csv
import json
import os
import sys
from collections import OrderedDict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, ks = None, OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = (int(d["ID"]), d["Kernel Name"])
            ks.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", "") or 0)
    return ks


def main(path, B=512, last=0):
    ks = load(path)
    if last:  # only the final `last` launches (e.g. the last forward of a multi-forward capture)
        ks = OrderedDict(list(ks.items())[-last:])
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))
    try:
        from paper_2512_18318_b200 import generator
        Ls, shapes = generator.layers(), generator.layer_shapes()
        names = [n for n in "fe0 fe1.0 fe1.1 fe1.2 fe2.0 fe2.1 fe2.2 fe2.3 fe3.0 fe3.1 fe3.2 fe4.0 fe4.1 fe4.2 fe5.0 fe5.1 "
                 "fe6.0 fe6.1 ae0 ae1 ae2 ae3 ae4 ae5 ae6 ae7 ae8 ae9 ae10 ae11 ae12 fd0 fd1.0 fd1.1 fd2.0 fd2.1 "
                 "fd2.2 fd3.0 fd3.1 fd3.2 fd4.0 fd4.1 fd4.2 fd5.0 fd5.1 fd5.2 fd6.0 fd6.1 fd6.2 out0+1".split()]
    except Exception:
        Ls = None
    tot = 0.0
    li = 0
    print(f"{'id':>3} {'layer':8} {'kernel':28} {'us':>9} {'TF/s':>7} {'frac':>6} {'DRAM MB':>8} {'HBM-us':>7}")
    for (i, name), m in ks.items():
        t = m.get("gpu__time_duration.sum", 0.0) / 1e3
        tot += t
        dram = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
        lname, tf, frac = "", 0.0, 0.0
        if Ls and ("conv_tc" in name or "conv_halo" in name or "audio_stem" in name):
            if li == len(names):  # next forward of a multi-rep capture
                print(f"subtotal {tot - t:.1f} us")
                li = 0
            L = Ls[li]
            hi, wi, ho, wo = shapes[li]
            pix = ho * wo if L.kind == 0 else hi * wi
            fl = 2 * pix * L.cin * L.cout * L.kh * L.kw * B
            if li == 49:
                fl += 2 * ho * wo * 32 * 3 * B
            tf = fl / (t * 1e-6) / 1e12
            frac = tf / peak["bf16_tflops"]
            lname = names[li]
            li += 1
        print(f"{i:3d} {lname:8} {name[:28]:28} {t:9.1f} {tf:7.1f} {frac:6.3f} {dram:8.1f} {dram / peak['hbm_gbs'] * 1e3:7.1f}")
    print(f"total {tot:.1f} us")


if __name__ == "__main__":
    # launches.py <csv> [B] [last N launches]
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 512, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
