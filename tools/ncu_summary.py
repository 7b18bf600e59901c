"""Summarise one-kernel `ncu --set full` captures: duration, throughput
breakdown, DRAM traffic, tensor-pipe activity and the hottest SASS lines.

    python tools/ncu_summary.py gpurun_out/prof_l1.ncu-rep [--top 25]

Reads the report with `ncu -i --page raw/source --csv` (the ncu in this image)
and prints a plain-text summary suitable for profiles/."""
import argparse
import csv
import io
import subprocess

RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_elapsed", "tcgen05 pipe active %"),
    ("sm__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem / CTA"),
    ("launch__registers_per_thread", "registers / thread"),
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True,
                         check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--cuda", action="store_true", help="also: hottest CUDA source lines (needs -lineinfo)")
    a = ap.parse_args()
    rows = ncu_csv(a.rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"kernel: {vals[col['Kernel Name']]}")
    for key, label in RAW:
        cands = [h for h in hdr if h == key] or [h for h in hdr if h.startswith(key.split(".")[0]) and
                                                  key.split(".")[-1] in h and key.split(".")[0] in h][:1]
        if not cands:
            continue
        h = cands[0]
        print(f"  {label:28s} {vals[col[h]]:>16s} {units[col[h]]}")
    src = ncu_csv(a.rep, "source", ["--print-source", "sass"])
    # first row is the kernel name line, second the header
    i0 = next(i for i, r in enumerate(src) if r and r[0] == "Address")
    h = src[i0]
    ia, isrc = h.index("Address"), h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    data = [r for r in src[i0 + 1:] if len(r) == len(h)]
    tot = sum(float(r[iss] or 0) for r in data) or 1.0
    print(f"  stall samples total {tot:.0f}; hottest SASS lines:")
    for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:a.top]:
        print(f"    {float(r[iss] or 0) / tot * 100:5.1f}%  exec {int(r[iex] or 0):>10d}  {r[isrc].strip()[:90]}")
    if a.cuda:
        for sec in ("WarpStateStats", "SchedulerStats"):
            out = subprocess.run(["ncu", "-i", a.rep, "--page", "details", "--section", sec, "--csv"],
                                 capture_output=True, text=True).stdout
            rows = list(csv.reader(io.StringIO(out)))
            if rows:
                h = rows[0]
                im, iu, iv = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
                print(f"  [{sec}]")
                for r in rows[1:]:
                    if len(r) == len(h):
                        print(f"    {r[im]:50s} {r[iv]:>12s} {r[iu]}")
        out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        files, cur, lines = [], None, []
        for r in rows:
            if len(r) == 1 and r[0].startswith("File"):
                cur = r[0]
                continue
            if r and r[0] == "Line":
                h = r
                continue
            if cur is not None and len(r) > 3 and r[0].isdigit():
                try:
                    lines.append((float(r[h.index("Warp Stall Sampling (All Samples)")] or 0), cur.split("/")[-1],
                                  r[0], r[h.index("Source")].strip()[:80]))
                except (ValueError, NameError):
                    pass
        tot2 = sum(x[0] for x in lines) or 1.0
        print(f"  hottest CUDA lines ({tot2:.0f} samples):")
        for smp, f, ln, src in sorted(lines, key=lambda x: -x[0])[:a.top]:
            print(f"    {smp / tot2 * 100:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
