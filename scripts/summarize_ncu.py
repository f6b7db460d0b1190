"""Summarise ncu artefacts into profiles/ (run on the CPU box after gpurun).

python scripts/summarize_ncu.py launches <launches.csv> <out.md>
python scripts/summarize_ncu.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
           "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot, dram, cnt = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    for r in data:
        try:
            v = float(r[vi].replace(",", "")) * (scale.get(r[ui], 1.0) if ui is not None else 1.0)
        except (ValueError, IndexError):
            continue
        k = r[ki].split("(")[0]
        m = r[mi] if mi is not None else "gpu__time_duration.sum"
        if m == "gpu__time_duration.sum":
            tot[k] += v
            cnt[k] += 1
        elif m.startswith("dram__bytes"):
            dram[k] += v
    T = sum(tot.values())
    D = sum(dram.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({path})\n\n")
        f.write("Per-launch gpu__time_duration.sum (+ DRAM read+write), --clock-control none, serialised and\n")
        f.write("cold-cache: compare SHARES, not absolute times.\n\n| kernel | launches | total us | share | DRAM MB |\n"
                "|---|---|---|---|---|\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"| {k} | {cnt[k]} | {v / 1e3:.1f} | {100 * v / T:.1f}% | {dram[k] / 1e6:.1f} |\n")
        f.write(f"\n{sum(cnt.values())} launches, {T / 1e3:.1f} us total, {D / 1e6:.1f} MB DRAM\n")


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary ({rep})\n\n")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            f.write(f"## {name[:120]}\n")
            for m in METRICS:
                if m in hdr:
                    f.write(f"{m:70s} {r[hdr.index(m)]}\n")
            f.write("\n")
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(src)))
        if len(srows) > 2:
            h = srows[1]
            si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
            data = [x for x in srows[2:] if len(x) > wi and x[wi].isdigit()]
            totw = sum(int(x[wi] or 0) for x in data) or 1
            f.write("## top warp-stall SASS lines (first kernel in report)\n")
            for x in sorted(data, key=lambda x: -int(x[wi] or 0))[:15]:
                f.write(f"{100 * int(x[wi]) / totw:5.1f}%  {x[si].strip()[:100]}\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
