"""Per-kernel table of an ncu --csv metrics log (time us, DRAM MB, L2 MB).
python scripts/ncu_table.py gpurun_out/x.csv [--last N] [--filter regex]"""
import csv, collections, re, sys
path = sys.argv[1]
flt = re.compile(sys.argv[sys.argv.index("--filter") + 1]) if "--filter" in sys.argv else None
rows = list(csv.reader(open(path)))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
scale = {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3,
         "Mbyte": 1, "Gbyte": 1e3, "KB": 1e-3, "MB": 1, "GB": 1e3}
d = collections.OrderedDict()
for r in rows[h + 1:]:
    d.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
items = list(d.values())
if "--last" in sys.argv:
    items = items[-int(sys.argv[sys.argv.index("--last") + 1]):]
tot = 0
for m in items:
    if flt and not flt.search(m["name"]):
        continue
    t = m.get("gpu__time_duration.sum", 0)
    tot += t
    dr = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    print(f"{m['name'][:50]:50s} {t:9.1f} us  dram {dr:8.1f} MB (r {m.get('dram__bytes_read.sum', 0):7.1f})"
          f"  L2 {m.get('lts__t_bytes.sum', 0):8.1f} MB  {dr / t * 1e-3 if t else 0:6.2f} TB/s")
print(f"total {tot:.1f} us")
