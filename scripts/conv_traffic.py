"""DRAM traffic of the feature-computation launches of one bench step, from one
`ncu --set full` capture of scripts/one_pass.py (run on the GPU box, repo root):

  ncu --set full --clock-control none --profile-from-start off -k regex:"k_conv_tc|k_convert" \
      -o gpurun_out/conv_all -f python scripts/one_pass.py --t-from profiles/r1_bench.json
  python scripts/conv_traffic.py gpurun_out/conv_all.ncu-rep profiles/r1_conv_traffic.json --config 2

Writes per-launch rows (kernel, us, DRAM read / write bytes, tensor-pipe %) and the per-step
sums that bench.py reports as roofline.traffic.  ncu replays each launch serialised and
cold-cache, so the bytes are an upper bound on what the graph-launched step moves.
"""
import argparse
import csv
import io
import json
import subprocess

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6, "%": 1, "": 1}

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("out")
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--n-voxels", type=int, default=None)
a = ap.parse_args()

raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]


def val(r, m):
    i = hdr.index(m)
    try:
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
    except ValueError:
        return 0.0


launches = []
for r in data:
    launches.append({
        "kernel": r[hdr.index("Kernel Name")].split("(")[0],
        "us": val(r, "gpu__time_duration.sum"),
        "dram_read": val(r, "dram__bytes_read.sum"),
        "dram_write": val(r, "dram__bytes_write.sum"),
        "tensor_pct": val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    })
tot = sum(x["dram_read"] + x["dram_write"] for x in launches)
us = sum(x["us"] for x in launches)
json.dump({"config": a.config, "n_voxels": a.n_voxels, "capture": "ncu --set full --clock-control none, "
           "scripts/one_pass.py (one bench step, same t), kernels k_conv_tc|k_convert",
           "n_launches": len(launches), "dram_bytes_per_step": tot, "time_us_sum": us,
           "dram_gbps_over_sum": tot / (us * 1e3) if us else None, "launches": launches},
          open(a.out, "w"), indent=1)
print(f"{len(launches)} launches, {tot / 1e6:.1f} MB DRAM, {us:.1f} us")
