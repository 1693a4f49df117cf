"""Summarise ncu captures into profiles/r2/ncu_summary.json (read by bench.py for
roofline.traffic) and print a short table.

    python tools/ncu_summary.py CONFIG report.ncu-rep [report2.ncu-rep ...]
    python tools/ncu_summary.py --launches CONFIG launches.csv
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r2", "ncu_summary.json")
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         # durations are stored in milliseconds
         "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def short(name):
    n = name.split("(")[0].replace("void ", "")
    return n.split("::")[-1].split("<")[0]


def from_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, out = rows[0], rows[1], {}
    for r in rows[2:]:
        k = short(r[hdr.index("Kernel Name")])
        rec = {}
        for m in WANT:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                rec[m] = v * SCALE.get(units[i], 1)
        rec["dram_bytes"] = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
        if "gpu__time_duration.sum" in rec:
            rec["duration_ms"] = rec.pop("gpu__time_duration.sum")
        rec["source"] = os.path.relpath(path, ROOT)
        out[k] = rec
    return out


def main():
    if sys.argv[1] == "--launches":
        cfg, path = sys.argv[2], sys.argv[3]
        rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
        tot = {}
        for r in rows:
            k = short(r[4])
            tot.setdefault(k, [0.0, 0])
            tot[k][0] += float(r[-1]) * 1e-6
            tot[k][1] += 1
        allms = sum(v[0] for v in tot.values())
        for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
            print(f"{v[0]:9.3f} ms {100 * v[0] / allms:5.1f}%  x{v[1]:3d}  {k}")
        return
    cfg = sys.argv[1]
    js = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for p in sys.argv[2:]:
        js.setdefault(cfg, {}).update(from_report(p))
    json.dump(js, open(OUT, "w"), indent=1, sort_keys=True)
    for k, v in js[cfg].items():
        print(k, {m: v[m] for m in v if m != "source"})


if __name__ == "__main__":
    main()
