"""Write profiles/flow_kernel_traffic.json from an ncu --set full capture of
flow_kernel (read by bench.py for roofline.traffic).

    python scripts/capture_traffic.py <report.ncu-rep> <label>
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def metric(d, key):
    v = d.get(key, "")
    return float(v.replace(",", "")) if v not in ("", "n/a") else None


def main():
    rep, label = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    recs = [dict(zip(hdr, r)) for r in rows[2:]]
    recs = [r for r in recs if "flow_kernel" in r.get("Kernel Name", "")]
    if not recs:
        sys.exit("no flow_kernel launch in the report")
    r = recs[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = metric(r, "dram__bytes_read.sum") * scale.get(units.get("dram__bytes_read.sum"), 1)
    wr = metric(r, "dram__bytes_write.sum") * scale.get(units.get("dram__bytes_write.sum"), 1)
    n, m, d = 2000, 10_000, 2
    algo = 8 * (n * d + m * d + 2 * n + n * d + 2 * n)  # X, Y, warm in; flow, warm out
    rec = {
        "kernel": r["Kernel Name"][:120],
        "dram_bytes_per_launch": rd + wr,
        "dram_read": rd,
        "dram_write": wr,
        "algorithmic_bytes_per_launch": algo,
        "duration_us": metric(r, "gpu__time_duration.sum") * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3,
                                                              "msecond": 1e3}.get(
            units.get("gpu__time_duration.sum"), 1.0),
        "source": f"ncu --set full capture {label} (one flow_kernel launch, config 2)",
    }
    with open(os.path.join(ROOT, "profiles", "flow_kernel_traffic.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
