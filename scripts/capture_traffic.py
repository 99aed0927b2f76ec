"""Write a traffic record (read by bench.py for roofline.traffic) from an ncu
--set full capture of one flow_kernel launch.

    python scripts/capture_traffic.py <report.ncu-rep> <label> [n m d out.json]

Defaults: config 2 (n=2000, m=1e4, d=2) -> profiles/flow_kernel_traffic.json.
Algorithmic bytes per launch: X and Y read once, warm potentials read and
written, the flow written (float64).
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
    n, m, d = (int(v) for v in sys.argv[3:6]) if len(sys.argv) > 5 else (2000, 10_000, 2)
    dest = sys.argv[6] if len(sys.argv) > 6 else os.path.join("profiles", "flow_kernel_traffic.json")
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
        "source": f"ncu --set full capture {label} (one flow_kernel launch, n={n} m={m} d={d})",
    }
    with open(os.path.join(ROOT, dest), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
