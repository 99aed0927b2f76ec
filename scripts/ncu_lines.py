"""Top source lines by warp-stall samples from an ncu report (cuda,sass view).

    python scripts/ncu_lines.py <file.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name") or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    try:
        tot = int(d["Warp Stall Sampling (All Samples)"])
    except (ValueError, KeyError):
        continue
    stalls = {k[6:]: int(v) for k, v in zip(hdr, r)
              if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    rows.append((tot, fname, r[0], r[1].strip()[:70], stalls))
total = sum(x[0] for x in rows)
rows.sort(key=lambda x: -x[0])
print(f"total samples {total}")
for tot, f, ln, src, st in rows[:top]:
    s3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
    print(f"{100 * tot / total:5.1f}% {f}:{ln:5s} {src:70s} | {s3}")
