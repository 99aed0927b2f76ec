"""Summarise ncu outputs into markdown for profiles/.

    python scripts/summarize_ncu.py launches <launches.csv>      per-kernel device-time shares
    python scripts/summarize_ncu.py report <file.ncu-rep> [...] key metrics of full captures
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += v * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(f"| kernel | launches | total us | share | avg us |\n|---|---:|---:|---:|---:|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"| `{k[:70]}` | {cnt[k]} | {v:.1f} | {100 * v / total:.1f}% | {v / cnt[k]:.2f} |")
    print(f"\n{sum(cnt.values())} launches, {total:.1f} us of device time "
          "(ncu: serialised, cold caches -- compare shares, not absolutes)")


KEYS = [
    "gpu__time_duration.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "smsp__inst_executed.sum",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"### `{d.get('Kernel Name', '?')[:110]}`\n")
        print("| metric | value |\n|---|---:|")
        for k in KEYS:
            if k in d:
                print(f"| {k} | {d[k]} |")
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): d[k] for k in d
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
        print("\nTop warp-stall samples: " + ", ".join(f"{k} {v}" for k, v in top) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        for p in sys.argv[2:]:
            report(p)
