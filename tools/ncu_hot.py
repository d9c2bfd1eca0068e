"""Summarise an ncu report: per-kernel headline metrics and the SASS
instructions with the most warp-stall samples (needs -lineinfo builds).

  python tools/ncu_hot.py gpurun_out/prof.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units = raw[0], raw[1]
    for r in raw[2:]:
        name = r[hdr.index("Kernel Name")]
        vals = []
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals.append(f"{m.split('.')[0].split('__')[1]}={r[i]}{units[i]}")
        print(name[:70], "|", " ".join(vals))
    src = run([rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "-c", "1"])
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h)]
    si = h.index("Warp Stall Sampling (All Samples)")
    ex = h.index("Instructions Executed")
    tot = sum(int(r[si]) for r in data if r[si].isdigit())
    print(f"-- {kre}: {tot} stall samples; top instructions:")
    for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:top]:
        print(f"{r[si]:>6} {r[ex]:>8} {r[0][-5:]} {r[h.index('Source')][:80]}")


if __name__ == "__main__":
    main()
