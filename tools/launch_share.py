"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch
list (cold-cache, serialised per-launch times):

  python tools/launch_share.py <launches.csv> <out.json> "<command it profiled>"
"""
import csv
import json
import sys


def main(path, out, command):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    iu = hdr.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        k = r[ik][:120]
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + v)
    total = sum(t for _, t in agg.values())
    # the bench's device-side gate (a spin kernel that holds the GPU while the
    # host enqueues a run) is not workload: shares are also given without it
    work = sum(t for k, (_, t) in agg.items() if "spin_kernel" not in k)
    share = [{"kernel": k, "launches": n, "total_us": round(t, 1), "pct": round(100 * t / total, 2),
              "pct_of_work": None if "spin_kernel" in k else round(100 * t / work, 2)}
             for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    json.dump({"command": command, "total_us": round(total, 1), "per_kernel_share": share}, open(out, "w"), indent=1)
    for s in share[:8]:
        print(f"{s['pct']:6.2f}% {s['pct_of_work'] or 0:6.2f}%  {s['launches']:5d}  {s['total_us']:10.1f} us  {s['kernel']}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
