"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of `bench.py --steps 1
--warmup W`: per-kernel totals of the last (timed) step, i.e. the launches from the last
k_init_prep on.  Usage: python tools/launch_summary.py launches.csv [--json out.json]"""
import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    h, rows = rows[0], rows[1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    names = [r[ki] for r in rows]
    vals = [float(r[vi]) for r in rows]
    starts = [i for i, n in enumerate(names) if n.startswith("k_init_prep")]
    s = starts[-1]
    agg = collections.OrderedDict()
    cnt = collections.Counter()
    for n, v in zip(names[s:], vals[s:]):
        k = n.split("(")[0]
        agg[k] = agg.get(k, 0) + v
        cnt[k] += 1
    tot = sum(agg.values())
    out = {"launches": len(names) - s, "total_ms": tot / 1e6, "kernels": {}}
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / 1e6:9.1f} ms {100 * v / tot:5.1f}%  x{cnt[k]:<3d} {k}")
        out["kernels"][k] = {"ms": v / 1e6, "share": v / tot, "launches": cnt[k]}
    print(f"total {tot / 1e6:.1f} ms, {len(names) - s} launches")
    if "--json" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
