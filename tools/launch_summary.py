#!/usr/bin/env python
"""Summarize an ncu --metrics gpu__time_duration.sum launch list (CSV):
time share per kernel (cold-cache, serialized: compare shares, not times)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
         "msecond": 1.0, "s": 1e3, "second": 1e3}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv, iu, im = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit",
                                             "Metric Name"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0][:80]
        tot[name] += float(r[iv].replace(",", "")) * SCALE[r[iu]]
        cnt[name] += 1
    total = sum(tot.values())
    print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.2f} {100 * v / total:5.1f}% {cnt[k]:8d}  {k}")
    print(f"{total:10.2f} total ms over {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
