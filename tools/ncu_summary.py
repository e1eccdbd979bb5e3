"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name: count, total ms, share."""
import csv
import sys
from collections import defaultdict


def summarise(path, skip_launches=0):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:][skip_launches:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ms = v / 1e6 if unit == "nsecond" else (v / 1e3 if unit == "usecond" else (v if unit == "msecond" else v / 1e6))
        name = r[ki].split("(")[0].split("<")[0]
        tot[name] += ms
        cnt[name] += 1
    all_ms = sum(tot.values())
    out = sorted(tot.items(), key=lambda x: -x[1])
    return all_ms, [(k, cnt[k], v, v / all_ms) for k, v in out]


if __name__ == "__main__":
    all_ms, out = summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    print(f"total kernel time {all_ms:.2f} ms over {sum(c for _, c, _, _ in out)} launches")
    for k, c, v, s in out:
        print(f"{k:45s} {c:7d} {v:10.3f} ms {100*s:6.2f}% avg {1e3*v/c:9.2f} us")
