"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of tools/profile_run.py: the LAST
factorization (from its init_j_kernel on), kernel time grouped by kernel name.
    python tools/launch_summary.py launches.csv [top]"""
import collections
import csv
import re
import sys


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = []
    for x in csv.DictReader(lines):
        if x["Metric Name"] == "gpu__time_duration.sum":
            rows.append((int(x["ID"]), x["Kernel Name"], float(x["Metric Value"]), x["Grid Size"], x["Block Size"]))
    starts = [i for i, x in enumerate(rows) if "init_j_kernel" in x[1]]
    return rows[starts[-1]:] if starts else rows


def short(n):
    n = re.sub(r"\(.*", "", n).replace("void ", "").replace("bqrrp::", "")
    return n[:64]


def main():
    seg = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, n, t, g, b in seg:
        a = agg[short(n)]
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values())
    print("total %.1f ms of kernel time (serialised) over %d launches" % (tot / 1e6, len(seg)))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print("%-64s %6d %9.2f ms %5.1f%%  avg %8.2f us" % (k, v[0], v[1] / 1e6, 100 * v[1] / tot, v[1] / v[0] / 1e3))


if __name__ == "__main__":
    main()
