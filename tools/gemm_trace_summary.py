"""Summarise a BQRRP_GEMM_TRACE csv: time and achieved TFLOP/s by shape class."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(open(sys.argv[1])))
tot = sum(float(r["ms"]) for r in rows)
flops = sum(2.0 * int(r["M"]) * int(r["N"]) * int(r["K"]) / (2 if int(r["tri"]) else 1) for r in rows)
print(f"{len(rows)} gemms, {tot:.1f} ms, {flops/tot/1e9:.2f} TFLOP/s overall")


def cls(r):
    M, N, K = int(r["M"]), int(r["N"]), int(r["K"])
    kb = "K<=64" if K <= 64 else ("K<=256" if K <= 256 else ("K<=1024" if K <= 1024 else "K>1024"))
    mb = "MN<1M" if M * N < 1 << 20 else ("MN<16M" if M * N < 1 << 24 else "MN>=16M")
    return f"{kb:8s} {mb:8s} t{r['ta']}{r['tb']} tri{r['tri']} split{int(r['nsplit'])>1}"


agg = defaultdict(lambda: [0, 0.0, 0.0])
for r in rows:
    a = agg[cls(r)]
    a[0] += 1
    a[1] += float(r["ms"])
    a[2] += 2.0 * int(r["M"]) * int(r["N"]) * int(r["K"]) / (2 if int(r["tri"]) else 1)
for k, (c, ms, fl) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} n={c:6d} {ms:9.2f} ms {100*ms/tot:5.1f}%  {fl/ms/1e9:6.2f} TF/s")
