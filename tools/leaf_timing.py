"""Per-phase cycle breakdown of the K-LU / K-SQR register leaves (experiment, not product): builds a separate copy
of the library with -DBQRRP_LEAF_TIMING into /tmp, runs one warm leaf through bqrrp_debug_lu_pivots /
bqrrp_debug_sketch_qr and prints the mean clock64 deltas per column for thread 0 of the first and the last CTA.
    python tools/leaf_timing.py [rows] [cols] [lu|qr]"""
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

LIB = "/tmp/libbqrrp_timing.so"


def build():
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2507_00976_b200", "csrc", "*.cu")))
    objs = []
    procs = []
    for s in srcs:
        o = "/tmp/lt_" + os.path.basename(s) + ".o"
        cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
               "--expt-relaxed-constexpr", "-DBQRRP_LEAF_TIMING", "-I", os.path.join(ROOT, "include"), "-c", s, "-o", o]
        procs.append(subprocess.Popen(cmd))
        objs.append(o)
    for p in procs:
        assert p.wait() == 0
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
                           "-lcudart_static", "-lrt", "-ldl", "-lpthread"])


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    cols = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    kind = sys.argv[3] if len(sys.argv) > 3 else "lu"
    build()
    if kind == "qr":
        return qr_main(rows)
    import torch

    import paper_2507_00976_b200 as bq

    bq._LIB_PATH = LIB
    L = bq.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    X0 = torch.randn(cols, rows, dtype=torch.float64, device="cuda", generator=g).t()
    for _ in range(3):
        X = X0.clone().t().contiguous().t()
        bq.debug_lu_pivots(X)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * (2 * 64 * 8))()
    assert L.bqrrp_debug_leaf_timing(buf) == 0
    names = ["wait", "reduce", "relabel", "lookahead->sync", "sync->pushed", "push->ret", "update"]
    for c in range(2):
        ts = [[buf[(c * 64 + j) * 8 + k] for k in range(8)] for j in range(min(cols, 32))]
        d = {n: 0.0 for n in names}
        nj = 0
        for j in range(1, min(cols, 32) - 1):
            t = ts[j]
            d["wait"] += t[1] - t[0]
            d["reduce"] += t[2] - t[1]
            d["relabel"] += t[3] - t[2]
            d["lookahead->sync"] += t[4] - t[3]
            d["sync->pushed"] += t[5] - t[4]
            d["push->ret"] += t[6] - t[5]
            d["update"] += t[7] - t[6]
            nj += 1
        tot = sum(d.values())
        print(f"{'first' if c == 0 else 'last'} CTA, rows={rows}: cycles per column " +
              ", ".join(f"{k} {v / nj:.0f}" for k, v in d.items()) + f" | total {tot / nj:.0f}")
        e = [buf[(c * 64 + 63) * 8 + k] for k in range(5)]
        print(f"   leaf (the last of the {cols}-column LU): prologue {e[1] - e[0]}, column loop {e[2] - e[1]}, "
              f"move lists {e[4] - e[2]}, row moves over all {cols} columns {e[3] - e[4]} cycles")


def qr_main(rows):
    import torch

    import paper_2507_00976_b200 as bq

    bq._LIB_PATH = LIB
    L = bq.lib()
    g = torch.Generator(device="cuda").manual_seed(0)
    X0 = torch.randn(rows, 32, dtype=torch.float64, device="cuda", generator=g).t()  # WT: 32 x rows -> one leaf
    for _ in range(3):
        X = X0.clone().t().contiguous().t()
        bq.debug_sketch_qr(X)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * (2 * 64 * 8))()
    assert L.bqrrp_debug_qleaf_timing(buf) == 0
    names = ["q+transpose-reduce", "block barrier", "CTA sum+push", "wait", "slot sum+beta/tau", "update"]
    for c in range(2):
        d = {n: 0.0 for n in names}
        nj = 0
        for j in range(1, 31):
            t = [buf[(c * 64 + j) * 8 + k] for k in range(8)]
            for k, n in enumerate(names):
                d[n] += t[k + 1] - t[k]
            nj += 1
        tot = sum(d.values())
        print(f"K-SQR {'first' if c == 0 else 'last'} CTA, rows={rows}: cycles per column " +
              ", ".join(f"{k} {v / nj:.0f}" for k, v in d.items()) + f" | total {tot / nj:.0f}")
        e = [buf[(c * 64 + 63) * 8 + k] for k in range(5)]
        print(f"   leaf: prologue {e[1] - e[0]}, column loop {e[2] - e[1]}, write-back {e[3] - e[2]}, "
              f"T (CTA 0) {e[4] - e[3]} cycles")


if __name__ == "__main__":
    main()
