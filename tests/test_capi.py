"""The C-ABI library builds, loads, and exports every entry point include/bqrrp.h declares (CPU-only)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bqrrp.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bqrrp_[a-z_0-9]+)\s*\(", src)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("bqrrp_factor", "bqrrp_factor_ex", "bqrrp_factor_host", "bqrrp_workspace_query",
                 "bqrrp_debug_sketch", "bqrrp_strerror"):
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2507_00976_b200 as bq
    from paper_2507_00976_b200 import build

    build.build()
    lib = bq.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.bqrrp_version()


def test_workspace_query_and_argument_checks_without_gpu():
    import paper_2507_00976_b200 as bq

    lib = bq.lib()
    n = bq.workspace_query(16384, 16384, 1024, 1024)
    assert n > 16384 * 1024 * 8 * 2
    out = ctypes.c_size_t(0)
    assert lib.bqrrp_workspace_query(-1, 4, 2, 2, ctypes.byref(out)) == -1
    assert lib.bqrrp_workspace_query(4, 4, 2, 1, ctypes.byref(out)) == -4  # d < b
    assert lib.bqrrp_workspace_query(4, 4, 2, 5, ctypes.byref(out)) == -4  # d > m
    # illegal arguments are rejected before any CUDA call (no device needed)
    rank = ctypes.c_int64(7)
    dummy = ctypes.c_void_p(16)
    st = lib.bqrrp_factor_ex(4, 4, dummy, 2, 2, 2, 0, dummy, dummy, ctypes.byref(rank), None, 0, None, None)
    assert st == -4  # lda < m
    st = lib.bqrrp_factor_ex(4, 4, dummy, 4, 0, 2, 0, dummy, dummy, ctypes.byref(rank), None, 0, None, None)
    assert st == -5  # b < 1
    assert lib.bqrrp_strerror(-5) == b"illegal argument"
    # K-NORM entries: argument checks first
    assert lib.bqrrp_column_norms(-1, 4, dummy, 4, dummy, None) == -1
    assert lib.bqrrp_column_norms(8, 4, dummy, 4, dummy, None) == -4  # lda < m
    assert lib.bqrrp_trailing_norms(8, 4, dummy, 8, None, None, 0, None) == -5
    assert lib.bqrrp_trailing_norms(8, 4, dummy, 8, dummy, dummy, 8, None) == -7  # workspace too small
    assert lib.bqrrp_trailing_norms_workspace(3000, 5000, ctypes.byref(out)) == 0
    assert out.value == 5 * 3000 * 8  # ceil(5000 / 1024) column chunks x min(m, n) rows of partial sums


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2507_00976_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "bqrrp_oracle" not in txt, f


def test_dist_entry_argument_checks_without_gpu():
    """The multi-GPU entries reject illegal arguments before any CUDA or NCCL call (LAPACK-style -i codes)."""
    from paper_2507_00976_b200.dist import _declare

    L = _declare()
    P = ctypes.c_void_p
    dummy = P(16)
    rank = ctypes.c_int64(0)
    h = P()
    assert L.bqrrp_comm_init(None, 0, 2, ctypes.byref(h)) == -1
    assert L.bqrrp_comm_init(dummy, 2, 2, ctypes.byref(h)) == -2
    assert L.bqrrp_comm_init_transport(None, ctypes.byref(h)) == -1
    assert L.bqrrp_comm_destroy(None) == 0
    args = (8, 8, dummy, 8, 2, 2, 0, dummy, dummy, ctypes.byref(rank))
    assert L.bqrrp_factor_dist(*args, None, None, 0, None, None) == -11  # no communicator
    out = ctypes.c_size_t(0)
    assert L.bqrrp_workspace_query_dist(64, 64, 8, 8, 2, 0, ctypes.byref(out)) == 0 and out.value > 0
    assert L.bqrrp_workspace_query_dist(64, 64, 8, 4, 2, 0, ctypes.byref(out)) == -4  # d < b
    n_loc = ctypes.c_int64(0)
    assert L.bqrrp_dist_local_columns(10, 0, 2, 0, ctypes.byref(n_loc)) == -2


def test_missing_library_fails_loudly(monkeypatch):
    """No CPU fallback: without the CUDA library the binding raises instead of computing anything."""
    import paper_2507_00976_b200 as bq

    monkeypatch.setattr(bq, "_lib", None)
    monkeypatch.setattr(bq, "_LIB_PATH", "/nonexistent/libbqrrp.so")
    with pytest.raises(ImportError):
        bq.lib()
    with pytest.raises(ImportError):
        bq.workspace_query(64, 64, 16, 16)


def test_options_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of bqrrp_options (the binding's Options) has the header's size and field offsets: a C
    program compiled against include/bqrrp.h prints them (gcc, no GPU)."""
    import shutil
    import subprocess

    import paper_2507_00976_b200 as bq

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    names = [f[0] for f in bq.Options._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"bqrrp.h\"\nint main(void) {\n"
                   "  printf(\"size %zu\\n\", sizeof(bqrrp_options));\n"
                   + "".join(f"  printf(\"{n} %zu\\n\", offsetof(bqrrp_options, {n}));\n" for n in names)
                   + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(root, "include"), str(src), "-o", str(exe)])
    out = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).splitlines())
    assert int(out["size"]) == ctypes.sizeof(bq.Options)
    for n in names:
        assert int(out[n]) == getattr(bq.Options, n).offset, n
