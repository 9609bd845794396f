"""CPU-side checks of the drop-in boundary: the library builds, loads and exports every
symbol include/dilithium_b200.h declares; the C++ shim compiles; without a GPU the
product fails loudly instead of falling back.  No compute calls here."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__ as g
    g.build()
    from paper_2211_12265_b200 import load_library
    return load_library()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "dilithium_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    declared = sorted(set(re.findall(r"\b(dlb_[a-z0-9_]+)\s*\(", hdr)))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), "library does not export %s" % name
    from paper_2211_12265_b200.engine import EXPORTED_SYMBOLS
    assert sorted(EXPORTED_SYMBOLS) == declared


def test_no_oracle_in_product():
    """The product must not link or reference the CPU checkers."""
    so = os.path.join(ROOT, "paper_2211_12265_b200", "libdilithium_b200.so")
    out = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_" not in out
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2211_12265_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "liboracle" not in txt and "cpu_checkers" not in txt, f


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2211_12265_b200 import Engine, EngineError
    with pytest.raises(EngineError):
        Engine(0)
    ctx = C.c_void_p()
    assert lib.dlb_create(C.byref(ctx), 0, 0) < 0


def test_cpp_shim_compiles(lib):
    out = "/tmp/dlb_test_api"
    cmd = ["g++", "-std=c++20", "-O1", "-pthread", "-I" + os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), "-o", out,
           "-L" + os.path.join(ROOT, "paper_2211_12265_b200"), "-ldilithium_b200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2211_12265_b200")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_level_tables_agree():
    from paper_2211_12265_b200 import LEVELS
    from tests.cpu_checkers import PARAMS
    for lv, (k, l, pk, sk, sig) in LEVELS.items():
        P = PARAMS[lv]
        assert (k, l, pk, sk, sig) == (P["k"], P["l"], P["pk"], P["sk"], P["sig"])


def test_message_flattening():
    from paper_2211_12265_b200.engine import _msgs
    flat, off = _msgs([b"", b"abc", b"", b"de"])
    assert off.tolist() == [0, 0, 3, 3, 5] and flat.tobytes() == b"abcde"
    flat, off = _msgs([b""])
    assert off.tolist() == [0, 0] and flat.size >= 1


def test_sharding_partition_matches_reference_rule():
    from paper_2211_12265_b200.sharding import shard_ranges, chunk_ranges, slice_messages
    for n in (0, 1, 7, 10000, 1000003):
        for g in (1, 2, 4, 8):
            r = shard_ranges(n, g)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[i][1] == r[i + 1][0] for i in range(g - 1))
            assert all(lo == n * i // g for i, (lo, hi) in enumerate(r))  # tools/dilithium_cli.cpp:323
    assert chunk_ranges(3, 10, 4) == [(3, 7), (7, 10)]
    flat = np.arange(20, dtype=np.uint8)
    off = np.array([0, 2, 2, 9, 20], np.uint64)
    m, o = slice_messages(flat, off, 1, 3)
    assert o.tolist() == [0, 0, 7] and m.tolist() == list(range(2, 9))


def test_bench_work_model():
    import bench
    # D2 verify ~0.6 M int32 ops, sign attempt ~0.27-0.29 M
    assert 0.55e6 < bench.int_ops(bench.WORK[2]["verify"]) < 0.70e6
    assert 0.25e6 < bench.int_ops(bench.WORK[2]["attempt"]) < 0.30e6
    assert bench.WORK[2]["bytes"]["sign"] == 32 + 2420


def test_cli_argument_errors_need_no_gpu(lib):
    """tools/dilithium_b200 rejects bad command lines with exit code 2 before it ever creates an
    engine (proj/tests/test_cli.cpp:172-175: `keygen --pk a --sk b` without --level fails)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tools")], check=True)
    cli = os.path.join(ROOT, "tools", "dilithium_b200")
    for argv in (["keygen", "--pk", "a", "--sk", "b"], ["frobnicate"], [],
                 ["verify", "--level", "4", "--pk", "a", "--in", "b", "--sig", "c"],
                 ["sign", "--level", "2", "--sk", "a", "--in", "b"],
                 ["batch-sign", "--level", "2", "--sk", "a", "--out-dir", "d"],
                 ["keygen", "--level", "2", "--pk", "a", "--sk", "b", "--out-format", "base64"],
                 ["bench", "--level", "2", "--phi", "x"]):
        r = subprocess.run([cli, *argv], capture_output=True, text=True, timeout=60)
        assert r.returncode == 2 and "error:" in r.stderr, (argv, r.returncode, r.stderr)
