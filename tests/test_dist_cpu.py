"""N > 1 path on CPU: two gloo ranks through bench.py's Dist plumbing, and the
--impl reference contract under torchrun (rank 0 prints, the others exit 0 silently)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(nproc, port, script_args, timeout=300):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
           "--master-addr", "127.0.0.1", "--master-port", str(port)] + script_args
    env = dict(os.environ, OMP_NUM_THREADS="1")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def test_two_rank_gloo_plumbing(tmp_path):
    r = _torchrun(2, 29631, [os.path.join(ROOT, "tests", "dist_worker.py"), str(tmp_path)])
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(line) == 1
    out = json.loads(line[0])
    assert out == {"t_max": 11.0, "total": 1001.0, "world": 2}
    a = json.load(open(tmp_path / "rank0.json"))
    b = json.load(open(tmp_path / "rank1.json"))
    assert a["lo"] == 0 and a["hi"] == b["lo"] and b["hi"] == 1001
    assert a["first"] != b["first"]  # ranks draw different synthetic shards


def test_three_rank_uneven_shards_merge(tmp_path):
    """Three ranks over 1001 tasks (333 / 334 / 334): the real partition, and the stats and
    failed-index rebasing that ShardedEngine (C++) and MultiEngine (Python) apply, through gloo."""
    r = _torchrun(3, 29635, [os.path.join(ROOT, "tests", "dist_worker.py"), str(tmp_path)])
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert out == {"t_max": 12.0, "total": 1001.0, "world": 3}
    shards = [json.load(open(tmp_path / ("rank%d.json" % g))) for g in range(3)]
    assert [(s["lo"], s["hi"]) for s in shards] == [(0, 333), (333, 667), (667, 1001)]
    m = json.load(open(tmp_path / "merged.json"))
    assert m["stats"] == {"rounds": 33, "attempts": 6000, "speculative": 21, "idle_slot_rounds": 3,
                          "accepted_attempt_sum": 5400, "failed_tasks": 6}
    assert m["failed"] == [0, 332, 333, 666, 667, 1000]  # shard-local first / last, rebased


def test_shard_helpers_cpp_and_python():
    """The C++ partition / merge helpers (api.hpp) against the Python ones, no GPU involved."""
    from paper_2211_12265_b200.sharding import merge_shard_stats, shard_ranges
    exe = "/tmp/dlb_shard_cpu"
    lib = os.path.join(ROOT, "paper_2211_12265_b200")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "test_shard_cpu.cpp"), "-o", exe, "-L" + lib,
                        "-ldilithium_b200", "-Wl,-rpath," + lib], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "all passed" in r.stdout, r.stdout + r.stderr
    assert shard_ranges(1001, 3) == [(0, 333), (333, 667), (667, 1001)]
    assert shard_ranges(2, 5) == [(0, 0), (0, 0), (0, 1), (1, 1), (1, 2)]  # more shards than tasks
    tot, failed = merge_shard_stats([{"attempts": 5}, {"attempts": 7}], [[1], [0, 2]], [(0, 2), (2, 5)])
    assert tot["attempts"] == 12 and failed == [1, 2, 4]
    with pytest.raises(IndexError):
        merge_shard_stats([{}, {}], [[2], []], [(0, 2), (2, 5)])


def test_reference_arm_under_torchrun():
    r = _torchrun(2, 29633, [os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                             "--steps", "1", "--warmup", "0", "--tasks", "64"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["metric"] == "dilithium2_sign_ops_per_s"
    assert out["value"] > 0 and out["cpu_baseline"]["kind"] in ("reference", "port")
    assert out["e2e"]["h2d_bytes_per_step"] == 0
