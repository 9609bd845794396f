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
