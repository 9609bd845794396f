"""Large randomised parity run against the UNMODIFIED reference (oracle/_ref, all host
threads): keys, signatures and verdicts byte for byte, every task, not a sample.

  python scripts/parity_campaign.py [tasks per level, default 200000] [seed]

Per level: `keys` random key pairs (GPU batch_keygen vs reference batch_keygen), then the
tasks spread over those keys with message lengths 0..300 (GPU mixed-key batch_sign vs the
reference's per-task-key batch_sign), then verification of the signatures with 2 % random
single-bit corruptions (GPU mixed-key batch_verify vs the reference's batch_verify).
This script is a checker (tests/ territory); it is not part of the product path."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2211_12265_b200 import Engine, LEVELS
from tests.cpu_checkers import load_ref

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20221112
keys = 64
ref = load_ref()
cores = max(1, ref.hw_threads())
eng = Engine(0)
total = 0
for level in (2, 3, 5):
    rs = np.random.default_rng(seed + level)
    k, l, pkb, skb, sgb = LEVELS[level]
    zetas = rs.integers(0, 256, (keys, 32), dtype=np.uint8)
    t0 = time.time()
    pks, sks = eng.batch_keygen(level, zetas)
    rpk, rsk = ref.batch_keygen(level, zetas, workers=cores)
    assert np.array_equal(pks, rpk) and np.array_equal(sks, rsk), "keygen mismatch"
    nk = min(n, 200000)  # key generation at scale
    zk = rs.integers(0, 256, (nk, 32), dtype=np.uint8)
    gpk, gsk = eng.batch_keygen(level, zk)
    cpk, csk = ref.batch_keygen(level, zk, workers=cores)
    assert np.array_equal(gpk, cpk) and np.array_equal(gsk, csk), "keygen mismatch (bulk)"
    lens = rs.integers(0, 301, n)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    flat = rs.integers(0, 256, int(off[-1]) + 1, dtype=np.uint8)
    kidx = rs.integers(0, keys, n).astype(np.uint32)
    sigs, att, failed, st = eng.batch_sign(level, sks, (flat, off), key_idx=kidx, return_info=True)
    assert not failed.any()
    rsig, rst = ref.batch_sign(level, sks[kidx], flat, off, workers=cores)
    bad_sig = np.flatnonzero((sigs != rsig).any(axis=1))
    assert bad_sig.size == 0, "sign mismatch at tasks %s" % bad_sig[:10]
    assert int(att.sum()) == int(st["accepted_attempt_sum"])
    victims = rs.choice(n, n // 50, replace=False)
    bad = sigs.copy()
    bad[victims, rs.integers(0, sgb, victims.size)] ^= (1 << rs.integers(0, 8, victims.size)).astype(np.uint8)
    flags = eng.batch_verify(level, pks, (flat, off), bad, key_idx=kidx)
    rflags = ref.batch_verify(level, pks[kidx], flat, off, bad, workers=cores)
    assert np.array_equal(flags, rflags), "verify mismatch"
    assert flags.sum() == n - victims.size
    total += n
    print("Dilithium%d: %d + %d keys, %d signatures (mean attempts %.3f), %d verdicts (%d corrupted, all rejected) "
          "identical to the reference; %.1f s" % (level, keys, nk, n, att.mean(), n, victims.size, time.time() - t0),
          flush=True)
print("parity campaign: %d tasks per op, 0 mismatches (reference on %d host threads)" % (total, cores))
