"""Edge cases the reference's tests cover for this path (tests/test_batch.cpp:190-297,
tests/test_scheme.cpp:73-202, tests/test_keccak.cpp:78-95): empty and single-task batches,
empty and multi-block messages, 16-bit nonce wrap, duplicate tasks, device-resident API.
-m gpu."""
import ctypes as C

import numpy as np
import pytest

from tests.cpu_checkers import PARAMS, mt19937_64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2211_12265_b200 import Engine
    e = Engine(0)
    yield e
    e.close()


@pytest.mark.parametrize("level", [2, 3, 5])
def test_empty_and_single(eng, oracle, level):
    P = PARAMS[level]
    pks, sks = eng.batch_keygen(level, np.zeros((0, 32), np.uint8))
    assert pks.shape == (0, P["pk"]) and sks.shape == (0, P["sk"])
    pk, sk = oracle.keygen(level, bytes(32))
    assert eng.batch_sign(level, np.frombuffer(sk, np.uint8), []).shape == (0, P["sig"])
    assert eng.batch_verify(level, np.frombuffer(pk, np.uint8), [], np.zeros((0, P["sig"]), np.uint8)).shape == (0,)
    sig, att = eng.sign(level, sk, b"")
    assert (sig, att) == oracle.sign(level, sk, b"")
    assert eng.verify(level, pk, b"", sig) == 1


@pytest.mark.parametrize("level", [2, 5])
def test_long_and_block_boundary_messages(eng, oracle, level):
    """mu = H(tr || M): message lengths around the SHAKE256 rate (136 - 32 = 104 first block)."""
    rng = mt19937_64(1234 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    lens = [0, 1, 103, 104, 105, 239, 240, 241, 376, 1000, 4096, 10001]
    msgs = [rng.bytes(n) for n in lens]
    sk_a, pk_a = np.frombuffer(sk, np.uint8), np.frombuffer(pk, np.uint8)
    sigs, att, _, _ = eng.batch_sign(level, sk_a, msgs, return_info=True)
    for i, m in enumerate(msgs):
        assert (sigs[i].tobytes(), int(att[i])) == oracle.sign(level, sk, m), lens[i]
    assert eng.batch_verify(level, pk_a, msgs, sigs).all()
    wrong = [m + b"\x00" for m in msgs]
    assert not eng.batch_verify(level, pk_a, wrong, sigs).any()


def test_duplicate_tasks_and_determinism(eng, oracle):
    level = 2
    pk, sk = oracle.keygen(level, bytes(range(32)))
    msgs = [b"same message"] * 257 + [b"other"]
    sigs = eng.batch_sign(level, np.frombuffer(sk, np.uint8), msgs)
    assert all(sigs[i].tobytes() == sigs[0].tobytes() for i in range(257))
    assert sigs[0].tobytes() == oracle.sign(level, sk, msgs[0])[0]
    assert sigs[257].tobytes() != sigs[0].tobytes()


@pytest.mark.parametrize("level", [2, 3, 5])
def test_nonce_wrap_single_attempts(eng, oracle, level):
    """kappa + j is truncated to 16 bits (scheme.hpp:143): attempts near 65535."""
    P = PARAMS[level]
    rng = mt19937_64(77 + level)
    _, sk = oracle.keygen(level, rng.bytes(32))
    n = 40
    mus = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    kappas = np.array([65535 - i for i in range(n)], np.uint32)
    acc, ct, z, h = eng.dbg_sign_attempt(level, np.frombuffer(sk, np.uint8), mus, rps, kappas)
    for t in range(n):
        ro, so, co, zo, ho = oracle.sign_attempt(level, sk, mus[t].tobytes(), rps[t].tobytes(), int(kappas[t]))
        assert acc[t] == ro and ct[t].tobytes() == co
        if ro:
            assert np.array_equal(z[t], zo) and np.array_equal(h[t], ho)


def test_device_resident_api_matches_host_api(eng, oracle):
    """dlb_*_batch_dev on caller-owned device buffers (torch) == host-buffer API."""
    import torch
    from paper_2211_12265_b200 import LEVELS
    from paper_2211_12265_b200.engine import SignStats
    level, n = 3, 777
    k, l, pkb, skb, sgb = LEVELS[level]
    rng = mt19937_64(99)
    zetas = np.frombuffer(rng.bytes(32 * n), np.uint8).reshape(n, 32).copy()
    msgs = np.frombuffer(rng.bytes(32 * n), np.uint8).copy()
    off = np.arange(n + 1, dtype=np.uint64) * 32
    pks, sks = eng.batch_keygen(level, zetas)
    sigs = eng.batch_sign(level, sks, (msgs, off))
    dev = torch.device("cuda:0")
    p = lambda t: C.c_void_p(t.data_ptr())
    d_z = torch.from_numpy(zetas).to(dev)
    d_pk = torch.empty((n, pkb), dtype=torch.uint8, device=dev)
    d_sk = torch.empty((n, skb), dtype=torch.uint8, device=dev)
    assert eng.lib.dlb_keygen_batch_dev(eng.ctx, level, n, p(d_z), p(d_pk), p(d_sk)) == 0
    assert np.array_equal(d_pk.cpu().numpy(), pks) and np.array_equal(d_sk.cpu().numpy(), sks)
    d_m = torch.from_numpy(msgs).to(dev)
    d_off = torch.from_numpy(off.astype(np.int64)).to(dev)
    d_sig = torch.zeros((n, sgb), dtype=torch.uint8, device=dev)
    d_att = torch.zeros(n, dtype=torch.int32, device=dev)
    d_fail = torch.zeros(n, dtype=torch.uint8, device=dev)
    st = SignStats()
    rc = eng.lib.dlb_sign_batch_dev(eng.ctx, level, n, p(d_sk), skb, p(d_m), p(d_off), None, 0, 1,
                                    p(d_sig), p(d_att), p(d_fail), C.byref(st))
    assert rc == 0 and np.array_equal(d_sig.cpu().numpy(), sigs)
    d_fl = torch.zeros(n, dtype=torch.uint8, device=dev)
    assert eng.lib.dlb_verify_batch_dev(eng.ctx, level, n, p(d_pk), pkb, p(d_m), p(d_off), p(d_sig), p(d_fl)) == 0
    assert bool(d_fl.all().item())
    # an external stream can drive the device-resident calls
    s = torch.cuda.Stream()
    eng.set_stream(s.cuda_stream)
    assert eng.lib.dlb_verify_batch_dev(eng.ctx, level, n, p(d_pk), pkb, p(d_m), p(d_off), p(d_sig), p(d_fl)) == 0
    eng.set_stream(0)
    assert bool(d_fl.all().item())


@pytest.mark.parametrize("level", [2, 3, 5, 65])
def test_hint_section_every_byte(eng, oracle, level):
    """Strict hint decoding (packing.hpp:122-140; tests/test_packing.cpp:111-184): every byte
    of the hint section of a valid signature is replaced by a few values -- out-of-order
    positions, counts that shrink / exceed omega, non-zero slack -- and the device verdict
    must equal the oracle's for each mutant."""
    P = PARAMS[level]
    rng = mt19937_64(6100 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    msg = rng.bytes(40)
    sig = np.frombuffer(oracle.sign(level, sk, msg)[0], np.uint8)
    hint0 = P["sig"] - (P["omega"] + P["k"])
    mutants = []
    for pos in range(hint0, P["sig"]):
        for val in (0, 1, 255, (int(sig[pos]) + 1) & 255, (int(sig[pos]) - 1) & 255, P["omega"], P["omega"] + 1):
            if val != sig[pos]:
                m = sig.copy()
                m[pos] = val
                mutants.append(m)
    mutants = np.stack(mutants)
    n = len(mutants)
    flags = eng.batch_verify(level, np.frombuffer(pk, np.uint8), [msg] * n, mutants)
    expect = np.array([oracle.verify(level, pk, msg, m.tobytes()) for m in mutants], np.uint8)
    assert np.array_equal(flags, expect)
    assert expect.sum() < n // 4  # nearly every mutation must be fatal


def test_random_batch_shapes(eng, oracle):
    """acceptance.cpp:186-244 / test_batch.cpp:190-228: random (level, Phi, Psi, speculate)
    batches are byte-identical to sequential signing whatever the slot count."""
    rng = mt19937_64(55)
    keys = {lv: oracle.keygen(lv, rng.bytes(32)) for lv in (2, 3, 5)}
    for it in range(36):
        level = (2, 3, 5)[it % 3]
        phi = 1 + int(rng()) % 160
        psi = 1 + int(rng()) % phi if it % 4 else 0
        spec = bool(int(rng()) & 1)
        pk, sk = keys[level]
        msgs = [rng.bytes(int(rng()) % 64) for _ in range(phi)]
        sigs, att, failed, st = eng.batch_sign(level, np.frombuffer(sk, np.uint8), msgs, psi=psi,
                                               speculate=spec, return_info=True)
        assert not failed.any()
        for i in range(phi):
            assert (sigs[i].tobytes(), int(att[i])) == oracle.sign(level, sk, msgs[i]), (it, level, phi, psi, spec, i)
        assert st["accepted_attempt_sum"] == int(att.sum()) and st["attempts"] >= st["accepted_attempt_sum"]
        if not spec:
            assert st["speculative"] == 0


@pytest.mark.parametrize("level,n,psi,spec", [(2, 3000, 0, True), (3, 700, 512, False), (5, 90, 0, True), (2, 40000, 0, True)])
def test_round_trace_accounts_for_every_attempt(eng, level, n, psi, spec):
    """BatchConfig::trace (batch.hpp:27,114; RoundTrace scheduler.hpp:21-28): the per-round
    records of all CTAs add up to the batch statistics, every CTA's rounds are numbered
    0, 1, 2, ... and every task is reported done exactly once."""
    rng = mt19937_64(7300 + n)
    pk, sk = eng.keygen(level, rng.bytes(32))
    msgs = np.frombuffer(rng.bytes(32 * n), np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * 32
    ref_sigs = eng.batch_sign(level, np.frombuffer(sk, np.uint8), (msgs, off), psi=psi, speculate=spec)
    eng.set_trace(1 << 18)
    try:
        sigs, att, failed, st = eng.batch_sign(level, np.frombuffer(sk, np.uint8), (msgs, off), psi=psi,
                                               speculate=spec, return_info=True)
        recs, total = eng.get_trace()
    finally:
        eng.set_trace(0)
    assert np.array_equal(sigs, ref_sigs)  # tracing never changes an output
    assert total == len(recs) == st["rounds"]
    f = {name: recs[:, i].astype(np.int64) for i, name in enumerate(eng.TRACE_FIELDS)}
    assert f["assigned"].sum() == st["attempts"] and f["speculative"].sum() == st["speculative"]
    assert f["idle_slots"].sum() == st["idle_slot_rounds"] and f["newly_done"].sum() == n
    assert (f["assigned"] >= np.minimum(f["unfinished"], 1)).all() and (f["newly_done"] <= f["unfinished"]).all()
    if not spec:
        assert (f["speculative"] == 0).all() and (f["assigned"] <= f["unfinished"]).all()
    for s in np.unique(f["stream"]):
        rounds = np.sort(f["round"][f["stream"] == s])
        assert np.array_equal(rounds, np.arange(len(rounds)))
