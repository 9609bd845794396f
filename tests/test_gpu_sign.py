"""Device parity of signing through the C ABI: single attempts (scheme.hpp:133-230),
whole signatures incl. attempt counts (scheme.hpp:253-273), batch_sign invariance under
(psi, speculate) (batch.hpp:46-49; tests/test_batch.cpp:190-228).  -m gpu."""
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
def test_kat_sign(eng, kat, level):
    sk = bytes.fromhex(kat["kKatSk%d" % level])
    msg = bytes.fromhex(kat["kKatMessage"])
    sig, att = eng.sign(level, sk, msg)
    assert sig.hex() == kat["kKatSig%d" % level]
    assert att == kat["kKatAttempts%d" % level]


@pytest.mark.parametrize("level", [2, 3, 5])
def test_sign_attempt_matches_oracle(eng, oracle, level):
    P = PARAMS[level]
    rng = mt19937_64(400 + level)
    n = 150
    _, sk = oracle.keygen(level, rng.bytes(32))
    mus = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    kappas = np.array([0, 65535 - P["l"] + 1, 65530] + [(int(rng()) % 3000) * P["l"] for _ in range(n - 3)], np.uint32)
    acc, ct, z, h = eng.dbg_sign_attempt(level, np.frombuffer(sk, np.uint8), mus, rps, kappas)
    n_acc = 0
    for t in range(n):
        ro, so, co, zo, ho = oracle.sign_attempt(level, sk, mus[t].tobytes(), rps[t].tobytes(), int(kappas[t]))
        assert acc[t] == ro, t
        assert ct[t].tobytes() == co, t
        if ro:
            n_acc += 1
            assert np.array_equal(z[t], zo) and np.array_equal(h[t], ho), t
    assert 0 < n_acc < n


@pytest.mark.parametrize("level,n", [(2, 300), (3, 120), (5, 100)])
def test_batch_sign_shared_key(eng, oracle, level, n):
    rng = mt19937_64(500 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    msgs = [rng.bytes(0 if i == 3 else 1 + int(rng()) % 200) for i in range(n)]
    exp = [oracle.sign(level, sk, m) for m in msgs]
    sk_arr = np.frombuffer(sk, np.uint8)
    sigs, att, failed, st = eng.batch_sign(level, sk_arr, msgs, return_info=True)
    for i in range(n):
        assert sigs[i].tobytes() == exp[i][0], i
        assert att[i] == exp[i][1], i
    assert not failed.any() and st["failed_tasks"] == 0
    assert st["accepted_attempt_sum"] == sum(e[1] for e in exp)
    assert st["attempts"] >= st["accepted_attempt_sum"]
    # output independent of slot count and speculation (batch.hpp:46-49)
    for psi, spec in [(128, True), (128, False), (1024, True), (100000, True), (0, False)]:
        s2, a2, f2, st2 = eng.batch_sign(level, sk_arr, msgs, psi=psi, speculate=spec, return_info=True)
        assert np.array_equal(s2, sigs) and np.array_equal(a2, att), (psi, spec)
        if not spec:
            assert st2["speculative"] == 0
            assert st2["attempts"] == st2["accepted_attempt_sum"]
    flags = eng.batch_verify(level, np.frombuffer(pk, np.uint8), msgs, sigs)
    assert flags.all()


@pytest.mark.parametrize("level,n", [(2, 60), (3, 30), (5, 24)])
def test_batch_sign_per_task_keys_and_override(eng, oracle, level, n):
    rng = mt19937_64(600 + level)
    keys = [oracle.keygen(level, rng.bytes(32)) for _ in range(n)]
    msgs = [rng.bytes(32) for _ in range(n)]
    sk_arr = np.frombuffer(b"".join(k[1] for k in keys), np.uint8).reshape(n, -1)
    sigs, att, failed, _ = eng.batch_sign(level, sk_arr, msgs, return_info=True)
    for i in range(n):
        assert (sigs[i].tobytes(), int(att[i])) == oracle.sign(level, keys[i][1], msgs[i]), i
    # randomised signing hook: explicit rho' (scheme.hpp:253-258, tests/test_scheme.cpp:110-123)
    rps = np.frombuffer(rng.bytes(64 * n), np.uint8).reshape(n, 64)
    sigs2, att2, _, _ = eng.batch_sign(level, sk_arr, msgs, rho_prime=rps, return_info=True)
    for i in range(n):
        assert (sigs2[i].tobytes(), int(att2[i])) == oracle.sign(level, keys[i][1], msgs[i], rps[i].tobytes()), i
    pk_arr = np.frombuffer(b"".join(k[0] for k in keys), np.uint8).reshape(n, -1)
    assert eng.batch_verify(level, pk_arr, msgs, sigs2).all()


def test_malformed_secret_key(eng, oracle):
    _, sk = oracle.keygen(2, bytes(32))
    bad = bytearray(sk)
    bad[96] = 0xFF
    with pytest.raises(ValueError):
        eng.sign(2, bytes(bad), b"m")


def test_config1_d2_1000_tasks(eng, ref):
    """BASELINE config 1: Dilithium2 keygen+sign+verify, 1,000 tasks, 32-byte messages,
    fixed seeds, deterministic signing -- byte for byte against the compiled reference."""
    level, n = 2, 1000
    rng = mt19937_64(20221112)
    zetas = np.frombuffer(rng.bytes(32 * n), np.uint8).reshape(n, 32)
    msgs = np.frombuffer(rng.bytes(32 * n), np.uint8)
    off = np.arange(n + 1, dtype=np.uint64) * 32
    pks, sks = eng.batch_keygen(level, zetas)
    rpk, rsk = ref.batch_keygen(level, zetas, workers=8)
    assert np.array_equal(pks, rpk) and np.array_equal(sks, rsk)
    # per-task keys
    sigs, att, failed, st = eng.batch_sign(level, sks, (msgs, off), return_info=True)
    rsigs, rst = ref.batch_sign(level, rsk, msgs, off, workers=8)
    assert np.array_equal(sigs, rsigs)
    assert st["accepted_attempt_sum"] == rst["accepted_attempt_sum"]
    flags = eng.batch_verify(level, pks, (msgs, off), sigs)
    assert flags.all()
    # shared key 0
    sigs0 = eng.batch_sign(level, sks[0], (msgs, off))
    rsigs0, _ = ref.batch_sign(level, rsk[0], msgs, off, workers=8)
    assert np.array_equal(sigs0, rsigs0)
    bad = sigs0.copy()
    bad[::7, 40] ^= 0x10
    f2 = eng.batch_verify(level, pks[0], (msgs, off), bad)
    assert np.array_equal(f2, ref.batch_verify(level, rpk[0], msgs, off, bad, workers=8))
    assert f2.sum() == n - len(range(0, n, 7))
