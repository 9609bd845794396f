"""Device parity of batched keygen and verify through the C ABI (host-buffer API)
against the CPU oracle / compiled reference.  -m gpu."""
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
def test_kat_keygen_verify(eng, kat, level):
    seed = bytes.fromhex(kat["kKatSeed"])
    msg = bytes.fromhex(kat["kKatMessage"])
    pk, sk = eng.keygen(level, seed)
    assert pk.hex() == kat["kKatPk%d" % level]
    assert sk.hex() == kat["kKatSk%d" % level]
    sig = bytes.fromhex(kat["kKatSig%d" % level])
    assert eng.verify(level, pk, msg, sig) == 1
    assert eng.verify(level, pk, msg + b"!", sig) == 0
    assert eng.verify(level, pk, msg, sig[:-1]) == 0


@pytest.mark.parametrize("level,n", [(2, 133), (3, 70), (5, 61)])
def test_batch_keygen_matches_oracle(eng, oracle, level, n):
    rng = mt19937_64(100 + level)
    zetas = np.frombuffer(rng.bytes(32 * n), np.uint8).reshape(n, 32)
    pks, sks = eng.batch_keygen(level, zetas)
    for i in range(n):
        pk, sk = oracle.keygen(level, zetas[i].tobytes())
        assert pks[i].tobytes() == pk, i
        assert sks[i].tobytes() == sk, i


@pytest.mark.parametrize("level,n", [(2, 96), (3, 48), (5, 40)])
def test_batch_verify_matches_oracle(eng, oracle, level, n):
    """Valid signatures, per-task keys, ragged messages (incl. empty), and every kind of
    corruption the reference's tests use: message/sig bit flips, hint-region edits
    (tests/test_scheme.cpp:73-108, tests/test_packing.cpp:111-184)."""
    P = PARAMS[level]
    rng = mt19937_64(200 + level)
    pks, sigs, msgs = [], [], []
    for i in range(n):
        pk, sk = oracle.keygen(level, rng.bytes(32))
        m = rng.bytes(0 if i == 0 else int(rng()) % 300)
        sig, _ = oracle.sign(level, sk, m)
        kind = i % 6
        if kind == 1:
            b = bytearray(sig); b[int(rng()) % len(b)] ^= 1 << (int(rng()) % 8); sig = bytes(b)
        elif kind == 2 and len(m):
            b = bytearray(m); b[int(rng()) % len(b)] ^= 1 << (int(rng()) % 8); m = bytes(b)
        elif kind == 3:
            b = bytearray(sig); b[-1 - int(rng()) % (P["omega"] + P["k"])] ^= 1 << (int(rng()) % 8); sig = bytes(b)
        elif kind == 4:
            b = bytearray(sig); off = 32 + int(rng()) % (P["l"] * 32 * P["z_bits"]); b[off] ^= 0x80; sig = bytes(b)
        pks.append(pk); sigs.append(sig); msgs.append(m)
    pk_arr = np.frombuffer(b"".join(pks), np.uint8).reshape(n, -1)
    sig_arr = np.frombuffer(b"".join(sigs), np.uint8).reshape(n, -1)
    flags = eng.batch_verify(level, pk_arr, msgs, sig_arr)
    expect = [oracle.verify(level, pks[i], msgs[i], sigs[i]) for i in range(n)]
    assert flags.tolist() == expect
    assert sum(expect) >= n // 6 and sum(expect) < n


@pytest.mark.parametrize("level", [2, 3, 5])
def test_batch_verify_shared_key(eng, oracle, level):
    rng = mt19937_64(300 + level)
    pk, sk = oracle.keygen(level, rng.bytes(32))
    n = 50
    msgs = [rng.bytes(32) for _ in range(n)]
    sigs = [oracle.sign(level, sk, m)[0] for m in msgs]
    sigs[7] = sigs[8]
    flags = eng.batch_verify(level, np.frombuffer(pk, np.uint8), msgs,
                             np.frombuffer(b"".join(sigs), np.uint8).reshape(n, -1))
    exp = [1] * n
    exp[7] = 0
    assert flags.tolist() == exp
