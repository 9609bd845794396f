"""ctypes front ends for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

  Oracle  -- oracle/liboracle.so, the plain-C restatement (always available; built by
             __graft_entry__.build() / oracle/Makefile)
  Ref     -- oracle/_ref/libdilithium_ref.so, the unmodified reference headers
             compiled in place (prebuilt in the build container, travels to the GPU box)

Both expose the same Python surface so parity tests can be parametrised over them.
"""
import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")

# level -> (k, l, eta, tau, beta, gamma1, gamma2, omega, eta_bits, z_bits, w1_bits, pk, sk, sig)
PARAMS = {
    2: dict(k=4, l=4, eta=2, tau=39, beta=78, gamma1=1 << 17, gamma2=(8380417 - 1) // 88,
            omega=80, eta_bits=3, z_bits=18, w1_bits=6, pk=1312, sk=2528, sig=2420),
    3: dict(k=6, l=5, eta=4, tau=49, beta=196, gamma1=1 << 19, gamma2=(8380417 - 1) // 32,
            omega=55, eta_bits=4, z_bits=20, w1_bits=4, pk=1952, sk=4000, sig=3293),
    5: dict(k=8, l=7, eta=2, tau=60, beta=120, gamma1=1 << 19, gamma2=(8380417 - 1) // 32,
            omega=75, eta_bits=3, z_bits=20, w1_bits=4, pk=2592, sk=4864, sig=4595),
}
# FIPS 204 parameter sets (ML-DSA-44 / 65 / 87): same ring and bounds, 64-byte tr,
# lambda/4-byte commitment hash (oracle only: the compiled reference has no FIPS 204)
for _lv, _base, _sk, _sig, _ct in ((44, 2, 2560, 2420, 32), (65, 3, 4032, 3309, 48), (87, 5, 4896, 4627, 64)):
    PARAMS[_lv] = dict(PARAMS[_base], sk=_sk, sig=_sig, ct=_ct)
for _lv in (2, 3, 5):
    PARAMS[_lv]["ct"] = 32
Q = 8380417

_u8p = C.POINTER(C.c_uint8)


def _p(buf):
    """bytes / bytearray / uint8 ndarray -> c_uint8 pointer (no copy for ndarrays)."""
    if buf is None:
        return None
    if isinstance(buf, np.ndarray):
        assert buf.dtype == np.uint8 and buf.flags["C_CONTIGUOUS"]
        return buf.ctypes.data_as(_u8p)
    if isinstance(buf, bytearray):
        return (C.c_uint8 * len(buf)).from_buffer(buf)
    return C.cast(C.c_char_p(bytes(buf)), _u8p)


class mt19937_64:
    """std::mt19937_64, vectorised; bytes(n) == n x static_cast<uint8_t>(rng())
    (the reference tests' byte source, tests/acceptance.cpp:34-38)."""

    N, M = 312, 156

    def __init__(self, seed):
        x = [0] * self.N
        x[0] = seed & (2**64 - 1)
        for i in range(1, self.N):
            x[i] = (6364136223846793005 * (x[i - 1] ^ (x[i - 1] >> 62)) + i) & (2**64 - 1)
        self.x = np.array(x, dtype=np.uint64)
        self.buf = np.empty(0, dtype=np.uint64)

    def _twist(self):
        x, N, M = self.x, self.N, self.M
        UM, LM = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)
        A = np.uint64(0xB5026F5AA96619E9)

        def mix(cur, nxt, far):
            y = (cur & UM) | (nxt & LM)
            return far ^ (y >> np.uint64(1)) ^ np.where(y & np.uint64(1), A, np.uint64(0))

        x[0:M] = mix(x[0:M], x[1:M + 1], x[M:2 * M])
        x[M:N - 1] = mix(x[M:N - 1], x[M + 1:N], x[0:M - 1])
        x[N - 1:N] = mix(x[N - 1:N], x[0:1], x[M - 1:M])
        y = x.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        return y

    def words(self, n):
        while len(self.buf) < n:
            self.buf = np.concatenate([self.buf, self._twist()])
        out, self.buf = self.buf[:n], self.buf[n:]
        return out

    def __call__(self):
        return int(self.words(1)[0])

    def bytes(self, n):
        return self.words(n).astype(np.uint8).tobytes()


def mt_bytes(seed):
    rng = mt19937_64(seed)
    return rng.bytes


def build_checkers():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class _Checker:
    prefix = ""

    def __init__(self, lib):
        self.lib = lib
        f = self._f
        f("keccak_f1600", None, [C.POINTER(C.c_uint64)])
        for nm in ("shake128", "shake256"):
            f(nm, None, [_u8p, C.c_size_t, _u8p, C.c_size_t])
        i32p = C.POINTER(C.c_int32)
        f("expand_a", None, [i32p, _u8p, C.c_uint, C.c_uint])
        f("expand_s", None, [i32p, _u8p, C.c_uint, C.c_int])
        f("expand_mask", None, [i32p, _u8p, C.c_uint, C.c_int, C.c_int])
        f("sample_in_ball", None, [i32p, _u8p, C.c_int])
        f("ntt", None, [i32p])
        f("intt", None, [i32p])
        f("power2round", None, [C.c_int32, i32p, i32p])
        f("decompose", None, [C.c_int32, C.c_int32, i32p, i32p])
        f("make_hint", C.c_int, [C.c_int32, C.c_int32, C.c_int32])
        f("use_hint", C.c_int32, [C.c_int, C.c_int32, C.c_int32])
        f("keygen", C.c_int, [C.c_int, _u8p, _u8p, _u8p])
        f("sign", C.c_int, [C.c_int, _u8p, _u8p, C.c_size_t, _u8p, _u8p, C.POINTER(C.c_uint32)])
        f("verify", C.c_int, [C.c_int, _u8p, C.c_size_t, _u8p, C.c_size_t, _u8p, C.c_size_t])
        f("sign_attempt", C.c_int, [C.c_int, _u8p, _u8p, _u8p, C.c_uint32, C.POINTER(C.c_int),
                                    _u8p, i32p, i32p])
        f("sign_attempt_bounded", C.c_int, [C.c_int, _u8p, _u8p, _u8p, C.c_uint32, C.c_int32, C.c_int32,
                                            C.c_int32, C.POINTER(C.c_int), _u8p, i32p, i32p])

    def _f(self, name, res, args):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype, fn.argtypes = res, args
        setattr(self, "_" + name, fn)

    # ---- primitives
    def keccak_f1600(self, state):
        s = np.array(state, dtype=np.uint64).copy()
        self._keccak_f1600(s.ctypes.data_as(C.POINTER(C.c_uint64)))
        return s

    def shake(self, bits, data, outlen):
        out = np.zeros(outlen, dtype=np.uint8)
        fn = self._shake128 if bits == 128 else self._shake256
        fn(_p(out), outlen, _p(bytes(data)), len(data))
        return out.tobytes()

    def _poly(self, fn, *args):
        out = np.zeros(256, dtype=np.int32)
        fn(out.ctypes.data_as(C.POINTER(C.c_int32)), *args)
        return out

    def expand_a(self, rho, i, j):
        return self._poly(self._expand_a, _p(rho), i, j)

    def expand_s(self, rho_prime, nonce, eta):
        return self._poly(self._expand_s, _p(rho_prime), nonce, eta)

    def expand_mask(self, rho_prime, nonce, gamma1, z_bits):
        return self._poly(self._expand_mask, _p(rho_prime), nonce, gamma1, z_bits)

    def sample_in_ball(self, c_tilde, tau):
        return self._poly(self._sample_in_ball, _p(c_tilde), tau)

    def ntt(self, a):
        a = np.array(a, dtype=np.int32).copy()
        self._ntt(a.ctypes.data_as(C.POINTER(C.c_int32)))
        return a

    def intt(self, a):
        a = np.array(a, dtype=np.int32).copy()
        self._intt(a.ctypes.data_as(C.POINTER(C.c_int32)))
        return a

    def power2round(self, a):
        x, y = C.c_int32(), C.c_int32()
        self._power2round(a, C.byref(x), C.byref(y))
        return x.value, y.value

    def decompose(self, r, gamma2):
        x, y = C.c_int32(), C.c_int32()
        self._decompose(r, gamma2, C.byref(x), C.byref(y))
        return x.value, y.value

    def make_hint(self, z, r, gamma2):
        return self._make_hint(z, r, gamma2)

    def use_hint(self, h, r, gamma2):
        return self._use_hint(h, r, gamma2)

    # ---- scheme
    def keygen(self, level, zeta):
        P = PARAMS[level]
        pk, sk = np.zeros(P["pk"], np.uint8), np.zeros(P["sk"], np.uint8)
        rc = self._keygen(level, _p(bytes(zeta)), _p(pk), _p(sk))
        assert rc == 0
        return pk.tobytes(), sk.tobytes()

    def sign(self, level, sk, msg, rho_prime=None):
        P = PARAMS[level]
        sig = np.zeros(P["sig"], np.uint8)
        att = C.c_uint32(0)
        rc = self._sign(level, _p(bytes(sk)), _p(bytes(msg)), len(msg),
                        _p(bytes(rho_prime)) if rho_prime is not None else None, _p(sig),
                        C.byref(att))
        if rc != 0:
            raise ValueError("sign failed rc=%d" % rc)
        return sig.tobytes(), att.value

    def verify(self, level, pk, msg, sig):
        return self._verify(level, _p(bytes(pk)), len(pk), _p(bytes(msg)), len(msg),
                            _p(bytes(sig)), len(sig))

    def sign_attempt(self, level, sk, mu, rho_prime, kappa):
        P = PARAMS[level]
        z = np.zeros((P["l"], 256), np.int32)
        h = np.zeros((P["k"], 256), np.int32)
        ct = np.zeros(P["ct"], np.uint8)
        st = C.c_int(0)
        i32p = C.POINTER(C.c_int32)
        rc = self._sign_attempt(level, _p(bytes(sk)), _p(bytes(mu)), _p(bytes(rho_prime)), kappa,
                                C.byref(st), _p(ct), z.ctypes.data_as(i32p),
                                h.ctypes.data_as(i32p))
        return rc, st.value, ct.tobytes(), z, h


    def sign_attempt_bounded(self, level, sk, mu, rho_prime, kappa, z_bound, r0_bound, vt_bound):
        """detail::sign_attempt_bounded (scheme.hpp:133-219): (accepted, stage, c_tilde, z, hints)."""
        P = PARAMS[level]
        z = np.zeros((P["l"], 256), np.int32)
        h = np.zeros((P["k"], 256), np.int32)
        ct = np.zeros(P["ct"], np.uint8)
        st = C.c_int(0)
        i32p = C.POINTER(C.c_int32)
        rc = self._sign_attempt_bounded(level, _p(bytes(sk)), _p(bytes(mu)), _p(bytes(rho_prime)), kappa,
                                        z_bound, r0_bound, vt_bound, C.byref(st), _p(ct),
                                        z.ctypes.data_as(i32p), h.ctypes.data_as(i32p))
        return rc, st.value, ct.tobytes(), z, h


class Oracle(_Checker):
    def set_mldsa_context(self, ctx=b""):
        """FIPS 204 context string for levels 44 / 65 / 87 (oracle only)."""
        fn = self.lib.orc_set_mldsa_context
        fn.restype, fn.argtypes = C.c_int, [_u8p, C.c_size_t]
        assert fn(_p(bytes(ctx)) if ctx else None, len(ctx)) == 0

    prefix = "orc_"


    def set_mldsa_prehash(self, oid=b"", ctx=b""):
        """HashML-DSA mode of the oracle (FIPS 204 Alg. 4 / 5); an empty OID returns to pure ML-DSA."""
        fn = self.lib.orc_set_mldsa_prehash
        fn.restype, fn.argtypes = C.c_int, [_u8p, C.c_size_t, _u8p, C.c_size_t]
        assert fn(_p(bytes(ctx)) if ctx else None, len(ctx), _p(bytes(oid)) if oid else None, len(oid)) == 0


class RefStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("rounds", "attempts", "speculative", "idle_slot_rounds", "accepted_attempt_sum",
                 "failed")]


class Ref(_Checker):
    prefix = "ref_"

    def __init__(self, lib):
        super().__init__(lib)
        u64p = C.POINTER(C.c_uint64)
        self._f("hw_threads", C.c_int, [])
        self._f("batch_keygen", C.c_int, [C.c_int, C.c_size_t, _u8p, _u8p, _u8p, C.c_size_t])
        self._f("batch_sign", C.c_int, [C.c_int, C.c_size_t, _u8p, C.c_size_t, _u8p, u64p,
                                        C.c_size_t, C.c_size_t, C.c_int, _u8p,
                                        C.POINTER(RefStats)])
        self._f("batch_verify", C.c_int, [C.c_int, C.c_size_t, _u8p, C.c_size_t, _u8p, u64p, _u8p,
                                          C.c_size_t, C.c_size_t, _u8p])
        self._f("scheduler_replay", C.c_int, [C.c_size_t, C.c_size_t, C.c_uint32, C.c_int, _u8p,
                                              C.c_size_t, C.POINTER(C.c_int64), u64p])

    def hw_threads(self):
        return self._hw_threads()

    def batch_keygen(self, level, zetas, workers=1):
        P = PARAMS[level]
        zetas = np.ascontiguousarray(zetas, dtype=np.uint8).reshape(-1, 32)
        n = len(zetas)
        pks, sks = np.zeros((n, P["pk"]), np.uint8), np.zeros((n, P["sk"]), np.uint8)
        assert self._batch_keygen(level, n, _p(zetas), _p(pks), _p(sks), workers) == 0
        return pks, sks

    def batch_sign(self, level, sks, msgs, msg_off, psi=0, workers=1, speculate=True):
        """sks: (sk_bytes,) shared key or (n, sk_bytes); msgs: flat uint8; msg_off: n+1 u64."""
        P = PARAMS[level]
        sks = np.ascontiguousarray(sks, dtype=np.uint8)
        msg_off = np.ascontiguousarray(msg_off, dtype=np.uint64)
        msgs = np.ascontiguousarray(msgs, dtype=np.uint8)
        n = len(msg_off) - 1
        stride = 0 if sks.ndim == 1 else P["sk"]
        sigs = np.zeros((n, P["sig"]), np.uint8)
        st = RefStats()
        rc = self._batch_sign(level, n, _p(sks), stride, _p(msgs),
                              msg_off.ctypes.data_as(C.POINTER(C.c_uint64)), psi, workers,
                              1 if speculate else 0, _p(sigs), C.byref(st))
        assert rc == 0
        return sigs, {f[0]: getattr(st, f[0]) for f in RefStats._fields_}

    def batch_verify(self, level, pks, msgs, msg_off, sigs, workers=1):
        P = PARAMS[level]
        pks = np.ascontiguousarray(pks, dtype=np.uint8)
        sigs = np.ascontiguousarray(sigs, dtype=np.uint8)
        msgs = np.ascontiguousarray(msgs, dtype=np.uint8)
        msg_off = np.ascontiguousarray(msg_off, dtype=np.uint64)
        n = len(msg_off) - 1
        stride = 0 if pks.ndim == 1 else P["pk"]
        flags = np.zeros(n, np.uint8)
        rc = self._batch_verify(level, n, _p(pks), stride, _p(msgs),
                                msg_off.ctypes.data_as(C.POINTER(C.c_uint64)), _p(sigs), P["sig"],
                                workers, _p(flags))
        assert rc == 0
        return flags

    def scheduler_replay(self, phi, psi, ell, speculate, valid):
        valid = np.ascontiguousarray(valid, dtype=np.uint8)
        depth = valid.shape[1]
        acc = np.zeros(phi, np.int64)
        ex = C.c_uint64(0)
        self._scheduler_replay(phi, psi, ell, 1 if speculate else 0, _p(valid), depth,
                               acc.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(ex))
        return acc, ex.value


_cache = {}


def load_oracle():
    if "o" not in _cache:
        path = os.path.join(ORACLE_DIR, "liboracle.so")
        if not os.path.exists(path):
            build_checkers()
        _cache["o"] = Oracle(C.CDLL(path))
    return _cache["o"]


def ref_available():
    return os.path.exists(os.path.join(ORACLE_DIR, "_ref", "libdilithium_ref.so"))


def load_ref():
    if "r" not in _cache:
        path = os.path.join(ORACLE_DIR, "_ref", "libdilithium_ref.so")
        if not os.path.exists(path):
            build_checkers()
        _cache["r"] = Ref(C.CDLL(path))
    return _cache["r"]
