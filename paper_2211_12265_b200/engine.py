"""ctypes binding of libdilithium_b200.so, mirroring the reference's batch API
(proj/include/dilithium/batch.hpp:53-166: batch_keygen / batch_sign / batch_verify)
with numpy arrays in place of std::span / std::vector."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# level -> (k, l, pk_bytes, sk_bytes, sig_bytes)   (params.hpp:53-55,77-82)
LEVELS = {2: (4, 4, 1312, 2528, 2420), 3: (6, 5, 1952, 4000, 3293), 5: (8, 7, 2592, 4864, 4595),
          # ML-DSA-44 / 65 / 87 (FIPS 204; deterministic signing, empty context string)
          44: (4, 4, 1312, 2560, 2420), 65: (6, 5, 1952, 4032, 3309), 87: (8, 7, 2592, 4896, 4627)}

_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)


class EngineError(RuntimeError):
    pass


class SignStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("rounds", "attempts", "speculative", "idle_slot_rounds",
                                          "accepted_attempt_sum", "failed_tasks", "t_first_start_ns",
                                          "t_last_start_ns", "t_first_exit_ns", "t_last_exit_ns")]


def lib_path():
    # DLB_LIB selects an alternative build of the same library (A/B kernel experiments)
    return os.environ.get("DLB_LIB") or os.path.join(_HERE, "libdilithium_b200.so")


_lib = None


def load_library():
    """Loads the CUDA library; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise EngineError("libdilithium_b200.so not built: run `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (nvcc, sm_100a) -- there is no CPU fallback")
    lib = C.CDLL(path)
    vp = C.c_void_p
    sz = C.c_size_t
    sig = {
        "dlb_create": (C.c_int, [C.POINTER(vp), C.c_int, sz]),
        "dlb_destroy": (None, [vp]),
        "dlb_version": (C.c_char_p, []),
        "dlb_last_kernel_ms": (C.c_float, [vp]),
        "dlb_last_main_kernel_ms": (C.c_float, [vp]),
        "dlb_last_launches": (C.c_uint, [vp]),
        "dlb_set_stream": (C.c_int, [vp, vp]),
        "dlb_measure_int32_peak": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "dlb_measure_imad_hi_peak": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "dlb_set_mldsa_context": (C.c_int, [vp, _u8p, sz]),
        "dlb_set_mldsa_prehash": (C.c_int, [vp, _u8p, sz, _u8p, sz]),
        "dlb_set_trace": (C.c_int, [vp, sz]),
        "dlb_get_trace": (C.c_longlong, [vp, vp, sz]),
        "dlb_bind_thread_to_device": (C.c_int, [C.c_int]),
        "dlb_device_numa_node": (C.c_int, [C.c_int]),
        "dlb_host_alloc": (vp, [sz]),
        "dlb_host_free": (None, [vp]),
        "dlb_keygen_batch": (C.c_int, [vp, C.c_int, sz, _u8p, _u8p, _u8p]),
        "dlb_sign_batch": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u8p, _u64p, _u8p, sz, C.c_int,
                                     _u8p, _u32p, _u8p, C.POINTER(SignStats)]),
        "dlb_verify_batch": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u8p, _u64p, _u8p, _u8p]),
        "dlb_sign_batch_keyed": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u32p, _u8p, _u64p, _u8p, sz, C.c_int,
                                           _u8p, _u32p, _u8p, C.POINTER(SignStats)]),
        "dlb_verify_batch_keyed": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u32p, _u8p, _u64p, _u8p, _u8p]),
        "dlb_sign_batch_keyed_dev": (C.c_int, [vp, C.c_int, sz, vp, sz, vp, vp, vp, vp, sz, C.c_int, vp,
                                               vp, vp, C.POINTER(SignStats)]),
        "dlb_verify_batch_keyed_dev": (C.c_int, [vp, C.c_int, sz, vp, sz, vp, vp, vp, vp, vp]),
        "dlb_keygen_batch_dev": (C.c_int, [vp, C.c_int, sz, vp, vp, vp]),
        "dlb_sign_batch_dev": (C.c_int, [vp, C.c_int, sz, vp, sz, vp, vp, vp, sz, C.c_int, vp, vp,
                                         vp, C.POINTER(SignStats)]),
        "dlb_verify_batch_dev": (C.c_int, [vp, C.c_int, sz, vp, sz, vp, vp, vp, vp]),
        "dlb_dbg_keccak_f1600": (C.c_int, [vp, sz, _u64p]),
        "dlb_dbg_shake256": (C.c_int, [vp, sz, _u8p, _u64p, _u8p]),
        "dlb_dbg_expand_a": (C.c_int, [vp, C.c_int, sz, _u8p, _i32p]),
        "dlb_dbg_expand_s": (C.c_int, [vp, C.c_int, sz, _u8p, _i8p]),
        "dlb_dbg_expand_mask": (C.c_int, [vp, C.c_int, sz, _u8p, _u32p, _i32p]),
        "dlb_dbg_sample_in_ball": (C.c_int, [vp, C.c_int, sz, _u8p, _i8p]),
        "dlb_dbg_rounding": (C.c_int, [vp, C.c_int, C.c_int32, sz, _i32p]),
        "dlb_dbg_ntt": (C.c_int, [vp, sz, _i32p, C.c_int]),
        "dlb_dbg_sign_attempt": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u8p, _u8p, _u32p, _u8p,
                                           _u8p, _i32p, _i32p]),
        "dlb_dbg_sign_attempt_bounded": (C.c_int, [vp, C.c_int, sz, _u8p, sz, _u8p, _u8p, _u32p, C.c_int32,
                                                   C.c_int32, C.c_int32, _u8p, _u8p, _u8p, _i32p, _i32p]),
        "dlb_dbg_set_max_attempt": (C.c_int, [vp, C.c_uint]),
        "dlb_set_assignment_log": (C.c_int, [vp, sz]),
        "dlb_get_assignment_log": (C.c_longlong, [vp, vp, sz]),
        "dlb_sign_submit": (C.c_int, [vp, C.c_int, sz, vp, sz, sz, vp, vp, vp, vp, sz, C.c_int, vp, vp, vp,
                                      C.POINTER(C.c_uint64)]),
        "dlb_sign_submit_dev": (C.c_int, [vp, C.c_int, sz, vp, sz, sz, vp, vp, vp, vp, sz, C.c_int, vp, vp, vp,
                                          C.POINTER(C.c_uint64)]),
        "dlb_sign_wait": (C.c_int, [vp, C.c_uint64, C.POINTER(SignStats)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)  # AttributeError here = header/library mismatch
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


EXPORTED_SYMBOLS = [
    "dlb_create", "dlb_destroy", "dlb_version", "dlb_last_kernel_ms", "dlb_last_main_kernel_ms", "dlb_last_launches",
    "dlb_set_stream", "dlb_set_mldsa_context", "dlb_set_trace", "dlb_get_trace", "dlb_measure_int32_peak", "dlb_measure_imad_hi_peak", "dlb_host_alloc", "dlb_host_free", "dlb_keygen_batch", "dlb_sign_batch", "dlb_verify_batch",
    "dlb_sign_batch_keyed", "dlb_verify_batch_keyed", "dlb_sign_batch_keyed_dev", "dlb_verify_batch_keyed_dev",
    "dlb_keygen_batch_dev", "dlb_sign_batch_dev", "dlb_verify_batch_dev", "dlb_dbg_keccak_f1600",
    "dlb_dbg_shake256", "dlb_dbg_expand_a", "dlb_dbg_expand_s", "dlb_dbg_expand_mask",
    "dlb_dbg_sample_in_ball", "dlb_dbg_rounding", "dlb_dbg_ntt", "dlb_dbg_sign_attempt",
    "dlb_dbg_sign_attempt_bounded", "dlb_dbg_set_max_attempt", "dlb_set_assignment_log",
    "dlb_get_assignment_log", "dlb_sign_submit", "dlb_sign_submit_dev", "dlb_sign_wait",
    "dlb_bind_thread_to_device", "dlb_device_numa_node", "dlb_set_mldsa_prehash",
]


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(_u8p)


def _msgs(messages):
    """list of bytes | (flat uint8, offsets) -> (flat uint8 array, uint64 offsets[n+1])"""
    if isinstance(messages, tuple):
        flat, off = messages
        return np.ascontiguousarray(flat, np.uint8), np.ascontiguousarray(off, np.uint64)
    off = np.zeros(len(messages) + 1, np.uint64)
    off[1:] = np.cumsum([len(m) for m in messages])
    flat = np.frombuffer(b"".join(bytes(m) for m in messages), dtype=np.uint8).copy()
    if flat.size == 0:
        flat = np.zeros(1, np.uint8)
    return flat, off


class Engine:
    """One engine per GPU.  Methods mirror batch.hpp; inputs/outputs are numpy arrays of
    packed bytes exactly as the reference's PkBytes / SkBytes / SigBytes."""

    def __init__(self, device=0, max_batch=0):
        self.lib = load_library()
        self.ctx = C.c_void_p()
        rc = self.lib.dlb_create(C.byref(self.ctx), device, max_batch)
        if rc != 0:
            raise EngineError("dlb_create failed: %d (no GPU? there is no CPU fallback)" % rc)

    def close(self):
        if self.ctx:
            self.lib.dlb_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc, what):
        if rc != 0:
            raise EngineError("%s failed: status %d" % (what, rc))

    @property
    def last_kernel_ms(self):
        return float(self.lib.dlb_last_kernel_ms(self.ctx))

    @property
    def last_main_kernel_ms(self):
        return float(self.lib.dlb_last_main_kernel_ms(self.ctx))

    @property
    def last_launches(self):
        return int(self.lib.dlb_last_launches(self.ctx))

    def set_stream(self, handle):
        self._chk(self.lib.dlb_set_stream(self.ctx, C.c_void_p(handle)), "dlb_set_stream")

    def measure_int32_peak(self):
        out = (C.c_double * 4)()
        self._chk(self.lib.dlb_measure_int32_peak(self.ctx, out), "dlb_measure_int32_peak")
        hi = (C.c_double * 2)()
        self._chk(self.lib.dlb_measure_imad_hi_peak(self.ctx, hi), "dlb_measure_imad_hi_peak")
        return {"lop3": out[0], "imad": out[1], "shf": out[2], "lop3_imad_mix": out[3],
                "imad_hi": hi[0], "imad_wide": hi[1]}

    TRACE_FIELDS = ("stream", "round", "unfinished", "assigned", "speculative", "idle_slots", "newly_done")

    def set_trace(self, cap):
        """Per-round scheduler trace of the following sign calls (BatchConfig::trace); 0 = off."""
        self._chk(self.lib.dlb_set_trace(self.ctx, cap), "dlb_set_trace")
        self._trace_cap = cap

    def get_trace(self):
        """(records as an (m, 7) uint32 array in TRACE_FIELDS order, records produced)."""
        buf = np.zeros((max(1, getattr(self, "_trace_cap", 0)), 8), np.uint32)
        total = self.lib.dlb_get_trace(self.ctx, buf.ctypes.data_as(C.c_void_p), len(buf))
        if total < 0:
            raise EngineError("dlb_get_trace failed: %d" % total)
        return buf[:min(total, len(buf)), :7].copy(), int(total)

    ASSIGNMENT_FIELDS = ("slot", "task", "attempt", "kappa")

    def set_assignment_log(self, cap):
        """Log of executed (task, attempt) pairs of the following synchronous sign calls
        (BatchConfig::assignment_hook, batch.hpp:28); 0 = off."""
        self._chk(self.lib.dlb_set_assignment_log(self.ctx, cap), "dlb_set_assignment_log")
        self._alog_cap = cap

    def get_assignment_log(self):
        """(records as an (m, 4) uint32 array in ASSIGNMENT_FIELDS order, records produced)."""
        buf = np.zeros((max(1, getattr(self, "_alog_cap", 0)), 4), np.uint32)
        total = self.lib.dlb_get_assignment_log(self.ctx, buf.ctypes.data_as(C.c_void_p), len(buf))
        if total < 0:
            raise EngineError("dlb_get_assignment_log failed: %d" % total)
        return buf[:min(total, len(buf))].copy(), int(total)

    def dbg_set_max_attempt(self, max_attempt):
        """Stage tests: tasks whose attempts 0..max_attempt all fail are reported failed; 0 = scheme limit."""
        self._chk(self.lib.dlb_dbg_set_max_attempt(self.ctx, max_attempt), "dlb_dbg_set_max_attempt")

    def set_mldsa_context(self, context=b""):
        """FIPS 204 context string (<= 255 bytes) for levels 44 / 65 / 87; sticky, default empty."""
        buf = np.frombuffer(bytes(context), np.uint8)
        self._chk(self.lib.dlb_set_mldsa_context(self.ctx, buf.ctypes.data_as(_u8p) if len(buf) else None,
                                                 len(buf)), "dlb_set_mldsa_context")

    def set_mldsa_prehash(self, oid=b"", context=b""):
        """HashML-DSA (FIPS 204 Alg. 4 / 5): with a hash OID (DER bytes) the messages passed to sign /
        verify are the digests PH(M); an empty OID returns to pure ML-DSA."""
        cb = np.frombuffer(bytes(context), np.uint8)
        ob = np.frombuffer(bytes(oid), np.uint8)
        self._chk(self.lib.dlb_set_mldsa_prehash(self.ctx, cb.ctypes.data_as(_u8p) if len(cb) else None, len(cb),
                                                 ob.ctypes.data_as(_u8p) if len(ob) else None, len(ob)),
                  "dlb_set_mldsa_prehash")

    # ---- batch.hpp:159-166
    def batch_keygen(self, level, zetas):
        k, l, pkb, skb, sgb = LEVELS[level]
        z, zp = _u8(zetas)
        n = z.size // 32
        pks, sks = np.zeros((n, pkb), np.uint8), np.zeros((n, skb), np.uint8)
        self._chk(self.lib.dlb_keygen_batch(self.ctx, level, n, zp, pks.ctypes.data_as(_u8p),
                                            sks.ctypes.data_as(_u8p)), "dlb_keygen_batch")
        return pks, sks

    # ---- batch.hpp:53-137
    def batch_sign(self, level, sks, messages, rho_prime=None, psi=0, speculate=True,
                   return_info=False, key_idx=None):
        """sks: one key (1-D), one key per task (n x sk_bytes), or -- with key_idx -- a table
        of distinct keys (n_keys x sk_bytes) indexed per task (SignJob.key sharing,
        batch.hpp:41-44)."""
        k, l, pkb, skb, sgb = LEVELS[level]
        sk, skp = _u8(sks)
        flat, off = _msgs(messages)
        n = len(off) - 1
        stride = 0 if sk.ndim == 1 else skb
        kidx = None
        if key_idx is not None:
            kidx = np.ascontiguousarray(key_idx, np.uint32)
            if kidx.size != n or sk.size % skb:
                raise ValueError("key_idx / key table have the wrong size")
        elif sk.size != (skb if stride == 0 else n * skb):
            raise ValueError("secret key array has the wrong size")
        sigs = np.zeros((n, sgb), np.uint8)
        att = np.zeros(n, np.uint32)
        failed = np.zeros(n, np.uint8)
        st = SignStats()
        rp = None
        if rho_prime is not None:
            rpa, rp = _u8(rho_prime)
            assert rpa.size == n * 64
        if kidx is not None:
            rc = self.lib.dlb_sign_batch_keyed(self.ctx, level, sk.size // skb, skp, n,
                                               kidx.ctypes.data_as(_u32p), flat.ctypes.data_as(_u8p),
                                               off.ctypes.data_as(_u64p), rp, psi, 1 if speculate else 0,
                                               sigs.ctypes.data_as(_u8p), att.ctypes.data_as(_u32p),
                                               failed.ctypes.data_as(_u8p), C.byref(st))
        else:
            rc = self.lib.dlb_sign_batch(self.ctx, level, n, skp, stride, flat.ctypes.data_as(_u8p),
                                         off.ctypes.data_as(_u64p), rp, psi, 1 if speculate else 0,
                                         sigs.ctypes.data_as(_u8p), att.ctypes.data_as(_u32p),
                                         failed.ctypes.data_as(_u8p), C.byref(st))
        if rc == -3:
            raise ValueError("sign: malformed secret key")  # scheme.hpp:271
        self._chk(rc, "dlb_sign_batch")
        if return_info:
            return sigs, att, failed, {f[0]: getattr(st, f[0]) for f in SignStats._fields_}
        return sigs

    # ---- batches in flight (tools/dilithium_cli.cpp:309-345)
    def sign_submit(self, level, sks, messages, rho_prime=None, psi=0, speculate=True, key_idx=None,
                    out=None):
        """Enqueues a batch and returns a handle at once; sign_wait(handle) returns what
        batch_sign(..., return_info=True) would.  `out`: optional (n, sig_bytes) uint8 array
        for the signatures (e.g. pinned memory); inputs are kept alive by the handle."""
        k, l, pkb, skb, sgb = LEVELS[level]
        sk, skp = _u8(sks)
        flat, off = _msgs(messages)
        n = len(off) - 1
        stride = 0 if sk.ndim == 1 else skb
        kidx = None
        n_keys = 0
        if key_idx is not None:
            kidx = np.ascontiguousarray(key_idx, np.uint32)
            n_keys = sk.size // skb
            stride = skb
        sigs = out if out is not None else np.zeros((n, sgb), np.uint8)
        att = np.zeros(n, np.uint32)
        failed = np.zeros(n, np.uint8)
        rpa = None
        if rho_prime is not None:
            rpa = np.ascontiguousarray(rho_prime, np.uint8)
            assert rpa.size == n * 64
        ticket = C.c_uint64(0)
        vp = C.c_void_p
        rc = self.lib.dlb_sign_submit(self.ctx, level, n_keys, vp(sk.ctypes.data), stride, n,
                                      vp(kidx.ctypes.data) if kidx is not None else None,
                                      vp(flat.ctypes.data), vp(off.ctypes.data),
                                      vp(rpa.ctypes.data) if rpa is not None else None, psi,
                                      1 if speculate else 0, vp(sigs.ctypes.data), vp(att.ctypes.data),
                                      vp(failed.ctypes.data), C.byref(ticket))
        if rc == -3:
            raise ValueError("sign: malformed secret key")  # scheme.hpp:271
        self._chk(rc, "dlb_sign_submit")
        return {"ticket": ticket.value, "sigs": sigs, "att": att, "failed": failed,
                "keep": (sk, flat, off, kidx, rpa)}

    def sign_wait(self, handle):
        st = SignStats()
        rc = self.lib.dlb_sign_wait(self.ctx, handle["ticket"], C.byref(st))
        handle["keep"] = None
        if rc == -3:
            raise ValueError("sign: malformed secret key")
        self._chk(rc, "dlb_sign_wait")
        return (handle["sigs"], handle["att"], handle["failed"],
                {f[0]: getattr(st, f[0]) for f in SignStats._fields_})

    # ---- batch.hpp:148-156
    def batch_verify(self, level, pks, messages, sigs, key_idx=None):
        k, l, pkb, skb, sgb = LEVELS[level]
        pk, pkp = _u8(pks)
        sg, sgp = _u8(sigs)
        flat, off = _msgs(messages)
        n = len(off) - 1
        stride = 0 if pk.ndim == 1 else pkb
        flags = np.zeros(n, np.uint8)
        if key_idx is not None:
            kidx = np.ascontiguousarray(key_idx, np.uint32)
            if kidx.size != n or pk.size % pkb or sg.size != n * sgb:
                raise ValueError("key_idx / key table / sig arrays have the wrong size")
            self._chk(self.lib.dlb_verify_batch_keyed(self.ctx, level, pk.size // pkb, pkp, n,
                                                      kidx.ctypes.data_as(_u32p), flat.ctypes.data_as(_u8p),
                                                      off.ctypes.data_as(_u64p), sgp,
                                                      flags.ctypes.data_as(_u8p)), "dlb_verify_batch_keyed")
            return flags
        if sg.size != n * sgb or pk.size != (pkb if stride == 0 else n * pkb):
            raise ValueError("pk/sig arrays have the wrong size")
        self._chk(self.lib.dlb_verify_batch(self.ctx, level, n, pkp, stride,
                                            flat.ctypes.data_as(_u8p), off.ctypes.data_as(_u64p),
                                            sgp, flags.ctypes.data_as(_u8p)), "dlb_verify_batch")
        return flags

    # ---- scheme.hpp single-task forms, served by batches of one
    def keygen(self, level, zeta):
        pks, sks = self.batch_keygen(level, np.frombuffer(bytes(zeta), np.uint8))
        return pks[0].tobytes(), sks[0].tobytes()

    def sign(self, level, sk, msg, rho_prime=None):
        sigs, att, failed, _ = self.batch_sign(level, np.frombuffer(bytes(sk), np.uint8), [msg],
                                               rho_prime=rho_prime, return_info=True)
        return sigs[0].tobytes(), int(att[0])

    def verify(self, level, pk, msg, sig):
        k, l, pkb, skb, sgb = LEVELS[level]
        if len(pk) != pkb or len(sig) != sgb:  # scheme.hpp:280-283: wrong length rejects
            return 0
        return int(self.batch_verify(level, np.frombuffer(bytes(pk), np.uint8), [msg],
                                     np.frombuffer(bytes(sig), np.uint8).reshape(1, -1))[0])

    # ---- stage-level (device parity tests)
    def dbg_keccak_f1600(self, states):
        s = np.ascontiguousarray(states, np.uint64).reshape(-1, 25).copy()
        self._chk(self.lib.dlb_dbg_keccak_f1600(self.ctx, len(s), s.ctypes.data_as(_u64p)), "keccak")
        return s

    def dbg_shake256(self, messages):
        flat, off = _msgs(messages)
        n = len(off) - 1
        out = np.zeros((n, 64), np.uint8)
        self._chk(self.lib.dlb_dbg_shake256(self.ctx, n, flat.ctypes.data_as(_u8p),
                                            off.ctypes.data_as(_u64p), out.ctypes.data_as(_u8p)),
                  "shake256")
        return out

    def dbg_expand_a(self, level, rhos):
        k, l = LEVELS[level][:2]
        r, rp = _u8(rhos)
        n = r.size // 32
        out = np.zeros((n, k, l, 256), np.int32)
        self._chk(self.lib.dlb_dbg_expand_a(self.ctx, level, n, rp, out.ctypes.data_as(_i32p)), "expand_a")
        return out

    def dbg_expand_s(self, level, rho_primes):
        k, l = LEVELS[level][:2]
        r, rp = _u8(rho_primes)
        n = r.size // 64
        out = np.zeros((n, k + l, 256), np.int8)
        self._chk(self.lib.dlb_dbg_expand_s(self.ctx, level, n, rp, out.ctypes.data_as(_i8p)), "expand_s")
        return out

    def dbg_expand_mask(self, level, rho_primes, kappas):
        k, l = LEVELS[level][:2]
        r, rp = _u8(rho_primes)
        n = r.size // 64
        kap = np.ascontiguousarray(kappas, np.uint32)
        out = np.zeros((n, l, 256), np.int32)
        self._chk(self.lib.dlb_dbg_expand_mask(self.ctx, level, n, rp, kap.ctypes.data_as(_u32p),
                                               out.ctypes.data_as(_i32p)), "expand_mask")
        return out

    def dbg_sample_in_ball(self, level, c_tildes):
        r, rp = _u8(c_tildes)
        n = r.size // 32
        out = np.zeros((n, 256), np.int8)
        self._chk(self.lib.dlb_dbg_sample_in_ball(self.ctx, level, n, rp, out.ctypes.data_as(_i8p)), "sib")
        return out

    def dbg_rounding(self, gamma2_divisor, first, n):
        """(p2r_hi, p2r_lo, dec_hi, dec_lo, use_hint0, use_hint1) for first .. first+n-1."""
        out = np.zeros((6, n), np.int32)
        self._chk(self.lib.dlb_dbg_rounding(self.ctx, gamma2_divisor, first, n, out.ctypes.data_as(_i32p)),
                  "rounding")
        return out

    def dbg_ntt(self, polys, inverse=False):
        p = np.ascontiguousarray(polys, np.int32).reshape(-1, 256).copy()
        self._chk(self.lib.dlb_dbg_ntt(self.ctx, len(p), p.ctypes.data_as(_i32p), int(inverse)), "ntt")
        return p

    def dbg_sign_attempt(self, level, sks, mus, rho_primes, kappas):
        k, l, pkb, skb, sgb = LEVELS[level]
        sk, skp = _u8(sks)
        mu, mup = _u8(mus)
        rp, rpp = _u8(rho_primes)
        kap = np.ascontiguousarray(kappas, np.uint32)
        n = kap.size
        stride = 0 if sk.ndim == 1 else skb
        acc = np.zeros(n, np.uint8)
        ct = np.zeros((n, {65: 48, 87: 64}.get(level, 32)), np.uint8)  # lambda/4 bytes at the FIPS 204 levels
        z = np.zeros((n, l, 256), np.int32)
        h = np.zeros((n, k, 256), np.int32)
        self._chk(self.lib.dlb_dbg_sign_attempt(self.ctx, level, n, skp, stride, mup, rpp,
                                                kap.ctypes.data_as(_u32p), acc.ctypes.data_as(_u8p),
                                                ct.ctypes.data_as(_u8p), z.ctypes.data_as(_i32p),
                                                h.ctypes.data_as(_i32p)), "sign_attempt")
        return acc, ct, z, h

    REJECT_STAGES = ("ZNorm", "R0Norm", "VtNorm", "HintWeight")  # scheme.hpp:34

    def dbg_sign_attempt_bounded(self, level, sks, mus, rho_primes, kappas, z_bound, r0_bound, vt_bound):
        """detail::sign_attempt_bounded (scheme.hpp:133-219): (accepted, stage, c_tilde, z, hints);
        stage 255 = accepted, else an index into REJECT_STAGES."""
        k, l, pkb, skb, sgb = LEVELS[level]
        sk, skp = _u8(sks)
        mu, mup = _u8(mus)
        rp, rpp = _u8(rho_primes)
        kap = np.ascontiguousarray(kappas, np.uint32)
        n = kap.size
        stride = 0 if sk.ndim == 1 else skb
        acc = np.zeros(n, np.uint8)
        stage = np.zeros(n, np.uint8)
        ct = np.zeros((n, {65: 48, 87: 64}.get(level, 32)), np.uint8)
        z = np.zeros((n, l, 256), np.int32)
        h = np.zeros((n, k, 256), np.int32)
        self._chk(self.lib.dlb_dbg_sign_attempt_bounded(
            self.ctx, level, n, skp, stride, mup, rpp, kap.ctypes.data_as(_u32p), z_bound, r0_bound,
            vt_bound, acc.ctypes.data_as(_u8p), stage.ctypes.data_as(_u8p), ct.ctypes.data_as(_u8p),
            z.ctypes.data_as(_i32p), h.ctypes.data_as(_i32p)), "sign_attempt_bounded")
        return acc, stage, ct, z, h
