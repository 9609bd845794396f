"""Contiguous sharding of a task batch over the GPUs of one box.

The path has no exchange step: every task is a pure function of its own inputs, so a
batch is cut into contiguous ranges lo = n*g/G, hi = n*(g+1)/G exactly as the reference's
multi-engine mode does (tools/dilithium_cli.cpp:319-339), one engine (one process or one
host thread) per GPU, results written to disjoint output ranges.  No collective, no NCCL.
"""
import threading

import numpy as np


def shard_ranges(n, parts):
    """[(lo, hi)] with lo = n*g//parts -- identical to the reference CLI's partition."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    return [(n * g // parts, n * (g + 1) // parts) for g in range(parts)]


def chunk_ranges(lo, hi, chunk):
    """Sub-ranges of at most `chunk` tasks for streamed execution."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    return [(a, min(a + chunk, hi)) for a in range(lo, hi, chunk)]


def slice_messages(flat, off, lo, hi):
    """Messages lo..hi of a CSR-style (flat, off) pair, re-based to offset 0."""
    off = np.asarray(off, dtype=np.uint64)
    base = int(off[lo])
    return np.ascontiguousarray(flat[base:int(off[hi])]), (off[lo:hi + 1] - np.uint64(base))


class MultiEngine:
    """One Engine per device, one host thread per engine; outputs land in order."""

    def __init__(self, devices):
        from .engine import Engine
        self.engines = [Engine(d) for d in devices]

    def close(self):
        for e in self.engines:
            e.close()

    def _run(self, n, fn):
        ranges = shard_ranges(n, len(self.engines))
        errs = []

        def work(g):
            lo, hi = ranges[g]
            try:
                if hi > lo:
                    fn(self.engines[g], lo, hi)
            except Exception as e:  # surfaced to the caller like WorkerPool::parallel_for
                errs.append(e)

        ts = [threading.Thread(target=work, args=(g,)) for g in range(len(self.engines))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]

    def batch_sign(self, level, sks, flat, off, chunk=65536):
        from .engine import LEVELS
        n = len(off) - 1
        out = np.zeros((n, LEVELS[level][4]), np.uint8)
        sks = np.asarray(sks, np.uint8)

        def fn(eng, lo, hi):
            for a, b in chunk_ranges(lo, hi, chunk):
                m, o = slice_messages(flat, off, a, b)
                out[a:b] = eng.batch_sign(level, sks if sks.ndim == 1 else sks[a:b], (m, o))

        self._run(n, fn)
        return out

    def batch_verify(self, level, pks, flat, off, sigs, chunk=65536):
        n = len(off) - 1
        out = np.zeros(n, np.uint8)
        pks = np.asarray(pks, np.uint8)

        def fn(eng, lo, hi):
            for a, b in chunk_ranges(lo, hi, chunk):
                m, o = slice_messages(flat, off, a, b)
                out[a:b] = eng.batch_verify(level, pks if pks.ndim == 1 else pks[a:b], (m, o), sigs[a:b])

        self._run(n, fn)
        return out

    def batch_keygen(self, level, zetas, chunk=65536):
        from .engine import LEVELS
        zetas = np.asarray(zetas, np.uint8).reshape(-1, 32)
        n = len(zetas)
        pks = np.zeros((n, LEVELS[level][2]), np.uint8)
        sks = np.zeros((n, LEVELS[level][3]), np.uint8)

        def fn(eng, lo, hi):
            for a, b in chunk_ranges(lo, hi, chunk):
                pks[a:b], sks[a:b] = eng.batch_keygen(level, zetas[a:b])

        self._run(n, fn)
        return pks, sks
