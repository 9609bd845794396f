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


STAT_COUNTERS = ("rounds", "attempts", "speculative", "idle_slot_rounds", "accepted_attempt_sum", "failed_tasks")


def merge_shard_stats(stats, failed, ranges):
    """Per-shard sign statistics -> statistics of the whole batch (ShardedEngine::batch_sign in
    include/dilithium_b200/api.hpp): counters add up; each shard's failed-task indices (local to the
    shard) are rebased by the shard's first task.  stats: dict per shard; failed: iterable of local
    indices per shard; ranges: [(lo, hi)] of shard_ranges.  Returns (totals, failed indices)."""
    if not (len(stats) == len(failed) == len(ranges)):
        raise ValueError("one stats record, failed list and range per shard")
    total = {k: 0 for k in STAT_COUNTERS}
    out = []
    for st, fl, (lo, hi) in zip(stats, failed, ranges):
        for k in STAT_COUNTERS:
            total[k] += int(st.get(k, 0))
        for t in fl:
            if not 0 <= int(t) < hi - lo:
                raise IndexError("failed index %d outside its shard of %d tasks" % (t, hi - lo))
            out.append(lo + int(t))
    return total, out


def bind_to_device(device):
    """Pins the calling thread to the CPUs local to a GPU (dlb_bind_thread_to_device): host
    buffers it allocates afterwards are NUMA-local to that GPU.  True when the affinity was set."""
    from .engine import load_library
    return load_library().dlb_bind_thread_to_device(int(device)) == 0


class MultiEngine:
    """One Engine per device, one host thread per engine (bound to the GPU's NUMA node);
    outputs land in order."""

    def __init__(self, devices):
        from .engine import Engine
        self.devices = list(devices)
        self.engines = [None] * len(self.devices)

        def make(g):  # created by a bound thread: its pinned staging is first touched node-locally
            bind_to_device(self.devices[g])
            self.engines[g] = Engine(self.devices[g])

        ts = [threading.Thread(target=make, args=(g,)) for g in range(len(self.devices))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if any(e is None for e in self.engines):
            raise RuntimeError("engine creation failed on some device")

    def close(self):
        for e in self.engines:
            e.close()

    def _run(self, n, fn):
        ranges = shard_ranges(n, len(self.engines))
        errs = []

        def work(g):
            lo, hi = ranges[g]
            try:
                bind_to_device(self.devices[g])
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

    def batch_sign(self, level, sks, flat, off, chunk=65536, return_info=False, depth=16):
        """Every engine streams its shard as chunks in flight (sign_submit / sign_wait)."""
        from .engine import LEVELS
        n = len(off) - 1
        out = np.zeros((n, LEVELS[level][4]), np.uint8)
        att = np.zeros(n, np.uint32)
        sks = np.asarray(sks, np.uint8)
        ranges = shard_ranges(n, len(self.engines))
        shard_stats = [dict() for _ in self.engines]
        shard_failed = [[] for _ in self.engines]

        def fn(eng, lo, hi):
            g = self.engines.index(eng)
            tot = {k: 0 for k in STAT_COUNTERS}
            pending = []

            def finish(a, b, h):
                sg, at, fl, st = eng.sign_wait(h)
                out[a:b], att[a:b] = sg, at
                for k in STAT_COUNTERS:
                    tot[k] += st[k]
                shard_failed[g].extend((a - lo + np.nonzero(fl)[0]).tolist())

            for a, b in chunk_ranges(lo, hi, chunk):
                if len(pending) >= depth:
                    finish(*pending.pop(0))
                m, o = slice_messages(flat, off, a, b)
                pending.append((a, b, eng.sign_submit(level, sks if sks.ndim == 1 else sks[a:b], (m, o))))
            for p in pending:
                finish(*p)
            shard_stats[g] = tot

        self._run(n, fn)
        if return_info:
            total, failed = merge_shard_stats(shard_stats, shard_failed, ranges)
            return out, att, failed, total
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
