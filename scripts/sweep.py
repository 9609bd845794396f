#!/usr/bin/env python3
"""Sensitivity sweep with the reference bench CSV schema (tools/dilithium_cli.cpp:27-30,
352-357: schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,
mean_latency_us,attempts_mean) plus two columns (gpus, roofline_frac).  Reproduces the
paper's throughput-vs-batch-size and throughput-vs-Psi studies on B200
through the host-buffer C ABI (pinned buffers, transfers included, medians over reps).

usage: python scripts/sweep.py [--levels 2,3,5] [--phi 1000,10000,100000] [--psi 0,...] [--reps 7]
"""
import argparse, ctypes as C, sys, time
import numpy as np
sys.path.insert(0, ".")
import bench
from paper_2211_12265_b200 import Engine, LEVELS

ap = argparse.ArgumentParser()
ap.add_argument("--levels", default="2,3,5")
ap.add_argument("--phi", default="1000,10000,100000")
ap.add_argument("--psi", default="0")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
import torch
eng = Engine(0)
lib, ctx = eng.lib, eng.ctx
peak = eng.measure_int32_peak()["lop3"]
print("schema,mode,op,level,phi,psi,workers,streams,reps,throughput_ops_s,mean_latency_us,attempts_mean,gpus,roofline_frac")
u8 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint8))
u64 = lambda t: C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_uint64))
for level in [int(x) for x in args.levels.split(",")]:
    k, l, pkb, skb, sgb = LEVELS[level]
    wk = bench.WORK[level]
    pk1, sk1 = eng.batch_keygen(level, np.arange(32, dtype=np.uint8))
    for phi in [int(x) for x in args.phi.split(",")]:
        msgs, off = bench.make_inputs(phi, 1000 + level)   # 32-byte messages
        h_m = torch.from_numpy(msgs).pin_memory(); h_off = torch.from_numpy(off.astype(np.int64)).pin_memory()
        h_z = torch.from_numpy(bench.make_inputs(phi, 7)[0]).pin_memory()
        h_sk = torch.from_numpy(sk1[0].copy()).pin_memory(); h_pk = torch.from_numpy(pk1[0].copy()).pin_memory()
        h_sig = torch.zeros((phi, sgb), dtype=torch.uint8).pin_memory()
        h_pks = torch.zeros((phi, pkb), dtype=torch.uint8).pin_memory(); h_sks = torch.zeros((phi, skb), dtype=torch.uint8).pin_memory()
        h_fl = torch.zeros(phi, dtype=torch.uint8).pin_memory(); h_att = torch.zeros(phi, dtype=torch.int32).pin_memory()
        def run(fn):
            fn(); fn()
            ts = []
            for _ in range(args.reps):
                t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
            return float(np.median(ts))
        t = run(lambda: lib.dlb_keygen_batch(ctx, level, phi, u8(h_z), u8(h_pks), u8(h_sks)))
        print("1,batch-gpu,keygen,%d,%d,0,0,3,%d,%.1f,%.3f,,1,%.4f" % (level, phi, args.reps, phi / t, t / phi * 1e6, phi / t * bench.int_ops(wk["keygen"]) / 1e12 / peak))
        for psi in [int(x) for x in args.psi.split(",")]:
            t = run(lambda: lib.dlb_sign_batch(ctx, level, phi, u8(h_sk), 0, u8(h_m), u64(h_off), None, psi, 1, u8(h_sig), C.cast(C.c_void_p(h_att.data_ptr()), C.POINTER(C.c_uint32)), None, None))
            am = float(h_att.float().mean())
            print("1,batch-gpu,sign,%d,%d,%d,0,1,%d,%.1f,%.3f,%.3f,1,%.4f" % (level, phi, psi, args.reps, phi / t, t / phi * 1e6, am, phi / t * am * bench.int_ops(wk["attempt"]) / 1e12 / peak))
        t = run(lambda: lib.dlb_verify_batch(ctx, level, phi, u8(h_pk), 0, u8(h_m), u64(h_off), u8(h_sig), u8(h_fl)))
        assert bool(h_fl.all())
        print("1,batch-gpu,verify,%d,%d,0,0,3,%d,%.1f,%.3f,,1," % (level, phi, args.reps, phi / t, t / phi * 1e6))
