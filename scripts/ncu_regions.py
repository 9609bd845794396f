#!/usr/bin/env python3
"""Splits a kernel's SASS (ncu source page, address order) into regions between block
barriers and prints per-region executed warp-instructions, stall samples and opcode mix.
usage: ncu_regions.py <report.ncu-rep> [kernel substring] [top opcodes]"""
import csv, io, subprocess, sys, collections, re
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
start = 0
for i, r in enumerate(rows):
    if len(r) >= 2 and r[0] == "Kernel Name" and kern in r[1]:
        start = i
        break
hdr = rows[start + 1]
body = []
for r in rows[start + 2:]:
    if len(r) >= 2 and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        body.append(dict(zip(hdr, r)))
regions, cur = [], []
for d in body:
    cur.append(d)
    if "BAR.SYNC" in d["Source"] or "EXIT" in d["Source"]:
        regions.append(cur)
        cur = []
if cur:
    regions.append(cur)
tot_i = sum(float(d["Instructions Executed"] or 0) for d in body)
tot_s = sum(float(d["# Samples"] or 0) for d in body)
print("total warp-inst %.3e samples %d sass %d" % (tot_i, tot_s, len(body)))
for k, reg in enumerate(regions):
    ie = sum(float(d["Instructions Executed"] or 0) for d in reg)
    sm = sum(float(d["# Samples"] or 0) for d in reg)
    if ie / tot_i < 0.003 and sm / tot_s < 0.003:
        continue
    ops = collections.Counter()
    for d in reg:
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", d["Source"])
        op = m.group(2) if m else "?"
        op = ".".join(op.split(".")[:2]) if op.startswith(("IMAD", "LDG", "STG", "LDS", "STS")) else op.split(".")[0]
        ops[op] += float(d["Instructions Executed"] or 0)
    print("region %2d  sass %5d  addr %s  inst %5.1f%%  samples %5.1f%%  | %s" % (
        k, len(reg), reg[0]["Address"] if "Address" in reg[0] else "", 100 * ie / tot_i, 100 * sm / tot_s,
        ", ".join("%s %.1f" % (o, 100 * v / tot_i) for o, v in ops.most_common(topn))))
