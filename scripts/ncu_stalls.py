#!/usr/bin/env python3
"""Per-stage warp-stall breakdown of a kernel from an `ncu --set full --import-source on` report:
the SASS (source page, address order) is split at block barriers, and for every region the
sampled warp states (stall_* columns) are summed.  Also prints the region's executed warp
instructions by pipe class.  usage: ncu_stalls.py <report.ncu-rep> [kernel substring] [min share %]"""
import csv, io, subprocess, sys, collections, re
rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
min_share = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
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
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
regions, cur = [], []
for d in body:
    cur.append(d)
    if "BAR.SYNC" in d["Source"] or "EXIT" in d["Source"]:
        regions.append(cur)
        cur = []
if cur:
    regions.append(cur)
f = lambda d, k: float(d[k] or 0)
tot_i = sum(f(d, "Instructions Executed") for d in body)
tot_s = sum(f(d, "# Samples") for d in body)
ALU = ("LOP3", "SHF", "IADD3", "VIADD", "VIADDMNMX", "ISETP", "SEL", "PRMT", "LEA", "IABS", "PLOP3", "FLO", "POPC", "BREV", "VIMNMX", "MOV")
FMA = ("IMAD",)
LSU = ("LDS", "STS", "LDG", "STG", "LD", "ST", "LDGSTS", "ATOMS", "ATOMG", "RED", "LDSM", "SHFL", "MATCH", "VOTE")


def pipe(op):
    base = op.split(".")[0]
    if base in FMA:
        return "fma(IMAD)"
    if base in ALU:
        return "alu"
    if base in LSU:
        return "lsu"
    return "other"


print("kernel %s: %.3e warp instructions, %d samples, %d SASS" % (kern, tot_i, tot_s, len(body)))
print("| region | SASS | inst %% | samples %% | inst / sample | pipes (inst %% of region) | top warp states (%% of region samples) |")
print("|---|---|---|---|---|---|---|")
for k, reg in enumerate(regions):
    ie = sum(f(d, "Instructions Executed") for d in reg)
    sm = sum(f(d, "# Samples") for d in reg)
    if 100 * ie / tot_i < min_share and 100 * sm / tot_s < min_share:
        continue
    st = collections.Counter()
    pp = collections.Counter()
    for d in reg:
        for c in stall_cols:
            st[c[6:]] += f(d, c)
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", d["Source"])
        pp[pipe(m.group(2) if m else "?")] += f(d, "Instructions Executed")
    ssum = sum(st.values()) or 1
    print("| %d | %d | %.1f | %.1f | %.0f | %s | %s |" % (
        k, len(reg), 100 * ie / tot_i, 100 * sm / tot_s, ie / max(sm, 1),
        ", ".join("%s %.0f" % (n, 100 * v / max(ie, 1)) for n, v in pp.most_common(4)),
        ", ".join("%s %.0f" % (n, 100 * v / ssum) for n, v in st.most_common(7))))
