#!/usr/bin/env python3
"""Per barrier-delimited region: executed warp-instructions by source line (joins ncu's SASS
page with nvdisasm -g line info).  usage: ncu_region_lines.py rep obj mangled region_idx [top]"""
import csv, io, os, re, subprocess, sys, tempfile, collections
rep, obj, kern, ridx = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis_all = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)], capture_output=True, text=True).stdout
lines, on, cur = [], False, ("?", 0)
for l in dis_all.splitlines():
    if l.startswith("//---------------------"):
        on = (".text." + kern + " ") in l
        continue
    if not on: continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
        lines.append(cur)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
want = "k_sign_persistent" if "k_sign_persistent" in kern else ""
start = 0
for i, r in enumerate(rows):  # the report may hold several kernels: pick the matching block
    if len(r) >= 2 and r[0] == "Kernel Name" and want in r[1]:
        start = i
        break
hdr = rows[start + 1]
body = []
for r in rows[start + 2:]:
    if len(r) >= 2 and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        body.append(dict(zip(hdr, r)))
assert len(body) == len(lines), (len(body), len(lines))
tot = sum(float(d["Instructions Executed"] or 0) for d in body)
reg = 0
agg = collections.Counter(); ops = collections.defaultdict(collections.Counter)
for d, ln in zip(body, lines):
    if reg == ridx:
        ie = float(d["Instructions Executed"] or 0)
        agg[ln] += ie
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_.]+)", d["Source"])
        ops[ln][m.group(2) if m else "?"] += ie
    if "BAR.SYNC" in d["Source"] or "EXIT" in d["Source"]:
        reg += 1
s = sum(agg.values())
print("region %d: %.1f%% of all instructions" % (ridx, 100 * s / tot))
for ln, v in agg.most_common(top):
    print("%5.2f%%  %s:%d   %s" % (100 * v / tot, ln[0], ln[1], ", ".join("%s %.2f" % (o, 100 * x / tot) for o, x in ops[ln].most_common(4))))
