#!/usr/bin/env python3
"""Maps an ncu SASS source page to CUDA source lines (development aid).

usage: ncu_hot.py <report.ncu-rep> <object.o> <mangled kernel name> [top N] [launch id]
Joins `ncu --page source --csv` (per-SASS stall samples) with `nvdisasm -g` line info of
the same kernel (both list instructions in address order) and prints the hottest lines."""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis_all = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cubin)],
                         capture_output=True, text=True).stdout
dis, on = [], False
for l in dis_all.splitlines():
    if l.startswith("//---------------------"):
        on = (".text." + kern + " ") in l or l.rstrip("- ").endswith(".text." + kern)
        continue
    if on:
        dis.append(l)
dis = "\n".join(dis)
lines = []  # (file, line) per instruction in order
cur = ("?", 0)
for l in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+\S", l):
        lines.append((cur, l.strip()))
cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
if len(sys.argv) > 5:
    cmd += ["--launch-skip", sys.argv[5], "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# first kernel block matching the demangled name prefix
start = None
short = re.sub(r"^_ZN\d+dlb\d+", "", kern)[:12]
for i, r in enumerate(rows):
    if len(r) >= 2 and r[0] == "Kernel Name" and short[:8] in r[1].replace("::", ""):
        start = i
        break
if start is None:
    start = 0
hdr = rows[start + 1]
body = []
for r in rows[start + 2:]:
    if len(r) >= 2 and r[0] == "Kernel Name":
        break
    if len(r) == len(hdr):
        body.append(dict(zip(hdr, r)))
print("sass rows ncu=%d nvdisasm=%d" % (len(body), len(lines)))
n = min(len(body), len(lines))
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for i in range(n):
    d = body[i]
    key = lines[i][0]
    s = float(d.get("# Samples") or 0)
    ie = float(d.get("Instructions Executed") or 0)
    agg[key]["samples"] += s
    agg[key]["inst"] += ie
    tot["samples"] += s
    tot["inst"] += ie
    for h in stall_cols:
        v = float(d.get(h) or 0)
        agg[key][h] += v
        tot[h] += v
print("total samples %d, warp-instructions %d" % (tot["samples"], tot["inst"]))
print("stall mix: " + ", ".join("%s %.1f%%" % (h[6:], 100 * tot[h] / max(tot["samples"], 1))
                                for h in sorted(stall_cols, key=lambda h: -tot[h])[:9]))
byfile = collections.Counter()
for (f, l), c in agg.items():
    byfile[f] += c["samples"]
print("by file: " + ", ".join("%s %.1f%%" % (f, 100 * v / tot["samples"]) for f, v in byfile.most_common()))
for (f, l), c in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    tops = sorted(stall_cols, key=lambda h: -c[h])[:3]
    print("%5.1f%% smp %5.1f%% inst  %s:%d  [%s]" % (
        100 * c["samples"] / tot["samples"], 100 * c["inst"] / tot["inst"], f, l,
        ", ".join("%s %.0f%%" % (h[6:], 100 * c[h] / max(c["samples"], 1)) for h in tops)))
