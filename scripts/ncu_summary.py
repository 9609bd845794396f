#!/usr/bin/env python3
"""Summarises an `ncu --set full` report into one row per kernel (first launch of each):
duration, registers, occupancy, issue / pipe utilisation, DRAM traffic.  Output: CSV +
markdown table.  usage: ncu_summary.py <report.ncu-rep> <out_prefix>"""
import csv, io, subprocess, sys, json

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
want = [
    ("time_us", "gpu__time_duration.sum"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("occ_theoretical_pct", "sm__maximum_warps_per_active_cycle_pct"),
    ("occ_achieved_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("fmaheavy_cycles_pct", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_gbs", "dram__bytes.sum.per_second"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("warp_insts", "smsp__inst_executed.sum"),
]
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3, "second": 1e6,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "byte/second": 1e-9, "Kbyte/second": 1e-6, "Mbyte/second": 1e-3, "Gbyte/second": 1.0, "Tbyte/second": 1e3,
         "byte/s": 1e-9, "Kbyte/s": 1e-6, "Mbyte/s": 1e-3, "Gbyte/s": 1.0, "Tbyte/s": 1e3}
seen, table = {}, []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("dlb::", "")
    key = name
    d = {"kernel": name, "launches": 1}
    for k, m in want:
        if m not in col:
            d[k] = None
            continue
        v = r[col[m]].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            d[k] = None
            continue
        u = units[col[m]]
        if k in ("time_us", "dram_read_bytes", "dram_write_bytes", "dram_gbs"):
            x *= scale.get(u, 1.0)
        d[k] = x
    if key in seen:  # keep the longest launch of each kernel (warm-up launches are tiny)
        d["launches"] = seen[key]["launches"] + 1
        if (d.get("time_us") or 0) < (seen[key].get("time_us") or 0):
            seen[key]["launches"] = d["launches"]
            continue
        table[table.index(seen[key])] = d
    else:
        table.append(d)
    seen[key] = d
keys = ["kernel", "launches"] + [k for k, _ in want]
with open(out + ".csv", "w") as f:
    w = csv.DictWriter(f, fieldnames=keys)
    w.writeheader()
    for d in table:
        w.writerow(d)
json.dump(table, open(out + ".json", "w"), indent=1)
with open(out + ".md", "w") as f:
    f.write("| kernel | time us | regs | occ ach % | issue % | alu pipe % | fma pipe % | lsu % | DRAM R+W MB | L2 hit % |\n|---|---|---|---|---|---|---|---|---|---|\n")
    for d in table:
        g = lambda k, fmt="%.1f": (fmt % d[k]) if d.get(k) is not None else "-"
        tr = ((d.get("dram_read_bytes") or 0) + (d.get("dram_write_bytes") or 0)) / 1e6
        f.write("| %s | %s | %s | %s | %s | %s | %s | %s | %.1f | %s |\n" % (
            d["kernel"][:60], g("time_us"), g("regs", "%d"), g("occ_achieved_pct"), g("issue_active_pct"),
            g("alu_pipe_pct"), g("fma_pipe_pct"), g("lsu_pipe_pct"), tr, g("l2_hit_pct")))
print(open(out + ".md").read())
