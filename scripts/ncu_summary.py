"""Summarise an ncu report: headline metrics, stall reasons, SASS opcode mix."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(raw))
d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
keys = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
for k in keys:
    if k in d: print(f"{k:70s} {d[k]}")
print("-- stalls per issued instruction")
for k, v in sorted(d.items()):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            if float(v) > 0.05: print(f"   {k[34:-23]:30s} {v}")
        except ValueError: pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(src)); hdr = rows[1]; data = rows[2:]
iS = hdr.index("Source"); iE = hdr.index("Instructions Executed"); iW = hdr.index("Warp Stall Sampling (All Samples)")
tot = collections.Counter(); st = collections.Counter()
for r in data:
    op = r[iS].strip().split()
    if not op: continue
    o = op[1] if op[0].startswith("@") else op[0]
    o = o.split(".")[0]
    tot[o] += int(r[iE] or 0); st[o] += int(r[iW] or 0)
T = sum(tot.values()); S = sum(st.values()) or 1
print(f"-- opcode mix (instructions {T}, stall samples {S})")
for o, c in tot.most_common(18):
    print(f"   {o:10s} {c:12d} {100*c/T:5.1f}%   stall {100*st[o]/S:5.1f}%")
