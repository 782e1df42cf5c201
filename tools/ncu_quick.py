"""Quick summary of an ncu report (run here, no GPU): key throughput metrics,
stall reasons per issue, and the top SASS lines by stall samples.
usage: python tools/ncu_quick.py REPORT.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, v = r[0], r[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_op_write.sum", "lts__t_sectors_op_read.sum"]
for k in keys:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
print("-- stalls per issue")
st = [(k, v[h.index(k)]) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
      and k.endswith("_per_issue_active.ratio")]
for k, x in sorted(st, key=lambda t: -float(t[1] or 0))[:10]:
    print(f"  {k[34:-27]:30s} {x}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
rows = r[2:]
i_s, i_src, i_ex = (h.index("Warp Stall Sampling (All Samples)"), h.index("Source"),
                    h.index("Instructions Executed"))
agg, cnt = collections.Counter(), collections.Counter()
for x in rows:
    ops = [o for o in x[i_src].split() if not o.startswith("@")]
    k = ops[0].split(".")[0] if ops else "?"
    agg[k] += int(x[i_s] or 0)
    cnt[k] += int(x[i_ex] or 0)
tot = sum(agg.values())
print(f"-- samples by opcode (total {tot})")
for k, n in agg.most_common(12):
    print(f"  {k:10s} {n:7d} ({100 * n / max(1, tot):4.1f}%)  executed {cnt[k]}")
print("-- top lines")
for x in sorted(rows, key=lambda x: -int(x[i_s] or 0))[:top]:
    print(f"  {x[i_s]:>6s}  {x[i_src][:90]}")

# stall reasons per opcode class (sampled), when the report has them
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
if cols:
    per = collections.defaultdict(collections.Counter)
    for x in rows:
        ops = [o for o in x[i_src].split() if not o.startswith("@")]
        k = ops[0].split(".")[0] if ops else "?"
        for c in cols:
            v_ = int(x[h.index(c)] or 0)
            if v_:
                per[c][k] += v_
    print("-- stall reason: top opcodes")
    for c in sorted(cols, key=lambda c: -sum(per[c].values()))[:8]:
        tot_c = sum(per[c].values())
        print(f"  {c:22s} {tot_c:6d}  " + ", ".join(f"{k} {n}" for k, n in per[c].most_common(4)))
