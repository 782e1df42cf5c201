"""Turns the round's ncu output (tools/profile_round.sh) into profiles/
summaries: the per-launch list of one VGG-16 b32 step with each kernel's
share, and the key `--set full` counters of the top conv kernels.

usage: python tools/ncu_summary.py gpurun_out/round profiles r2
(full captures are read from the .ncu-rep, or from the `--page raw --csv`
text export NAME.raw.csv plus NAME.src.csv that tools/profile_round.sh keeps)
"""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__cluster_dim_x",
    "launch__registers_per_thread",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def short(name: str) -> str:
    n = re.sub(r"\(.*", "", name)
    return n.split("::")[-1] if ("conv" in n or "pool" in n or "pack" in n) else n[:60]


def launches(src_csv: str):
    rows = [r for r in csv.reader(open(src_csv)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    out = []
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3,
                 "msecond": 1e3}.get(r[ix["Metric Unit"]], 1e-3)
        out.append((short(r[ix["Kernel Name"]]), float(r[ix["Metric Value"]]) * scale,
                    r[ix["Grid Size"]]))
    return out


def step_summary(ls, first="conv_first"):
    """The last complete step: launches between the last two first-layer
    launches (the final one belongs to the e2e/event passes)."""
    idx = [i for i, (n, _, _) in enumerate(ls) if n.startswith(first)]
    a, b = idx[-3], idx[-2]
    step = ls[a:b]
    tot = sum(t for _, t, _ in step)
    agg = defaultdict(lambda: [0, 0.0])
    for n, t, _ in step:
        k = next((p for p in ("conv_ffma_kernel", "conv_tf32x3_kernel", "conv_tf32_kernel")
                  if n.startswith(p)), n)
        agg[k][0] += 1
        agg[k][1] += t
    return {
        "step_launches": [{"kernel": n, "us": round(t, 2), "grid": g} for n, t, g in step],
        "step_us_serialised": round(tot, 1),
        "share_by_kernel": {k: {"launches": c, "us": round(t, 1), "share": round(t / tot, 4)}
                            for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])},
    }


def stall_by_opcode(src_csv: str, top: int = 4):
    """Sampled warp stalls of a capture's source page, per stall reason: the
    opcodes they sit on (e.g. long_scoreboard on the BRA of an mbarrier
    try_wait loop = a producer / epilogue warp idling, not the math warps)."""
    rows = list(csv.reader(open(src_csv)))
    h = rows[1]
    body = rows[2:]
    i_src = h.index("Source")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    per = defaultdict(lambda: defaultdict(int))
    for x in body:
        ops = [o for o in x[i_src].split() if not o.startswith("@")]
        k = ops[0].split(".")[0] if ops else "?"
        for c in cols:
            v = int(x[h.index(c)] or 0)
            if v:
                per[c][k] += v
    tot = sum(sum(d.values()) for d in per.values())
    out = {}
    for c in sorted(per, key=lambda c: -sum(per[c].values()))[:8]:
        n = sum(per[c].values())
        out[c] = {"share": round(n / tot, 3),
                  "top_opcodes": dict(sorted(per[c].items(), key=lambda kv: -kv[1])[:top])}
    return out


def full_metrics(rep: str):
    if rep.endswith(".raw.csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    d = {"Kernel Name": vals[h.index("Kernel Name")]}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            d[m] = f"{vals[i]} {units[i]}".strip()
    stalls = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")],
                               float(vals[i])))
            except ValueError:
                pass
    d["top_stalls_per_issue"] = sorted(stalls, key=lambda t: -t[1])[:8]
    src = rep.replace(".raw.csv", ".src.csv")
    if src != rep and os.path.exists(src):
        d["sampled_stalls_by_opcode"] = stall_by_opcode(src)
    return d


def find_rep(src: str, name: str):
    for ext in (".ncu-rep", ".raw.csv"):
        p = os.path.join(src, name + ext)
        if os.path.exists(p):
            return p
    return None


def main():
    src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    ls = launches(os.path.join(src, "launches_vgg16.csv"))
    summ = step_summary(ls, first="conv_reader")
    summ["source"] = ("ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 "
                      "python bench.py --steps 2 --warmup 3 --no-cpu-baseline (cold-cache, "
                      "serialised launches; the share is what must agree with bench.py)")
    json.dump(summ, open(os.path.join(dst, f"{tag}_ncu_launches_vgg16_b32.json"), "w"), indent=1)
    full = {}
    for name, rep in (("vgg16_conv1_2_b32", "full_conv1_2"),
                      ("vgg16_conv4_2_b32", "full_conv4_2"),
                      ("resnet50_1x1_64_256_skip_b256", "full_ffma_r50_s1c3"),
                      ("resnet50_1x1_256_1024_skip_b256", "full_ffma_r50_s3c3")):
        p = find_rep(src, rep)
        if p:
            full[name] = full_metrics(p)
    json.dump(full, open(os.path.join(dst, f"{tag}_ncu_full_conv_ffma.json"), "w"), indent=1)
    rd = {}
    for name, rep in (("vgg16_conv1_1_b32", "full_reader_conv1_1"),
                      ("googlenet_stem_7x7s2_b64", "full_reader_stem")):
        p = find_rep(src, rep)
        if p:
            rd[name] = full_metrics(p)
    if rd:
        json.dump(rd, open(os.path.join(dst, f"{tag}_ncu_full_conv_reader.json"), "w"), indent=1)
    x3 = {}
    for name, rep in (("vgg16_conv4_2_b32", "full_x3_conv4_2"),
                      ("resnet50_1x1_1024_256_b256", "full_x3_r50_1x1")):
        p = find_rep(src, rep)
        if p:
            x3[name] = full_metrics(p)
    if x3:
        json.dump(x3, open(os.path.join(dst, f"{tag}_ncu_full_conv_tf32x3.json"), "w"), indent=1)
    xl = os.path.join(src, "launches_vgg16_tf32x3.csv")
    if os.path.exists(xl):
        sx = step_summary(launches(xl), first="pack")
        sx["source"] = summ["source"].replace("--no-cpu-baseline", "--no-cpu-baseline --algo tf32x3")
        json.dump(sx, open(os.path.join(dst, f"{tag}_ncu_launches_vgg16_b32_tf32x3.json"), "w"),
                  indent=1)
        print(json.dumps(sx["share_by_kernel"], indent=1))
    print(json.dumps(summ["share_by_kernel"], indent=1))
    for k, v in full.items():
        print(k, {m: v.get(m) for m in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                        "dram__bytes_write.sum",
                                        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")})


if __name__ == "__main__":
    main()
