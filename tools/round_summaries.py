"""Derived summaries of a tools/profile_round.sh run (gpurun_out/round):
profiles/<tag>_scaling_per_rank_workloads.json (the batch-sharded configs at
the per-rank batch of 2 / 4 / 8 ranks) and profiles/<tag>_streamk_ab.json
(stream-K against full waves + split-K tail, same box).
usage: python tools/round_summaries.py [src] [dst] [tag]"""
import json
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/round"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles"
tag = sys.argv[3] if len(sys.argv) > 3 else "r2"


def load(f):
    for l in open(f):
        if l.startswith("{") and '"metric"' in l:
            return json.loads(l)
    raise SystemExit(f"no bench line in {f}")


d = load(f"{src}/bench_default.log")
r = [e for e in d["extra_configs"] if e["config"] == "resnet50" and e["global_batch"] == 256][0]
out = {"note": "Per-rank workloads of the batch-sharded configs on ONE B200 (gpurun has one GPU): "
               "the batch-sharded path has no collective, so N ranks run N of these side by side; "
               "aggregate = N x the per-rank rate, efficiency = per-rank rate at global_batch/N "
               "over the rate at the full batch. bench.py --gpus N runs the real thing (torchrun, "
               "NCCL barrier, max over ranks)."}
for key, head, cfg, batches in (("vgg16_global_batch_32", d, "vgg16", (16, 8, 4)),
                                ("resnet50_global_batch_256", r, "resnet50", (128, 64, 32))):
    base = head["value"]
    rows = {"1": {"per_rank_batch": batches[0] * 2, "gflops_per_rank": base,
                  "ms_per_step": head["ms_per_step"], "efficiency": 1.0}}
    for n, b in zip((2, 4, 8), batches):
        x = load(f"{src}/scale_{cfg}_b{b}.log")
        rows[str(n)] = {"per_rank_batch": b, "gflops_per_rank": x["value"],
                        "aggregate_gflops": round(x["value"] * n, 1),
                        "ms_per_step": x["ms_per_step"],
                        "efficiency": round(x["value"] / base, 3)}
    out[key] = rows
json.dump(out, open(f"{dst}/{tag}_scaling_per_rank_workloads.json", "w"), indent=1)
ab = {"note": "[us without stream-K, us with]; same box, same run of tools/profile_round.sh"}
for c, y in (("vgg16", d), ("resnet50", r)):
    x = load(f"{src}/nostreamk_{c}.log")
    ab[c] = {"stream_k": {"gflops": y["value"], "ffma_frac": y["roofline"]["frac"]},
             "waves_plus_split_tail (DCONV_NO_STREAMK=1)": {"gflops": x["value"],
                                                            "ffma_frac": x["roofline"]["frac"]},
             "layers_changed_over_1.5pct": {
                 a["name"]: [round(b["ms"] * 1e3, 1), round(a["ms"] * 1e3, 1)]
                 for a, b in zip(y["layers"], x["layers"])
                 if abs(a["ms"] - b["ms"]) / b["ms"] > 0.015}}
json.dump(ab, open(f"{dst}/{tag}_streamk_ab.json", "w"), indent=1)
for k in ("vgg16_global_batch_32", "resnet50_global_batch_256"):
    print(k, [(n, v["gflops_per_rank"], v["efficiency"]) for n, v in out[k].items()])
print({c: [ab[c]["stream_k"]["gflops"], ab[c]["waves_plus_split_tail (DCONV_NO_STREAMK=1)"]["gflops"]]
       for c in ("vgg16", "resnet50")})
