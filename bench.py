#!/usr/bin/env python
"""Benchmark of the direct-convolution hot path (BASELINE.json metric:
"direct-conv GFLOP/s per layer & % of B200 FP32 (TF32) peak, zero workspace").

Default workload: BASELINE configs[2], the VGG-16 chain (13 x 3x3 convs +
ReLU + 4 max-pools, every activation in the blocked layout), global batch 32,
fp32, batch-sharded over the ranks with no collective.  One *step* = one pass
of the whole chain over the batch.  `--config` selects the other configs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config vgg16]
  python bench.py --impl reference ...      # CPU reference arm

One JSON line on rank 0.  `value` = whole-job GFLOP/s with inputs resident in
HBM (CUDA-graph replay, CUDA events, max over ranks); `e2e` = the same work
through the public API with the input batch copied H2D from pinned memory and
the network output copied D2H inside the timed region; `roofline` = the FFMA
direct-conv kernel's achieved FLOP/s (algorithmic conv_flops / its average
launch duration, CUDA events on its stream) over the FP32 FFMA peak measured
live on this GPU; `cpu_baseline` = the restated reference algorithm (Alg. 3,
oracle/oracle.c) on the host cores over a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "direct-conv GFLOP/s per layer & % of B200 FP32 (TF32) peak, zero workspace"
DEFAULT_BATCH = {"cfg1": 1, "alexnet": 1, "vgg16": 32, "googlenet": 64, "resnet50": 256}
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.45 at clocks.max.sm


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg16", choices=sorted(DEFAULT_BATCH))
    ap.add_argument("--batch", type=int, default=0, help="global batch (0 = config default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-tune", action="store_true",
                    help="skip the per-layer CTA-tile autotune at plan build")
    ap.add_argument("--algo", default="ffma", choices=["ffma", "tf32", "tf32x3"],
                    help="ffma: the fp32 FFMA path (the headline); tf32: stride-1 layers on "
                         "the tcgen05/TMEM TF32 variant (reduced precision, reported apart)")
    ap.add_argument("--shard", default="batch", choices=["batch", "co"],
                    help="batch: image ranges per rank, no collective; co: batch-1 "
                         "output-block sharding with an NCCL all-gather per layer")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer"],
                    help="--shard co exchange: nccl all-gather of slices, or peer = each "
                         "conv/pool epilogue stores into every rank's map over NVLink "
                         "(symmetric memory) + a device barrier")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="target CPU work for the cpu_baseline sample")
    return ap.parse_args()


# ------------------------------------------------------------------ CPU arm
def cpu_reference(config: str, steps: int, warmup: int, budget_s: float):
    """Restated reference Alg. 3 (oracle/oracle.c conv_direct: j' parallel,
    i', l, k', n, m, ii, kk, jj; AVX2 tile kernels) on every host core, one
    image of the workload through every layer of the config per sample."""
    import numpy as np

    from oracle import pyoracle as po  # CPU baseline leg only
    from paper_1809_10170_b200 import nets

    layers = nets.CONFIGS[config]
    threads = os.cpu_count() or 1
    data = []
    for idx, l in enumerate(layers):
        cib = l.c_i if l.first else 8
        xb = po.pack_feature_map(po.uniform((l.c_i, l.h_i, l.w_i), 1809, 2 * idx), cib)
        kb = po.pack_kernel(po.uniform((l.c_i, l.c_o, l.h_f, l.w_f), 1809, 1000 + 2 * idx),
                            8, cib)
        data.append((l, xb, kb))
    flops = sum(l.flops for l in layers)

    def one():
        t0 = time.perf_counter()
        for l, xb, kb in data:
            po.conv_direct(xb, kb, l.c_i, l.c_o, l.s, w_ob=14, threads=threads)
        return time.perf_counter() - t0

    times = [one() for _ in range(max(1, warmup))]
    per = statistics.median(times)
    n_samples = max(1, min(steps, int(budget_s / max(per, 1e-6))))
    times = [one() for _ in range(n_samples)]
    t = statistics.median(times)
    return {
        "value": flops / t / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
        "sample": (f"1 image of {config} ({len(layers)} layers, {flops / 1e9:.2f} GFLOP) "
                   f"through restated Alg. 3 (oracle/oracle.c, c_ob=8 w_ob=14 AVX2 tile, "
                   f"OpenMP over j'), median of {len(times)} after warm-up; "
                   f"reference's own conv_direct is absent from the snapshot"),
        "seconds_per_sample": t,
    }


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cb = cpu_reference(args.config, args.steps, args.warmup, 1e9)
    batch = args.batch or DEFAULT_BATCH[args.config]
    line = {
        "metric": METRIC, "impl": "reference", "value": round(cb["value"], 2),
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(cb["seconds_per_sample"] * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} chain, 1-image sample of the b{batch} job",
                   "global_batch": batch, "c_b": 8},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": round(cb["value"], 2), "unit": "GFLOP/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # NVML absent: report nulls
            self.nv = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                bits = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def tf32_gemm_peak(stream) -> float:
    """TF32 tensor-core roofline denominator: cuBLAS TF32 GEMM (8192^3),
    best of 5, CUDA events (same convention as MEASURED_PEAKS.json's bf16)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        with torch.cuda.stream(stream):
            a = torch.randn(8192, 8192, device="cuda")
            b = torch.randn(8192, 8192, device="cuda")
            best = 0.0
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                torch.matmul(a, b)
                e1.record(stream)
                e1.synchronize()
                best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        del a, b
        return best
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


# ------------------------------------------------------------------ GPU arm
def main_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_1809_10170_b200 import _abi, nets

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    co_shard = args.shard == "co"
    if world > 1 or co_shard:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", local))
    lib = _abi.lib()
    batch = args.batch or DEFAULT_BATCH[args.config]
    if co_shard:
        batch = args.batch or 1
        if batch != 1:
            raise SystemExit("--shard co is the batch-1 mode")
        n_local = 1
        args.no_graph = True  # NCCL collectives stay outside graph capture
    else:
        if batch % world:
            raise SystemExit(f"global batch {batch} not divisible by {world} ranks")
        n_local = batch // world  # batch sharding: contiguous image range per rank

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        plan = nets.build_plan(args.config, n_local, seed=1809 + (0 if co_shard else rank),
                               shard=(rank, world, None) if co_shard else None,
                               algo=args.algo, gather_mode=args.gather)
    torch.cuda.synchronize()
    flops_local = plan.flops

    def barrier():
        if dist.is_initialized():
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- per-layer tile autotune (plan build, untimed), warm-up, graph capture
    # per-layer FFMA tile autotune (also for the FFMA layers of tensor-core
    # plans, e.g. batch-1 layers of a split-TF32 plan)
    tiles = {} if args.no_tune else plan.autotune(stream)
    for _ in range(args.warmup):
        plan.run(stream)
    stream.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            plan.run(stream)
        for _ in range(2):
            graph.replay()
        stream.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            plan.run(stream)

    # ---- timed region: inputs resident in HBM
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.dconv_cuda_launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    n_launch_steps = len(plan.steps)
    gpu_launches = sum(1 for s in plan.steps if s.kind not in ("gather", "barrier")) * args.steps \
        if graph is not None else lib.dconv_cuda_launch_count() - launches0
    ms_step = ms_total / args.steps
    flops_job = flops_local * world  # equal shards in both modes
    value = flops_job / (ms_step * 1e-3) / 1e9

    # ---- e2e: public API with host buffers, H2D + D2H inside the timed region
    ins = plan.io_inputs()
    outs = plan.io_outputs()
    in_host = [t.cpu().pin_memory() for t in ins]
    out_host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs]
    h2d = sum(t.numel() * t.element_size() for t in in_host)
    d2h = sum(t.numel() * t.element_size() for t in out_host)
    e2e_steps = max(3, args.steps // 2)

    def e2e_step():
        for d, h in zip(ins, in_host):
            d.copy_(h, non_blocking=True)
        step()
        for h, d in zip(out_host, outs):
            h.copy_(d, non_blocking=True)

    with torch.cuda.stream(stream):
        e2e_step()
    stream.synchronize()
    barrier()
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        e1.record(stream)
    e1.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
    e2e_value = flops_job / (e2e_ms * 1e-3) / 1e9

    # ---- per-launch durations (CUDA events on the launching stream, eager)
    per = {s.name: [] for s in plan.steps}
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in plan.steps]
    prof_steps = max(2, min(args.steps, 5))
    for _ in range(prof_steps):
        with torch.cuda.stream(stream):
            for s, (a, b) in zip(plan.steps, evs):
                a.record(stream)
                s.fn(stream)
                b.record(stream)
        stream.synchronize()
        for s, (a, b) in zip(plan.steps, evs):
            per[s.name].append(a.elapsed_time(b))
    layers, ffma_flops, ffma_ms, other_ms = [], 0, 0.0, 0.0
    for s in plan.steps:
        ms = statistics.median(per[s.name])
        rec = {"name": s.name, "kind": s.kind, "ms": round(ms, 4)}
        if s.flops:
            rec["gflops"] = round(s.flops / (ms * 1e-3) / 1e9, 1)
        layers.append(rec)
        if s.kind == "conv":
            ffma_flops += s.flops
            ffma_ms += ms
        else:
            other_ms += ms
    # the roofline follows the kernel that ran: a split-TF32 plan whose layers
    # all fell back to the FFMA kernel (batch 1, few units) reports FFMA's
    roof_algo = args.algo if any(s.kind == "tf32" for s in plan.steps) else "ffma"
    if roof_algo in ("tf32", "tf32x3"):
        # tensor-core roofline: the tcgen05 launches against a cuBLAS TF32 GEMM
        # (8192^3, torch.matmul with TF32 allowed) measured live on this GPU
        ffma_flops = sum(s.flops for s in plan.steps if s.kind == "tf32")
        ffma_ms = sum(statistics.median(per[s.name]) for s in plan.steps if s.kind == "tf32")
        other_ms = sum(statistics.median(per[s.name]) for s in plan.steps if s.kind != "tf32")
        peak = tf32_gemm_peak(stream)
        pattern = None
        if roof_algo == "tf32x3":
            # split-TF32 issues three TF32 MMAs per product: the tensor pipe
            # does 3x the algorithmic FLOPs (reported as such against the
            # TF32 peak; fp32-equivalent rate = achieved / 3)
            ffma_flops *= 3
    else:
        peak = float(lib.dconv_cuda_fp32_peak_probe(stream.cuda_stream))
        # the kernel's own FFMA2 operand pattern without memory traffic: the
        # practical ceiling of its instruction mix (reported beside the peak)
        pattern = float(lib.dconv_cuda_ffma2_pattern_probe(stream.cuda_stream))
    achieved = ffma_flops / (ffma_ms * 1e-3) / 1e12 if ffma_ms else 0.0
    for rec in layers:
        if "gflops" in rec:
            rec["frac_fp32_peak"] = round(rec["gflops"] / 1e3 / peak, 3)

    traffic, traffic_note = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            key = args.config if roof_algo == "ffma" else f"{args.config}_{roof_algo}"
            t = json.load(open(tfile)).get(key)
            if t:
                traffic = t["dram_bytes"]
                traffic_note = (f"{t['kernel']}: dram {t['dram_bytes']} B vs algorithmic "
                                f"{t['algorithmic_bytes']} B per launch ({t['source']})")
        except Exception:
            traffic = None

    if rank != 0:
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cb = cpu_reference(args.config, 1000, 1, args.cpu_seconds)
            cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["value"] = round(cpu["value"], 2)
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "error": repr(ex)}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": {"ffma": "f32", "tf32": "tf32 (stride-1 layers) + f32",
                  "tf32x3": "f32 (split-TF32 x3 on tcgen05, fp32 tolerance) + f32"}[args.algo],
        "data": "synthetic (seeded uniform[-1,1), counter-based generator)",
        "mode": ("C_o-block sharding + " + ("fused peer-store gather (symmetric memory, "
                                            "NVLink) + device barrier per layer"
                                            if args.gather == "peer" else
                                            "NCCL all-gather per layer")) if co_shard else
                "batch sharding, no collective",
        "config": {"workload": f"{args.config} chain" if args.config in ("vgg16", "resnet50")
                   else f"{args.config} layers", "global_batch": batch,
                   "per_rank_batch": n_local, "c_b": 8,
                   "parallelism": (f"co-shard x{world}, {args.gather} gather" if co_shard
                                   else f"batch-shard x{world}, no collective"),
                   "l2": "per-step working set > 126 MB L2 (activations streamed)"
                   if args.config in ("vgg16", "resnet50", "googlenet") else
                   "working set fits L2 (batch-1 config): warm-L2 numbers",
                   "graph": graph is not None, "gflop_per_step": round(flops_job / 1e9, 3),
                   "tiles": {k: ["", "128x128", "256x64", "128x64"][v]
                             for k, v in tiles.items()}},
        "roofline": {"bound": "fp32" if roof_algo == "ffma" else "tensor",
                     "achieved": round(achieved, 2), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if peak > 0 else None,
                     "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": ("conv_ffma_kernel (all blocked conv launches of the step)"
                                if roof_algo == "ffma" else
                                "conv_tf32_kernel (all stride-1 blocked conv launches)"
                                if roof_algo == "tf32" else
                                "conv_tf32x3_kernel (all tensor-core launches; achieved counts "
                                "the 3 TF32 MMAs per product, fp32-equivalent = achieved / 3)"),
                     "peak_source": ("FFMA2 throughput probe measured live on this GPU "
                                     f"(nominal {NOMINAL_FP32_TFLOPS:.1f} at 1965 MHz)"
                                     if roof_algo == "ffma" else
                                     "cuBLAS TF32 GEMM 8192^3 measured live (nominal 1100 dense)"),
                     "share_of_step": round(ffma_ms / (ffma_ms + other_ms), 4)
                     if ffma_ms + other_ms else None,
                     **({"pattern_ceiling": round(pattern, 2),
                         "frac_of_pattern_ceiling": round(achieved / pattern, 4),
                         "pattern_note": "FFMA2 broadcast-scalar x pair from LDS.128, 8 px x 8 ch "
                                         "per thread, no memory traffic "
                                         "(dconv_cuda_ffma2_pattern_probe)"}
                        if pattern else {})},
        "cpu_baseline": cpu,
        "e2e": {"value": round(e2e_value, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4)},
        "gpu_launches": int(gpu_launches),
        "clocks": clk.summary(),
        "layers": layers,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    main_gpu(args)


if __name__ == "__main__":
    main()
