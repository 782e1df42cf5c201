#!/usr/bin/env python
"""Benchmark of the direct-convolution hot path (BASELINE.json metric:
"direct-conv GFLOP/s per layer & % of B200 FP32 (TF32) peak, zero workspace").

Default workload: BASELINE configs[2], the VGG-16 chain (13 x 3x3 convs +
ReLU + 4 max-pools, every activation in the blocked layout), global batch 32,
fp32, batch-sharded over the ranks with no collective.  One *step* = one pass
of the whole chain over the batch.  `--config` selects the other configs;
`--extra` (default: every other config at its BASELINE batch, ResNet-50 at
b256 included) measures them in the same run and reports them under
"extra_configs" -- the driver-visible line carries every config.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config vgg16]
  python bench.py --impl reference ...      # CPU reference arm
  python bench.py --gpus N --dry-run        # launcher check on CPU (gloo)

`--gpus N` with N > 1 and no torchrun environment re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU,
NCCL; NCCL_DEBUG=INFO shows the communicator).

One JSON line on rank 0.  `value` = whole-job GFLOP/s with inputs resident in
HBM (CUDA-graph replay, CUDA events, max over ranks); `e2e` = the same work
through the public API with the input batch copied H2D from pinned memory and
the network output copied D2H inside the timed region; `roofline` = the FFMA
direct-conv kernel's achieved FLOP/s (algorithmic conv_flops / its launch
durations, CUDA events on its stream) over the nominal FP32 peak
(148 SMs x 128 lanes x 2 x the SM max clock); `cpu_baseline` = the restated
reference algorithm (Alg. 3, oracle/oracle.c) scheduled on the reference's
own ThreadPool (oracle/_ref) with DCONV_THREADS = physical cores - 1, over a
bounded sample, run twice (spread reported).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "direct-conv GFLOP/s per layer & % of B200 FP32 (TF32) peak, zero workspace"
DEFAULT_BATCH = {"cfg1": 1, "alexnet": 1, "vgg16": 32, "googlenet": 64, "resnet50": 256}
SMS, FP32_LANES = 148, 128
# TF32 dense tensor peak = half the bf16 dense rate (same MMA shape, 2x bytes
# per element); denominators from MEASURED_PEAKS.json (driver-written)
FALLBACK_BF16_TFLOPS = 1590.0  # B200_PROFILING.md fallback (burst)


def nominal_fp32_tflops(sm_max_mhz: float = 1965.0) -> float:
    return SMS * FP32_LANES * 2 * sm_max_mhz * 1e6 / 1e12  # 74.45 at 1965 MHz


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg16", choices=sorted(DEFAULT_BATCH))
    ap.add_argument("--batch", type=int, default=0, help="global batch (0 = config default)")
    ap.add_argument("--extra", default="cfg1,alexnet,googlenet,resnet50,vgg16:1,googlenet:1,resnet50:1",
                    help="other configs measured in the same run: comma list of CONFIG "
                         "(BASELINE batch) or CONFIG:BATCH; 'none'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-tune", action="store_true",
                    help="skip the per-layer CTA-tile autotune at plan build")
    ap.add_argument("--algo", default="ffma", choices=["ffma", "tf32", "tf32x3"],
                    help="ffma: the fp32 FFMA path (the headline); tf32: blocked layers on "
                         "the tcgen05/TMEM TF32 variant (reduced precision, reported apart); "
                         "tf32x3: split-TF32 on the tensor cores at the fp32 tolerance")
    ap.add_argument("--shard", default="batch", choices=["batch", "co"],
                    help="batch: image ranges per rank, no collective; co: batch-1 "
                         "output-block sharding with an NCCL all-gather per layer")
    ap.add_argument("--gather", default="nccl", choices=["nccl", "peer"],
                    help="--shard co exchange: nccl all-gather of slices, or peer = each "
                         "conv/pool epilogue stores into every rank's map over NVLink "
                         "(symmetric memory) + a device barrier")
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target CPU work per cpu_baseline run (two runs)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without GPUs: gloo ranks report their shards")
    return ap.parse_args(argv)


# ------------------------------------------------------------------ launcher
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args) -> bool:
    """`--gpus N` (N > 1) outside torchrun: re-execute this command under
    torch.distributed.run with N ranks (one per GPU).  Returns True when the
    ranks ran here (the caller exits with their status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("MASTER_ADDR", "127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd, env=env)
    sys.exit(rc)


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def run_dry(args) -> None:
    """CPU launcher check: every rank joins a gloo group and reports its image
    range (batch sharding) or output-block range (C_o sharding)."""
    import torch.distributed as dist

    from paper_1809_10170_b200 import nets, shard
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = args.batch or DEFAULT_BATCH[args.config]
    if args.shard == "co":
        l = nets.CONFIGS[args.config][-1]
        mine = {"rank": rank, "pid": os.getpid(),
                "co_blocks": list(shard.block_range(nets.nblk(l.c_o), world, rank))}
    else:
        mine = {"rank": rank, "pid": os.getpid(),
                "images": list(shard.batch_range(batch, world, rank))}
    ranks = [None] * world
    if world > 1:
        dist.all_gather_object(ranks, mine)
    else:
        ranks = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": args.config,
                          "global_batch": batch, "shard": args.shard, "ranks": ranks}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------ host CPU
def host_cpu() -> dict:
    """nproc, physical cores (unique (package, core) pairs of /proc/cpuinfo),
    CPU model, and the cores this process may run on."""
    info = {"nproc": os.cpu_count() or 1, "model": None, "physical_cores": None}
    try:
        info["usable"] = len(os.sched_getaffinity(0))
    except Exception:
        info["usable"] = info["nproc"]
    try:
        pairs, phys = set(), None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and info["model"] is None:
                info["model"] = v
            elif k == "physical id":
                phys = v
            elif k == "core id":
                pairs.add((phys, v))
        if pairs:
            info["physical_cores"] = len(pairs)
    except Exception:
        pass
    if not info["physical_cores"]:
        info["physical_cores"] = info["nproc"]
    return info


def _cpu_layers(config: str):
    import numpy as np  # noqa: F401

    from oracle import pyoracle as po  # CPU baseline leg only
    from paper_1809_10170_b200 import nets
    layers = nets.CONFIGS[config]
    data = []
    for idx, l in enumerate(layers):
        cib = l.c_i if l.first else 8
        xb = po.pack_feature_map(po.uniform((l.c_i, l.h_i, l.w_i), 1809, 2 * idx), cib)
        kb = po.pack_kernel(po.uniform((l.c_i, l.c_o, l.h_f, l.w_f), 1809, 1000 + 2 * idx),
                            8, cib)
        data.append((l, xb, kb))
    return layers, data


def cpu_reference(config: str, budget_s: float, trials: int = 9, warm: int = 2,
                  runs: int = 3, alg2: bool = True) -> dict:
    """Restated reference Alg. 3 (oracle/oracle.c: j' parallel, i', l, k', n,
    m, ii, kk, jj; AVX2 8 x 14 tile) on the reference's own ThreadPool
    (thread_pool.cpp:64-97, oracle/_ref) with DCONV_THREADS = physical
    cores - 1 workers plus the calling thread, one image of the workload
    through every layer per sample.  SPEC.md:522 timing policy: median of
    up to 9 samples after 2 warm-ups (bounded by ``budget_s`` per run), min
    recorded; ``runs`` independent runs, spread reported."""
    import numpy as np

    from oracle import pyoracle as po
    cpu = host_cpu()
    threads = max(1, min(cpu["physical_cores"], cpu["usable"]))
    workers = threads - 1
    layers, data = _cpu_layers(config)
    flops = sum(l.flops for l in layers)
    outs = []
    for l, xb, kb in data:
        outs.append(np.empty((1, kb.shape[0], l.h_o, l.w_o, 8), np.float32))

    def one():
        t0 = time.perf_counter()
        for (l, xb, kb), o in zip(data, outs):
            po.conv_direct_pool(xb[None], kb, l.c_i, l.c_o, l.s, workers, w_ob=14, out=o)
        return time.perf_counter() - t0

    # settle the host first (pool threads spun up, pages touched, clocks
    # ramped): without it the first run read ~25% below the second
    settle_s = float(os.environ.get("DCONV_CPU_SETTLE", "1.5"))
    t_settle = time.perf_counter()
    while time.perf_counter() - t_settle < settle_s:
        one()
    run_vals, all_min, samples = [], None, 0
    for _ in range(runs):
        ws = [one() for _ in range(warm)]
        per = min(ws)
        n = max(1, min(trials, int(budget_s / max(per, 1e-6))))
        ts = [one() for _ in range(n)]
        samples += n
        run_vals.append(flops / statistics.median(ts) / 1e9)
        m = flops / min(ts) / 1e9
        all_min = m if all_min is None else max(all_min, m)
    value = statistics.median(run_vals)
    out = {
        "value": round(value, 2), "unit": "GFLOP/s", "cores": threads, "kind": "port",
        "threads": threads, "pool_workers": workers, "nproc": cpu["nproc"],
        "physical_cores": cpu["physical_cores"], "cpu_model": cpu["model"],
        "runs": [round(v, 2) for v in run_vals],
        "spread": round((max(run_vals) - min(run_vals)) / max(run_vals), 4),
        "best_sample": round(all_min, 2),
        "sample": (f"1 image of {config} ({len(layers)} layers, {flops / 1e9:.2f} GFLOP) through "
                   f"restated Alg. 3 (oracle/oracle.c, c_ob=8 w_ob=14 AVX2 tile) on the "
                   f"reference ThreadPool (DCONV_THREADS={workers} + caller = {threads} threads "
                   f"= physical cores); after 1.5 s of settling passes, median of <=9 samples "
                   f"after 2 warm-ups, {runs} runs (median reported); "
                   f"the reference's own conv_direct is absent from the snapshot"),
        "seconds_per_sample": flops / value / 1e9,
    }
    if alg2:
        try:
            out["reference_alg2"] = cpu_reference_alg2(config, threads)
        except Exception as ex:  # report, never fake
            out["reference_alg2"] = {"error": repr(ex)}
    return out


def cpu_reference_alg2(config: str, threads: int) -> dict:
    """The reference's OWN compiled code (oracle/_ref: conv_reordered, Alg. 2,
    reference.cpp:54-68, unmodified) on its ThreadPool, one image per chunk,
    `threads` images of the config's largest-FLOP layer (a bounded sample)."""
    import numpy as np

    from oracle import pyoracle as po
    from paper_1809_10170_b200 import nets
    r = po.ref()
    if r is None:
        raise RuntimeError("oracle/_ref not built")
    l = max(nets.CONFIGS[config], key=lambda q: q.flops)
    n = threads
    x = po.uniform((n, l.c_i, l.h_i, l.w_i), 1809, 7)
    k = po.uniform((l.c_i, l.c_o, l.h_f, l.w_f), 1809, 8)
    y = np.empty((n, l.c_o, l.h_o, l.w_o), np.float32)
    t0 = time.perf_counter()
    rc = r.ref_conv_reordered_batch(po._fp(x), po._fp(k), n, l.c_i, l.c_o, l.h_i, l.w_i, l.h_f,
                                    l.w_f, l.s, threads, po._fp(y))
    dt = time.perf_counter() - t0
    if rc:
        raise RuntimeError("ref_conv_reordered_batch failed")
    return {"value": round(n * l.flops / dt / 1e9, 2), "unit": "GFLOP/s", "threads": threads,
            "sample": f"{n} images of {config} {l.name} ({n * l.flops / 1e9:.2f} GFLOP), "
                      f"conv_reordered (reference Alg. 2) on the reference ThreadPool, one "
                      f"image per chunk, 1 run"}


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cb = cpu_reference(args.config, args.cpu_seconds, runs=3)
    batch = args.batch or DEFAULT_BATCH[args.config]
    line = {
        "metric": METRIC, "impl": "reference", "value": cb["value"],
        "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(cb["seconds_per_sample"] * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config} chain, 1-image sample of the b{batch} job",
                   "global_batch": batch, "c_b": 8},
        "cpu_baseline": {k: v for k, v in cb.items() if k != "seconds_per_sample"},
        "e2e": {"value": cb["value"], "unit": "GFLOP/s",
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


def measured_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ GPU arm
class Ctx:
    """Per-process GPU state shared by the headline and the extra configs."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world, self.rank, self.local = dist_env()
        torch.cuda.set_device(self.local)
        self.co_shard = args.shard == "co"
        if self.world > 1 or self.co_shard:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            dist.init_process_group("nccl", rank=self.rank, world_size=self.world,
                                    device_id=torch.device("cuda", self.local))
        from paper_1809_10170_b200 import _abi
        self.lib = _abi.lib()
        self.stream = torch.cuda.Stream()
        self.flush_buf = None

    def barrier(self):
        if self.dist.is_initialized():
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def flush_l2(self):
        """Write 512 MB (> 4x the 126 MB L2) on the stream: the next step
        starts with a cold L2."""
        if self.flush_buf is None:
            self.flush_buf = self.torch.empty(128 << 20, dtype=self.torch.float32, device="cuda")
        with self.torch.cuda.stream(self.stream):
            self.flush_buf.fill_(1.0)


def build(ctx, args, config: str, batch: int, co_shard: bool):
    from paper_1809_10170_b200 import nets
    torch = ctx.torch
    if co_shard:
        if batch != 1:
            raise SystemExit("--shard co is the batch-1 mode")
        n_local = 1
    else:
        if batch % ctx.world:
            raise SystemExit(f"global batch {batch} not divisible by {ctx.world} ranks")
        n_local = batch // ctx.world  # batch sharding: contiguous image range per rank
    with torch.cuda.stream(ctx.stream):
        plan = nets.build_plan(config, n_local, seed=1809 + (0 if co_shard else ctx.rank),
                               shard=(ctx.rank, ctx.world, None) if co_shard else None,
                               algo=args.algo, gather_mode=args.gather)
    torch.cuda.synchronize()
    return plan, n_local


def co_shard_parity(ctx, args, plan, config: str) -> dict:
    """--shard co: the gathered output of the real multi-rank run against
    (1) every rank's launches replayed on this device into one map (the
    emulated ranks; identical kernel configurations -> bitwise), and (2) the
    unsharded single-rank plan (different split-K -> within a normwise
    bound).  Rank 0 checks; all ranks run the real step first."""
    from paper_1809_10170_b200 import nets
    torch = ctx.torch
    plan.run(ctx.stream)
    torch.cuda.synchronize()
    ctx.barrier()
    if ctx.rank != 0:
        return {}
    got = plan.output.buf.clone()
    with torch.cuda.stream(ctx.stream):
        emu = nets.build_plan(config, 1, seed=1809, shard=(0, ctx.world, None),
                              algo=args.algo, gather_mode="emulate")
        emu.tiles.update(plan.tiles)
        emu.run(ctx.stream)
        ref = nets.build_plan(config, 1, seed=1809, algo=args.algo)
        ref.run(ctx.stream)
    torch.cuda.synchronize()
    a, b = got, emu.output.buf
    bitwise = bool(torch.equal(a, b))
    c = ref.output.buf
    scale = float(c.abs().max())
    err = float((a - c).abs().max())
    # normwise: the unsharded plan splits K differently (rounding only)
    ok = bitwise and err <= 1e-4 * max(1.0, scale)
    del emu, ref
    return {"status": "ok" if ok else "FAIL", "emulated_ranks_bitwise": bitwise,
            "unsharded_max_abs_err": err, "unsharded_max_abs": scale,
            "checked": "whole network output (every element)"}


def time_steps(ctx, step, steps: int):
    """K steps between two events on the plan's stream (barrier + sync on both
    sides); returns (ms per step, max over ranks)."""
    torch = ctx.torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    torch.cuda.synchronize()
    with torch.cuda.stream(ctx.stream):
        e0.record(ctx.stream)
        for _ in range(steps):
            step()
        e1.record(ctx.stream)
    e1.synchronize()
    torch.cuda.synchronize()
    ctx.barrier()
    return ctx.max_over_ranks(e0.elapsed_time(e1)) / steps


def per_step_times(ctx, step, trials: int, flush: bool):
    """SPEC.md:522 policy on the device: `trials` single steps, each between
    its own events (optionally after an L2 flush outside the events)."""
    torch = ctx.torch
    ts = []
    for _ in range(trials):
        if flush:
            ctx.flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ctx.stream):
            a.record(ctx.stream)
            step()
            b.record(ctx.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return ts


def layer_profile(ctx, plan, reps: int):
    """Median CUDA-event duration of every launch of the plan (eager, on the
    plan's stream)."""
    torch = ctx.torch
    per = {s.name: [] for s in plan.steps}
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in plan.steps]
    for _ in range(reps):
        with torch.cuda.stream(ctx.stream):
            for s, (a, b) in zip(plan.steps, evs):
                a.record(ctx.stream)
                s.fn(ctx.stream)
                b.record(ctx.stream)
        ctx.stream.synchronize()
        for s, (a, b) in zip(plan.steps, evs):
            per[s.name].append(a.elapsed_time(b))
    return {k: statistics.median(v) for k, v in per.items()}


def roofline_for(ctx, args, plan, med, clk_max):
    """Achieved FLOP/s of the dominant kernel class over its summed launch
    durations, against the nominal FP32 peak (FFMA) or the measured TF32
    peak (tensor-core plans)."""
    pk = measured_peaks()
    roof_algo = args.algo if any(s.kind == "tf32" for s in plan.steps) else "ffma"
    if roof_algo in ("tf32", "tf32x3"):
        kflops = sum(s.flops for s in plan.steps if s.kind == "tf32")
        kms = sum(med[s.name] for s in plan.steps if s.kind == "tf32")
        if roof_algo == "tf32x3":
            kflops *= 3  # three TF32 MMAs per product on the tensor pipe
        bf16 = pk.get("bf16_tflops")
        peak = (bf16 or FALLBACK_BF16_TFLOPS) / 2
        src = (f"MEASURED_PEAKS.json bf16_tflops {bf16} / 2 (TF32 = half the bf16 dense rate), "
               "of measured" if bf16 else
               f"fallback bf16 {FALLBACK_BF16_TFLOPS} / 2 (B200_PROFILING.md), of fallback")
        bound = "tensor"
    else:
        kflops = sum(s.flops for s in plan.steps if s.kind == "conv")
        kms = sum(med[s.name] for s in plan.steps if s.kind == "conv")
        peak = nominal_fp32_tflops(clk_max or 1965.0)
        src = (f"nominal FP32: {SMS} SMs x {FP32_LANES} lanes x 2 FLOP x "
               f"{clk_max or 1965.0:.0f} MHz (SM max clock)")
        bound = "fp32"
    total = sum(med.values())
    achieved = kflops / (kms * 1e-3) / 1e12 if kms else 0.0
    # per-launch roofline: max(FLOPs / compute peak, compulsory bytes / HBM);
    # the step's bound is their sum (ResNet's 64-channel 1x1 layers sit near
    # the FP32 ridge and below the TF32 one: there HBM is the limit)
    hbm = pk.get("hbm_gbs") or 6650.0
    fp_peak = nominal_fp32_tflops(clk_max or 1965.0)
    tc_peak = (pk.get("bf16_tflops") or FALLBACK_BF16_TFLOPS) / 2
    bound_ms, meas_ms = 0.0, 0.0
    for s in plan.steps:
        if not (s.flops or s.bytes):
            continue
        if s.kind == "tf32":
            t_c = s.flops * (3 if args.algo == "tf32x3" else 1) / (tc_peak * 1e12) * 1e3
        else:
            t_c = s.flops / (fp_peak * 1e12) * 1e3
        t_m = s.bytes / (hbm * 1e9) * 1e3
        bound_ms += max(t_c, t_m)
        meas_ms += med[s.name]
    return roof_algo, {"bound": bound, "achieved": round(achieved, 2), "peak": round(peak, 2),
                       "unit": "TFLOP/s", "frac": round(achieved / peak, 4) if peak else None,
                       "peak_source": src,
                       "share_of_step": round(kms / total, 4) if total else None,
                       "step_bound_ms": round(bound_ms, 4),
                       "frac_of_step_bound": round(bound_ms / meas_ms, 4) if meas_ms else None,
                       "step_bound_note": (f"sum over launches of max(FLOPs / {fp_peak:.1f} FP32 "
                                           f"or {tc_peak:.0f} TF32 TFLOP/s, compulsory bytes / "
                                           f"{hbm:.0f} GB/s HBM (MEASURED_PEAKS.json))")}


def measure_config(ctx, args, config: str, batch: int, headline: bool) -> dict:
    """Build, autotune, warm up, capture and time one config; returns the
    fields of its JSON record."""
    torch = ctx.torch
    co_shard = ctx.co_shard and headline
    plan, n_local = build(ctx, args, config, batch, co_shard)
    parity = co_shard_parity(ctx, args, plan, config) if co_shard else None
    tiles = {} if args.no_tune else plan.autotune(ctx.stream)
    for _ in range(args.warmup):
        plan.run(ctx.stream)
    ctx.stream.synchronize()
    graph = None
    if not (args.no_graph or co_shard):  # collectives stay outside graph capture
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=ctx.stream):
            plan.run(ctx.stream)
        for _ in range(2):
            graph.replay()
        ctx.stream.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            plan.run(ctx.stream)

    launches0 = ctx.lib.dconv_cuda_launch_count()
    with ClockSampler(ctx.local) as clk:
        ms_step = time_steps(ctx, step, args.steps)
    gpu_launches = (sum(1 for s in plan.steps if s.kind not in ("gather", "barrier")) * args.steps
                    if graph is not None else ctx.lib.dconv_cuda_launch_count() - launches0)
    flops_job = plan.flops * ctx.world  # equal shards in both modes
    value = flops_job / (ms_step * 1e-3) / 1e9
    # median of 9 single steps after the warm-ups, min recorded;
    # warm L2 and with an L2 flush before every step
    warm = per_step_times(ctx, step, 9, flush=False)
    cold = per_step_times(ctx, step, 9, flush=True)
    policy = {
        "warm_l2": {"median_ms": round(statistics.median(warm), 4),
                    "min_ms": round(min(warm), 4),
                    "gflops_median": round(flops_job / (statistics.median(warm) * 1e-3) / 1e9, 1)},
        "l2_flushed": {"median_ms": round(statistics.median(cold), 4),
                       "min_ms": round(min(cold), 4),
                       "gflops_median": round(flops_job / (statistics.median(cold) * 1e-3) / 1e9,
                                              1)},
        "policy": "9 single steps after the warm-ups, each between CUDA events; "
                  "l2_flushed writes 512 MB before each step (outside the events)"}

    # e2e: the public streaming API (nets.Pipeline) with pinned host buffers:
    # every step copies its inputs H2D and its result D2H inside the timed
    # region; the copies of neighbouring steps overlap this step's kernels
    from paper_1809_10170_b200 import nets
    ins, outs = plan.io_inputs(), plan.io_outputs()
    in_host = [t.cpu().pin_memory() for t in ins]
    out_host = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs]
    h2d = sum(t.numel() * t.element_size() for t in in_host)
    d2h = sum(t.numel() * t.element_size() for t in out_host)
    if not co_shard:
        pipe = nets.Pipeline(plan, in_host, out_host, ctx.stream)
        pipe.run(2)
        torch.cuda.synchronize()
        e2e_steps = max(3, args.steps // 2)
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        torch.cuda.synchronize()
        e_a.record(pipe.copy_in)
        pipe.run(e2e_steps)
        pipe.copy_out.wait_stream(pipe.compute)
        pipe.copy_out.wait_stream(pipe.copy_in)
        e_b.record(pipe.copy_out)
        e_b.synchronize()
        torch.cuda.synchronize()
        ctx.barrier()
        e2e_ms = ctx.max_over_ranks(e_a.elapsed_time(e_b)) / e2e_steps
        e2e_mode = ("nets.Pipeline: eager launches on the compute stream, H2D / D2H on two "
                    "copy streams overlapping neighbouring steps")
    else:
        def e2e_step():
            for d, h in zip(ins, in_host):
                d.copy_(h, non_blocking=True)
            step()
            for h, d in zip(out_host, outs):
                h.copy_(d, non_blocking=True)

        with torch.cuda.stream(ctx.stream):
            e2e_step()
        ctx.stream.synchronize()
        e2e_ms = time_steps(ctx, e2e_step, max(3, args.steps // 2))
        e2e_mode = "copy in, step, copy out on one stream"
    e2e_value = flops_job / (e2e_ms * 1e-3) / 1e9

    med = layer_profile(ctx, plan, max(2, min(args.steps, 5)))
    roof_algo, roof = roofline_for(ctx, args, plan, med, clk.max_mhz)
    layers = []
    for s in plan.steps:
        rec = {"name": s.name, "kind": s.kind, "ms": round(med[s.name], 4)}
        if s.flops:
            rec["gflops"] = round(s.flops / (med[s.name] * 1e-3) / 1e9, 1)
            if s.kind in ("conv", "first"):
                rec["frac_fp32_peak"] = round(rec["gflops"] / 1e3 / nominal_fp32_tflops(
                    clk.max_mhz or 1965.0), 3)
        if s.bytes:
            rec["gbps"] = round(s.bytes / (med[s.name] * 1e-3) / 1e9, 1)
            if s.flops:
                rec["flop_per_byte"] = round(s.flops / s.bytes, 1)
        layers.append(rec)
    # working set ~ the compulsory bytes of one step against the 126 MB L2
    ws_bytes = sum(s.bytes for s in plan.steps)
    fits_l2 = ws_bytes < 126e6
    rec = {
        "config": config, "global_batch": batch, "per_rank_batch": n_local,
        "value": round(value, 1), "ms_per_step": round(ms_step, 4),
        "gflop_per_step": round(flops_job / 1e9, 3), "graph": graph is not None,
        "e2e": {"value": round(e2e_value, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4), "mode": e2e_mode},
        "timing_policy": policy,
        "l2": (f"working set ~{ws_bytes / 1e6:.0f} MB fits the 126 MB L2: warm-L2 value, "
               "l2_flushed beside it" if fits_l2 else
               f"per-step working set ~{ws_bytes / 1e6:.0f} MB > 126 MB L2 (streamed)"),
        "roofline": roof, "roof_algo": roof_algo, "gpu_launches": int(gpu_launches),
        "clocks": clk.summary(),
        "tiles": {k: ["", "128x128", "256x64", "128x64", "256x32"][v] for k, v in tiles.items()},
        "layers": layers,
    }
    if parity is not None:
        rec["parity"] = parity
    del plan, graph
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


def main_gpu(args):
    ctx = Ctx(args)
    world, rank = ctx.world, ctx.rank
    batch = args.batch or (1 if ctx.co_shard else DEFAULT_BATCH[args.config])
    head = measure_config(ctx, args, args.config, batch, headline=True)
    if head.get("parity", {}).get("status") == "FAIL":
        print(json.dumps({"error": "co-shard parity failed", "parity": head["parity"]}),
              file=sys.stderr, flush=True)
    extras = []
    if args.extra != "none" and not ctx.co_shard:
        for item in [c for c in args.extra.split(",") if c]:
            cfg, _, b = item.partition(":")
            eb = int(b) if b else DEFAULT_BATCH[cfg]
            if cfg == args.config and eb == batch:
                continue
            try:
                extras.append(measure_config(ctx, args, cfg, eb, False))
            except SystemExit as ex:  # e.g. batch not divisible by the ranks
                extras.append({"config": cfg, "global_batch": eb, "skipped": str(ex)})

    traffic, traffic_note = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            ra = head["roof_algo"]
            key = args.config if ra == "ffma" else f"{args.config}_{ra}"
            t = json.load(open(tfile)).get(key)
            if t:
                traffic = t["dram_bytes"]
                traffic_note = (f"{t['kernel']}: dram {t['dram_bytes']} B vs algorithmic "
                                f"{t['algorithmic_bytes']} B per launch ({t['source']})")
        except Exception:
            traffic = None
    probe = None
    if head["roof_algo"] == "ffma":
        probe = {"ffma2_probe_tflops": round(float(
                     ctx.lib.dconv_cuda_fp32_peak_probe(ctx.stream.cuda_stream)), 2),
                 "ffma2_pattern_ceiling_tflops": round(float(
                     ctx.lib.dconv_cuda_ffma2_pattern_probe(ctx.stream.cuda_stream)), 2),
                 "note": "live probes (side fields, not the denominator): FFMA2 on constant "
                         "registers, and the kernel's own operand pattern (8 px x 8 ch per "
                         "thread, LDS.128 operands) with no memory traffic"}

    if rank != 0:
        if ctx.dist.is_initialized():
            ctx.dist.barrier()
            ctx.dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_reference(args.config, args.cpu_seconds)
            cpu.pop("seconds_per_sample", None)
        except Exception as ex:  # report, never fake
            cpu = {"value": None, "error": repr(ex)}

    roof = dict(head["roofline"], traffic=traffic, traffic_note=traffic_note)
    roof["kernel"] = {"ffma": "conv_ffma_kernel (all blocked conv launches of the step)",
                      "tf32": "conv_tf32_kernel (all tensor-core launches)",
                      "tf32x3": "conv_tf32x3_kernel (all tensor-core launches; achieved counts "
                                "the 3 TF32 MMAs per product, fp32-equivalent = achieved / 3)"}[
        head["roof_algo"]]
    if probe:
        roof.update(probe)
    line = {
        "metric": METRIC, "value": head["value"], "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong",  # the global batch is fixed; ranks split it
        "vs_baseline": None,
        "dtype": {"ffma": "f32", "tf32": "tf32 (tensor-core layers) + f32",
                  "tf32x3": "f32 (split-TF32 x3 on tcgen05, fp32 tolerance) + f32"}[args.algo],
        "data": "synthetic (seeded uniform[-1,1), counter-based generator)",
        "mode": ("C_o-block sharding + " + ("fused peer-store gather (symmetric memory, "
                                            "NVLink) + device barrier per layer"
                                            if args.gather == "peer" else
                                            "NCCL all-gather per layer")) if ctx.co_shard else
                "batch sharding, no collective",
        "config": {"workload": f"{args.config} chain" if args.config in ("vgg16", "resnet50")
                   else f"{args.config} layers", "global_batch": batch,
                   "per_rank_batch": head["per_rank_batch"], "c_b": 8,
                   "parallelism": (f"co-shard x{world}, {args.gather} gather" if ctx.co_shard
                                   else f"batch-shard x{world}, no collective"),
                   "l2": head["l2"], "graph": head["graph"],
                   "gflop_per_step": head["gflop_per_step"], "tiles": head["tiles"]},
        "timing_policy": head["timing_policy"],
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"],
        "clocks": head["clocks"],
        "layers": head["layers"],
        "extra_configs": extras,
    }
    if "parity" in head:
        line["parity"] = head["parity"]
    print(json.dumps(line), flush=True)
    if ctx.dist.is_initialized():
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()


def main():
    args = parse()
    maybe_relaunch(args)
    if args.dry_run:
        run_dry(args)
        return
    if args.impl == "reference":
        run_reference_arm(args)
        return
    main_gpu(args)


if __name__ == "__main__":
    main()
