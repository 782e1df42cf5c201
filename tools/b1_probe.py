"""Batch-1 latency probe: per-launch kernel time (CUDA events, eager) of the
cfg1 / AlexNet plans, plus graph replay per step with 1 and with 20 plan
passes per graph (launch gaps between graph replays)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1809_10170_b200 import nets  # noqa: E402

for cfg in ("cfg1", "alexnet"):
    plan = nets.build_plan(cfg, 1)
    plan.autotune()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(5):
            plan.run(s)
    s.synchronize()
    for st in plan.steps:
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                a.record(s)
                st.fn(s)
                b.record(s)
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        print(f"{cfg} {st.name}: eager {statistics.median(ts):.1f} us "
              f"({st.flops / statistics.median(ts) / 1e6:.1f} TFLOP/s)", flush=True)
    for per_graph in (1, 20):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_graph):
                plan.run(s)
        for _ in range(3):
            g.replay()
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200 // per_graph
        with torch.cuda.stream(s):
            a.record(s)
            for _ in range(reps):
                g.replay()
            b.record(s)
        b.synchronize()
        us = a.elapsed_time(b) * 1e3 / (reps * per_graph)
        print(f"{cfg}: graph with {per_graph} passes: {us:.2f} us per pass, "
              f"{plan.flops / us / 1e6:.1f} TFLOP/s", flush=True)
