"""bench.py contract checks that run without a GPU: the reference (CPU) arm
prints one well-formed JSON line, and the GPU arm's rank logic is importable."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg1", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "cpu_baseline"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GFLOP/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "port"


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg1", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0 and not r.stdout.strip()


def test_reference_arm_reports_host_and_pool():
    """The CPU baseline states nproc, physical cores, the CPU model and the
    thread count, runs on the reference ThreadPool with DCONV_THREADS =
    physical - 1, and carries the reference's own Alg. 2 beside it."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg1", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    cb = d["cpu_baseline"]
    for k in ("nproc", "physical_cores", "cpu_model", "threads", "pool_workers", "runs",
              "spread", "best_sample", "reference_alg2"):
        assert k in cb, k
    assert cb["pool_workers"] == cb["threads"] - 1 and cb["cores"] == cb["threads"]
    assert cb["reference_alg2"]["value"] > 0


def test_gpus_flag_launches_ranks_dry_run():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself
    (torch.distributed.run); in --dry-run they join a gloo group and rank 0
    reports n_gpus = 2 with both ranks' image ranges."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-run", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and [q["rank"] for q in d["ranks"]] == [0, 1]
    assert len({q["pid"] for q in d["ranks"]}) == 2
    assert [q["images"] for q in d["ranks"]] == [[0, 16], [16, 16]]
