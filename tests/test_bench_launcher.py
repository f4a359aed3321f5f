"""bench.py's multi-GPU entry point on CPU: `--gpus N` without a torchrun environment launches
N ranks itself, the ranks go through the bench's own rank loop, barriers and max-over-ranks
reduction (gloo here, NCCL on the GPU box), and rank 0 alone prints one JSON line with
n_gpus == N.  `--dry-run` replaces the device frames with no-ops (nothing else changes).
The reference arm runs the CPU path only: it never imports the product package."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_n_ranks_and_reports_n_gpus(n):
    out = subprocess.run([sys.executable, BENCH, "--gpus", str(n), "--dry-run", "--steps", "6", "--warmup", "1",
                          "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True, env=_env(), timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n
    assert d["config"]["parallelism"].startswith(f"frame-sharded x{n}")
    assert d["steps"] == 6 and d["value"] > 0 and d["frame_latency_ms"]["frames"] >= 1


def test_bench_rejects_world_size_mismatch():
    env = _env()
    env.update(RANK="0", WORLD_SIZE="3", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run", "--steps", "2"], capture_output=True,
                         text=True, env=env, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=3" in (out.stderr + out.stdout)


def test_reference_arm_is_cpu_only_and_times_full_frames():
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0'];"
            "runpy.run_path(%r, run_name='__main__');"
            "bad = [m for m in sys.modules if m.startswith('paper_2007_13988_b200')];"
            "assert not bad, bad" % BENCH)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=_env(), timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "port"
    assert "FULL" in d["cpu_baseline"]["sample"]
    # the timed region is real: ms_per_step x steps is what the run took, no extrapolation
    assert d["ms_per_step"] / 1e3 == pytest.approx(1.0 / d["value"], rel=1e-9)
    assert d["e2e"]["value"] == d["value"]
