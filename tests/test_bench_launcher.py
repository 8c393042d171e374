"""CPU checks of bench.py's plumbing (no GPU): the --gpus N launcher re-executes under torchrun
with N ranks and the rank-0 JSON line carries n_gpus = N and the max-over-ranks time (gloo
self-test); the reference arm prints the same config dict as our arm (driver's same_config)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_gpus_flag_spawns_ranks_gloo():
    d = _run(["--gpus", "2", "--selftest-dist", "--steps", "2"])
    assert d["n_gpus"] == 2
    assert abs(d["max_over_ranks_s"] - 0.004) < 1e-12      # rank 1's 2 x 2 ms, not rank 0's
    assert d["config"]["global_batch"] == 2 * 8192


def test_reference_arm_line_and_config():
    sys.path.insert(0, ROOT)
    import bench
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--pairs", "32", "--ref-step-s", "0.05"])
    assert d["impl"] == "reference" and d["unit"] == "traces/s" and d["higher_is_better"] is True
    assert d["config"] == bench.headline_config(1)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["cpu_model"]
