"""bench.py's launch contract on CPU: `--gpus N` without a torchrun
environment re-launches itself as N ranks (torch.distributed.run, 127.0.0.1)
and rank 0 alone prints the reference arm's one JSON line; the reference arm
imports nothing from the product package and prints the same metric string
as our arm."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_self_launch_two_ranks():
    lines = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-streams", "2",
                  "--ref-seconds", "3", "--ref-gen-frames", "1"])
    assert len(lines) == 1, lines           # rank 0 only
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0
    import bench  # noqa: E402 -- the module constant both arms print
    assert d["metric"] == bench.METRIC
    assert "256 streams" in d["config"]["workload"] and d["scaling"] == "strong"


def test_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
