"""bench.py --impl reference (the CPU arm the driver times beside ours):
runs without a GPU, prints one JSON line with the contract's keys, and under
torchrun only rank 0 works and reports the measured arm's replica count."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--steps", "3", "--warmup", "3",
           "--ref-seconds", "1", "--n", str(1 << 20)]
    return subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_line():
    r = _run({"WORLD_SIZE": "1", "RANK": "0"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["higher_is_better"] is True and line["steps"] == 3 and line["warmup"] == 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["parallelism"].startswith("1 independent")


def test_reference_arm_under_torchrun_env():
    r1 = _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r1.returncode == 0 and r1.stdout.strip() == ""  # non-zero ranks exit without work
    r0 = _run({"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r0.returncode == 0, r0.stderr[-2000:]
    line = json.loads(r0.stdout.strip().splitlines()[-1])
    assert line["config"]["parallelism"].startswith("2 independent")


def test_gpus_flag_spawns_ranks_without_torchrun():
    """`bench.py --gpus 2` outside torchrun launches 2 ranks itself (one per
    GPU; here the CPU reference arm, where rank 0 alone reports)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--ref-seconds", "1", "--n", str(1 << 20)]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"].startswith("2 independent")


def test_variant_switches_refused():
    r = _run({"WORLD_SIZE": "1", "RANK": "0", "OFL_HEAT_TB": "8"})
    assert r.returncode != 0 and "run-changing switches" in (r.stderr + r.stdout)


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--steps", "3", "--warmup", "3"],
                       cwd=REPO, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
