"""bench.py contract on the CPU: the reference arm (`--impl reference`, the FP64 oracle as it stands) prints
one JSON line with the keys the driver reads; under torchrun only rank 0 prints (other ranks exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, extra_args=()):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "1",
                           "--warmup", "1", *extra_args], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=600)


def test_reference_arm_prints_one_json_line():
    p = _run()
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "pair-evals/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["config"]["workload"] == "tiny" and d["steps"] == 1 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_are_silent():
    p = _run({"RANK": "1", "LOCAL_RANK": "1", "WORLD_SIZE": "2"}, ("--gpus", "2"))
    assert p.returncode == 0, p.stderr[-2000:]
    assert p.stdout.strip() == ""


def test_gpus_n_never_runs_a_silent_single_rank():
    # the native arm with --gpus 2: without WORLD_SIZE it must start 2 ranks itself (it needs 2 visible GPUs —
    # none here, so it stops with a message); under torchrun the world size must equal --gpus
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1", "--warmup", "1"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode != 0 and "needs 2 visible GPUs" in p.stderr and p.stdout.strip() == ""
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--steps", "1", "--warmup", "1"], cwd=ROOT,
                       env=dict(env, RANK="0", LOCAL_RANK="0", WORLD_SIZE="2"), capture_output=True, text=True,
                       timeout=600)
    assert p.returncode != 0 and "WORLD_SIZE=2" in p.stderr
