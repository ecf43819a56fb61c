"""bench.py's launch contract on a CPU box: `--gpus N` is never silently a 1-GPU run, and the
reference arm (the float64 oracle on the host cores) prints the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env_extra=None, timeout=300):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=ROOT)


def test_gpus_mismatch_with_world_size_fails_loudly():
    r = run(["--gpus", "2", "--steps", "1", "--warmup", "3"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in r.stderr and "n_gpus" not in r.stdout


def test_gpus_n_without_torchrun_relaunches_under_torchrun():
    """Without WORLD_SIZE, --gpus 2 re-executes under torch.distributed.run (2 ranks); on this
    CPU box the ranks then fail to find a GPU -- the point is that no 1-GPU line is printed."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300, cwd=ROOT)
    assert "torch.distributed.run" in r.stderr and "--nproc-per-node=2" in r.stderr
    assert '"n_gpus": 1' not in r.stdout


def test_reference_arm_prints_contract_line():
    r = run(["--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "tokens/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
