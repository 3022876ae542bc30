"""bench.py plumbing on CPU: --gpus 2 without torchrun re-launches itself under
torch.distributed.run (rendezvous on 127.0.0.1); under the reference arm rank 0 alone times the
oracle and prints the one JSON line, the other rank exits 0 without work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_spawns_two_ranks_and_prints_one_line():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["HCOV_ORACLE_THREADS"] = "2"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--config", "C1", "--cpu-sample", "512"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "evals/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["value"] > 0 and d["higher_is_better"] is True
