"""bench.py's launcher and CPU reference arm, without a GPU.

* `--gpus N` outside torch.distributed re-launches bench.py as N ranks (torch.distributed.run,
  127.0.0.1 rendezvous); `--dry-run` makes every rank join a gloo group, so the line reports the
  world the driver's SCALE run would get.
* `--impl reference` runs the reference's own prefill_with_reuse (baseline/_ref when installed,
  else the oracle port) at full depth and prints the contract's line.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_flag_launches_n_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    ln = _line(p.stdout)
    assert ln["n_gpus"] == 2 and ln["ranks_joined"] == 2


def test_reference_arm_full_depth_c1():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "C1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    ln = _line(p.stdout)
    assert ln["impl"] == "reference" and ln["unit"] == "ms" and ln["value"] > 0
    assert ln["cpu_baseline"]["kind"] in ("reference", "port") and ln["cpu_baseline"]["cores"] >= 1
    assert "full depth (4/4 layers)" in ln["cpu_baseline"]["sample"]
    assert ln["e2e"]["h2d_bytes_per_step"] == 0 and ln["warmup"] >= 3
