"""bench.py --gpus N outside torchrun re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1 rendezvous) and prints ONE JSON line with
n_gpus = N. Dry-run on CPU through the reference arm (rank 0 alone runs the
oracle pipeline; the other ranks exit 0 without work)."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_gpus2_relaunch_prints_one_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "1", "--warmup", "1", "--ref-seconds", "2"],
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["workload"].startswith("c1")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
