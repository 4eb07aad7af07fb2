"""bench.py's N-GPU launcher on a node with too few GPUs (CPU: this container has
none): `--gpus N` without WORLD_SIZE must refuse loudly, never run N = 1."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_bench_refuses_more_gpus_than_the_node_has():
    import torch
    n = torch.cuda.device_count() + 1
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(max(n, 2)),
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       cwd=str(ROOT), timeout=300,
                       env={k: v for k, v in __import__("os").environ.items()
                            if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert r.returncode == 2, (r.returncode, r.stderr[-2000:])
    assert "refusing to run a smaller world" in r.stderr
    assert r.stdout.strip() == ""
