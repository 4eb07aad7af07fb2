"""bench.py's JSON-line contract, at a reduced size (the driver runs the full one)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run_bench(*extra, launcher=()):
    r = subprocess.run([sys.executable, *launcher, str(ROOT / "bench.py"), "--steps", "3",
                        "--warmup", "3", "--rays", "65536", "--res", "65", "--width", "320",
                        "--height", "180", "--keyframes", "3", "--no-cpu", *extra],
                       capture_output=True, text=True, cwd=str(ROOT), timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    # stdout is exactly the one JSON line (NCCL's banner etc. go to stderr)
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 1 and lines[0].startswith("{"), r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_has_the_contract_keys():
    d = run_bench()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks", "tracking"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 65536 * 12 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # achieved counts compulsory HBM bytes, so it is a real fraction of the peak
    assert 0 < r["frac"] <= 1.2
    assert d["tracking"]["frames_per_s"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_bench_distributed_path_prints_one_line():
    """The N>1 code path (torchrun, NCCL, fused p2p exchange) at world size 1."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    d = run_bench("--dist-path", "--no-tracking",
                  launcher=("-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                            "--master-addr", "127.0.0.1", "--master-port", str(port)))
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["exchange"] == "p2p"
    assert d["e2e"]["value"] > 0
