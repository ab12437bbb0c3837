"""bench.py's JSON-line contract on the GPU: the default single-GPU line, and the N > 1 code
path (strong-scaling N-shard with the label all-gather in the step) run as two ranks on one
GPU over gloo -- the same code the driver's multi-GPU run takes with NCCL, one rank per GPU."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks")


def _line(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_single_gpu_line(cuda_device):
    r = subprocess.run([sys.executable, "bench.py", "--config", "cfg1", "--steps", "3", "--warmup", "3",
                        "--no-peaks", "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert all(k in d for k in KEYS) and d["n_gpus"] == 1 and d["value"] > 0
    roof = d["roofline"]
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"]) and roof["kernel"] == "tc"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["single_thread"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 256 * 561 * 4


def test_two_ranks_nshard_gather_path(cuda_device):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--same-device", "--config", "cfg2", "--no-cpu-baseline", "--no-peaks",
           "--steps", "3", "--warmup", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"] == "nshard2" and d["config"]["rows_per_rank"] == 8192
    assert "all_gather" in d["config"]["collective"]
