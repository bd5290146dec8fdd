"""bench.py's N > 1 path (the driver's scaling run: torchrun, one rank per GPU) on a one-GPU
box: TS_BENCH_ONE_GPU=1 puts both ranks on cuda:0 over gloo, so the view sharding, gradient
all-reduce, barriers, max-over-ranks timing and the single rank-0 JSON line run end to end
(the numbers are not measurements).  The reference arm under torchrun: rank 0 alone prints."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(args, port, extra_env):
    env = dict(os.environ, **extra_env)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", *args]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 only
    return json.loads(lines[0])


@pytest.mark.parametrize("sync_free", ["0", "1"])
def test_bench_two_ranks_one_json_line(sync_free):
    """threaded lanes and the sync-free path (the default when ranks share few host CPUs)"""
    d = _torchrun(["--steps", "1", "--warmup", "3"], 29611 + int(sync_free),
                  {"TS_BENCH_ONE_GPU": "1", "TS_SYNC_FREE": sync_free})
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["steps"] == 1 and d["warmup"] == 3
    assert d["config"]["global_batch_views"] == 2 * d["config"]["views_per_gpu"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["cpu_baseline"] is None  # (rank 0 at N = 1 only)


def test_reference_arm_two_ranks():
    d = _torchrun(["--impl", "reference", "--steps", "1", "--warmup", "1"], 29613, {})
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
