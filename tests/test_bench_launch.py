"""bench.py's launch contract: `--gpus N` without a launcher spawns N ranks itself (one process
per GPU under torch.distributed.run on 127.0.0.1) and rank 0 prints one JSON line with
n_gpus == N (VERDICT r1 'Next round' #2)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    lines = []
    for ln in out.splitlines():
        ln = ln.strip()
        if ln.startswith("{") and ln.endswith("}"):
            try:
                lines.append(json.loads(ln))
            except ValueError:
                pass
    return lines


def test_reference_arm_spawns_ranks():
    """CPU: the reference arm (the oracle) under a self-spawned 2-rank launch: rank 0 alone
    prints the line, the other rank exits 0."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--config", "c1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout[-2000:]
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_gpus_must_match_launcher():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1"], capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu():
    """GPU: `bench.py --gpus 2 --dist-backend gloo` on one GPU: two TIME parts, correlators
    all-reduced, one JSON line with n_gpus == 2."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--c4", "0", "--config", "c2s"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout[-3000:]
    assert lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0 and lines[0]["e2e"]["value"] > 0
