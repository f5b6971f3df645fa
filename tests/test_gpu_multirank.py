"""Multi-process peer-HBM tier + cross-GPU leaf sharing (readings E-10, E-11): two ranks on the
GPU(s) of this box (tests/multirank_peer_worker.py) — TREES parts, each evicting into the other
rank's HBM through CUDA IPC and reading shared leaves from their owner's HBM.  The summed
correlators equal the oracle's; each rank's executor moved exactly its plan's bytes; across
the job every leaf crossed PCIe once."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from synth import dags  # noqa: E402
from oracle import values  # noqa: E402
from oracle.dag import Dag  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("flags", [0, 16, 64])
@pytest.mark.parametrize("mode", ["plain", "tier", "leaves", "both"])
def test_two_ranks_peer_tier_and_shared_leaves(flags, mode):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "multirank_peer_worker.py"), str(flags), mode],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    res = json.loads(line)
    assert res["world"] == 2 and res["bytes_ok"]
    assert sum(res["evictions"]) > 0 and (sum(res["p2p_out"]) > 0) == (mode in ("tier", "both"))
    w = dags.config_c4(N=16, Lt=2, S=4, n_snk=3, n_src=3, n_mes=4, n_trees=24)
    dag = Dag(w)
    r_or, c_or = values.run_workload(w, dag)
    scale = values.term_scale(dag, r_or)
    for c, want in c_or.items():
        got = np.array(res["corr"][str(c)][0]) + 1j * np.array(res["corr"][str(c)][1])
        assert np.all(np.abs(got - want) <= 1e-10 * scale[c]), c
    # E-11: with shared leaves no rank's plan fetches a leaf over PCIe (the owners' staging
    # copies each leaf once, outside the plans); without, every leaf crosses PCIe at least once
    leaf_bytes = sum(dag.nodes[u].size for u, n in dag.nodes.items() if not n.child)
    if mode in ("leaves", "both"):
        assert sum(res["h2d_bytes"]) < leaf_bytes
    else:
        assert sum(res["h2d_bytes"]) >= leaf_bytes
