"""GPU parity of the peer-HBM tier (readings E-10, E-11) on one GPU: the
peer tier region and the peer-homed leaves' copies are buffers on the same device (a loopback
stand-in for a peer GPU's HBM: the executor issues the same cudaMemcpyAsync(cudaMemcpyDefault)
it issues for a CUDA IPC mapping of a peer's buffer).  Values match the oracle, and the bytes
the executor enqueues on each path (H2D, D2H, peer in, peer out) equal the oracle plan's."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from synth import dags  # noqa: E402
from oracle import values, lru  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu, assert_roots_close, assert_corr_close  # noqa: E402
from paper_2511_02257_b200 import cc  # noqa: E402


def _small_c4():
    return dags.config_c4(N=16, Lt=2, S=4, n_snk=3, n_src=3, n_mes=4, n_trees=16)


@pytest.mark.parametrize("flags", [0, 16, 64])
@pytest.mark.parametrize("nu", [False, True])
@pytest.mark.parametrize("peer", ["tier", "tier+homed", "homed"])
def test_peer_tier_values_and_bytes(flags, nu, peer):
    w = _small_c4()
    dag = Dag(w)
    baryon = 16 * w.Lt * w.S * w.N ** 3
    cap = 5 * baryon
    leaves = sorted(n[0] for n in w.nodes if n[1] in (dags.LEAF_M, dags.LEAF_B))
    homed = set(leaves[::2]) if "homed" in peer else set()
    pc = 2 * baryon if "tier" in peer else 0
    ctx, roots, corr, st, ex = run_gpu(w, cap=cap, flags=flags, evict_next_use=nu, peer_cap=pc, peer_leaves=homed,
                                       peer_tier_mb=8 if pc else 0, arena_mb=64)
    r_or = values.evaluate(dag, lambda u: values.synthetic_leaf(w, u, dag.nodes[u].op))
    assert_roots_close(roots, r_or)
    assert_corr_close(dag, r_or, corr, values.correlators(dag, r_or))
    order, _ = ctx.schedule(cc.CC_TREE, cap_bytes=cap, evict_next_use=nu, peer_cap_bytes=pc, peer_leaves=homed)
    p = lru.plan(dag, order, cap, policy="next_use" if nu else "lru", peer_cap=pc, peer_leaves=homed)
    assert st["evictions"] == p["evictions"] > 0
    if pc:
        assert p["p2p_out_count"] > 0
    assert (ex["h2d_bytes"], ex["d2h_bytes"], ex["p2p_in_bytes"], ex["p2p_out_bytes"]) == \
        (p["h2d_bytes"], p["d2h_bytes"], p["p2p_in_bytes"], p["p2p_out_bytes"])


def test_peer_tier_required_region():
    w = _small_c4()
    baryon = 16 * w.Lt * w.S * w.N ** 3
    with pytest.raises(cc.CCError) as ei:
        run_gpu(w, cap=5 * baryon, peer_cap=2 * baryon, arena_mb=64)     # no cc_set_peer_tier
    assert ei.value.code == "STATE"
