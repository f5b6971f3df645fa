"""Small c1 / c2 / c4 / c6 DAGs through the dataflow, op-by-op and Ozaki executors, values
checked against the oracle: the workload the compute-sanitizer runs (memcheck, racecheck,
synccheck; tools/sanitize.sh) exercise.  Sizes are tiny so the instrumented kernels finish.

python tools/sanitize_run.py [--flags 0,16,64] [--configs c1,c2,c4,c6]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from synth import dags  # noqa: E402
from oracle import values  # noqa: E402
from oracle.dag import Dag  # noqa: E402
from gpu_helpers import run_gpu  # noqa: E402


def small(name):
    if name == "c1":
        return dags.config_c1(N=32, Lt=2), 0
    if name == "c2":
        return dags.config_c2(N=72, Lt=2, n_loop4=12, n_loop2=2, n_corr=2), 0
    if name == "c4":
        # two-baryon shape at N=16, S=4, a cap that forces evictions and D2H of dressed nodes
        w = dags.config_c4(N=16, Lt=1, S=4, n_snk=3, n_src=3, n_mes=4, n_trees=12)
        return w, 5 * 16 * 4 * 16 ** 3
    if name == "c6":
        return dags.config_c6(N=16, Lt=2, S=4, n_snk=2, n_src=2, n_trees=6), 0
    raise SystemExit("unknown config " + name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--flags", default="0,16,64")
    ap.add_argument("--configs", default="c1,c2,c4,c6")
    a = ap.parse_args()
    worst_all = 0.0
    for name in a.configs.split(","):
        w, cap = small(name)
        dag = Dag(w)
        roots = values.evaluate(dag, lambda u: values.synthetic_leaf(w, u, dag.nodes[u].op))
        for fl in [int(x) for x in a.flags.split(",")]:
            _, got, _, st, ex = run_gpu(w, flags=fl, cap=cap, arena_mb=64)
            worst = max(float(np.max(np.abs(got[t] - roots[t]) / np.abs(roots[t]))) for t in roots)
            worst_all = max(worst_all, worst)
            print("%s flags=%d: %d contractions, evictions %d, d2h %d B, worst rel err %.2e"
                  % (name, fl, st["n_contr"], st["evictions"], st["d2h_bytes"], worst), flush=True)
            assert worst <= 1e-10, (name, fl, worst)
    print("sanitize_run ok, worst %.2e" % worst_all)


if __name__ == "__main__":
    main()
