"""Scheduler comparison report (the paper's Fig. 6-7 / Table III-IV
metrics on synthetic workloads): RS-GS-like baseline vs sibling vs tree
(LRU eviction, E-1) and tree with next-use eviction (E-9, "tree+nu").

For each workload and seed: logical peak and transient peak (§II-C), and under a device
capacity (default: the workload's cap, else a fraction of the RS-GS peak) the LRU plan's
evictions, transfers and bytes moved, plus scheduling wall time.  Values are normalised to
RS-GS as in Fig. 7 (lower is better).  Everything runs in libcc.so (host-only context).

Usage: python tools/compare_schedulers.py [--seeds 10] [--cap-frac 0.75] [--json out.json]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_02257_b200 import cc  # noqa: E402
from synth import dags  # noqa: E402

ALGOS = (("rsgs-like", cc.CC_RSGS, False), ("sibling", cc.CC_SIBLING, False), ("tree", cc.CC_TREE, False),
         ("tree+nu", cc.CC_TREE, True))   # tree order, next-use eviction (reading E-9)


def workloads(seed):
    return [
        ("c2 pi-pi (MxM)", dags.config_c2(seed=seed), None),
        ("c4 two-baryon (deuteron-like)", dags.config_c4(seed=seed), 32 * 10 ** 9),
        ("c5 MxM sweep N=256", dags.config_c5(N=256, seed=seed), None),
    ]


def run(seeds, cap_frac):
    rows = []
    for seed in range(1, seeds + 1):
        for name, w, cap in workloads(seed):
            c = cc.Context(-1)
            c.load_workload(w)
            base = {}
            res = {}
            for label, algo, _ in ALGOS:
                _, st = c.schedule(algo)
                res[label] = {"peak": st["peak"], "transient_peak": st["transient_peak"],
                              "sched_ms": st["sched_seconds"] * 1e3}
            cap_b = cap if cap is not None else int(cap_frac * res["rsgs-like"]["transient_peak"])
            for label, algo, nu in ALGOS:
                try:
                    _, st = c.schedule(algo, cap_bytes=cap_b, evict_next_use=nu)
                    res[label].update(evictions=st["evictions"], transfers=st["h2d_count"] + st["d2h_count"],
                                      moved_bytes=st["h2d_bytes"] + st["d2h_bytes"])
                except cc.CCError as e:
                    res[label].update(evictions=None, transfers=None, moved_bytes=None, error=e.code)
            rows.append({"workload": name, "seed": seed, "cap_bytes": cap_b, "results": res})
    return rows


def summarise(rows):
    out = []
    names = sorted({r["workload"] for r in rows}, key=lambda n: [r["workload"] for r in rows].index(n))
    for name in names:
        rs = [r for r in rows if r["workload"] == name]
        line = {"workload": name, "seeds": len(rs)}
        for metric in ("peak", "transient_peak", "evictions", "transfers", "moved_bytes", "sched_ms"):
            for label, _, _ in ALGOS[1:]:
                ratios = []
                for r in rs:
                    b, v = r["results"]["rsgs-like"].get(metric), r["results"][label].get(metric)
                    if b is None or v is None:
                        continue
                    ratios.append(v / b if b else (1.0 if v == 0 else float("inf")))
                line["%s/%s" % (label, metric)] = float(np.median(ratios)) if ratios else None
            wins = sum(1 for r in rs if r["results"]["tree"]["peak"] <= r["results"]["rsgs-like"]["peak"])
            line["tree_peak_le_rsgs_seeds"] = wins
        out.append(line)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=10)
    ap.add_argument("--cap-frac", type=float, default=0.75)
    ap.add_argument("--json")
    a = ap.parse_args()
    rows = run(a.seeds, a.cap_frac)
    summ = summarise(rows)
    print("median ratio vs RS-GS-like over %d seeds (lower is better; cap = workload cap or %.2f x RS-GS "
          "transient peak)" % (a.seeds, a.cap_frac))
    hdr = "%-32s %-8s %8s %10s %9s %9s %9s %9s" % ("workload", "sched", "peak", "trans.peak", "evict",
                                                   "transfers", "bytes", "sched_t")
    print(hdr)
    for s in summ:
        for label, _, _ in ALGOS[1:]:
            def f(m):
                v = s.get("%s/%s" % (label, m))
                return "%.3f" % v if v is not None else "-"
            print("%-32s %-8s %8s %10s %9s %9s %9s %9s" % (s["workload"], label, f("peak"), f("transient_peak"),
                                                            f("evictions"), f("transfers"), f("moved_bytes"),
                                                            f("sched_ms")))
        print("%-32s tree peak <= RS-GS peak in %d/%d seeds" % ("", s["tree_peak_le_rsgs_seeds"], s["seeds"]))
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"rows": rows, "summary": summ}, f, indent=1)


if __name__ == "__main__":
    main()
