"""O2 — the §II-C memory model and schedule validity.

TEST INFRASTRUCTURE (see oracle/__init__.py).

For a sequence of contractions c_1..c_n, processing c_i:
  (i)   bring the leaf tensors c_i depends on into memory, if not there;
  (ii)  perform c_i and produce its output;
  (iii) release the tensors no remaining contraction depends on, including the
        output of c_i (always true for a ROOT).
M_i = memory after (iii); M_0 = 0; M_n = 0; peak = max_i M_i.
Reading G-5: transient_i = memory after (ii), before (iii) — the quantity the
§IV-A trace records after a contract op; transient_peak = max_i.
Reading G-6: leaf loads are lazy (at first use), for every scheduler.
"""


class ScheduleError(Exception):
    pass


def check_schedule(dag, order):
    """Violations of: every non-leaf exactly once; no node before a non-leaf child."""
    errs = []
    contr = set(dag.contractions())
    pos = {}
    for i, u in enumerate(order):
        if u not in dag.nodes:
            errs.append("unknown node %r at %d" % (u, i))
        elif u not in contr:
            errs.append("leaf %r scheduled at %d" % (u, i))
        elif u in pos:
            errs.append("node %r scheduled twice" % u)
        else:
            pos[u] = i
    for u in contr:
        if u not in pos:
            errs.append("missing contraction %r" % u)
    for u, i in pos.items():
        for c in dag.nodes[u].child:
            if c in contr and (c not in pos or pos[c] > i):
                errs.append("node %r before its child %r" % (u, c))
    return errs


def simulate(dag, order, record_sets=False):
    """Replay P:211 steps (i)-(iii).  Returns dict with residency [M_0..M_n],
    transient [T_1..T_n], peak, transient_peak and (optionally) resident sets."""
    errs = check_schedule(dag, order)
    if errs:
        raise ScheduleError("; ".join(errs[:5]))
    remaining = {u: len(n.parents) for u, n in dag.nodes.items()}   # unscheduled dependents
    resident = set()
    used = 0
    residency = [0]
    transient = []
    sets = [frozenset()] if record_sets else None
    for u in order:
        node = dag.nodes[u]
        for c in node.child:                       # (i) load leaves not yet in memory
            if not dag.nodes[c].child and c not in resident:
                resident.add(c)
                used += dag.nodes[c].size
        resident.add(u)                            # (ii) produce the output
        used += node.size
        transient.append(used)
        for c in node.child:                       # (iii) release dead tensors
            remaining[c] -= 1
            if remaining[c] == 0:
                resident.discard(c)
                used -= dag.nodes[c].size
        if remaining[u] == 0:                      # output nothing depends on (ROOT)
            resident.discard(u)
            used -= node.size
        residency.append(used)
        if record_sets:
            sets.append(frozenset(resident))
    out = {"residency": residency, "transient": transient,
           "peak": max(residency), "transient_peak": max(transient) if transient else 0}
    if record_sets:
        out["sets"] = sets
    return out
