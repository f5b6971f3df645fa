"""O4 — tree scheduler, Alg. 4-8 (§III-B).

TEST INFRASTRUCTURE (see oracle/__init__.py).  Follows the pseudocode line by
line with the corrections and pins of DESIGN.md §Readings:
  G-2 Alg. 5 l.20 adds the individual gain igain, not g   (P:574 vs text P:587)
  G-3 Alg. 7 l.14 is x.outAv = x.outAv - u                 (P:663 vs text P:695)
  G-4 Alg. 8 l.19 INMMEM = INMEM
  T-1 ties in max tgain -> lowest tree id                  (Alg. 4 l.4)
  T-2 "topologically sorted order from left to right"
      = post-order DFS from the tree root, left operand first, skipping
        members that are no longer AVAIL
  T-3 members processed by an earlier tree are skipped; leaves get PROCESS-NODE
  T-4 the selected tree's own gains are updated too (moot)
  T-5 trees are closed under operands, so the static igain stays exact.
`recompute_gains` is the from-scratch gain of P:517-519 (M - M'), used
only by tests to pin the incremental bookkeeping.
"""
import heapq

AVAIL, INMEM, RELEASED = "AVAIL", "INMEM", "RELEASED"


class CounterUnderflow(Exception):
    pass


class TreeScheduler:
    def __init__(self, dag):
        self.dag = dag
        self._tr_init()

    # Alg. 5 TR-INIT ---------------------------------------------------
    def _tr_init(self):
        dag = self.dag
        self.state = {u: AVAIL for u in dag.nodes}
        self.outAv = {u: set(n.parents) for u, n in dag.nodes.items()}
        self.ctree = {u: list(dag.ctree[u]) for u in dag.nodes}
        self.members = {t: dag.trees[t][1] for t in dag.tree_ids}
        self.pred = {t: set() for t in dag.tree_ids}
        self.succ = {u: set() for u in dag.nodes}        # {T : u in T.pred}
        self.cgain = {t: 0 for t in dag.tree_ids}
        self.tgain = {t: 0 for t in dag.tree_ids}
        self.tau = {}
        self.delta = {}
        g = {}
        for t in dag.tree_ids:                            # l.10-15
            for u in self.members[t]:
                g[(u, t)] = len(self.outAv[u])
        for v, vn in dag.nodes.items():                   # l.16-20: edges (u, v)
            for u in vn.child:
                for t in self.ctree[u]:
                    if v in self.members[t]:
                        g[(u, t)] -= 1
        self.igain = {}
        for (u, t), gv in g.items():                      # l.21-27
            self.igain[(t, u)] = 0 if gv == 0 else -dag.nodes[u].size
            self.tgain[t] += self.igain[(t, u)]           # G-2: igain, not g

    # Alg. 4 TR-SCHEDULER ----------------------------------------------
    def run(self, on_select=None):
        """Returns the contraction order.  on_select(tid, {alive tid: tgain}) is
        called at every selection, before PROCESS-CTREE (test hook)."""
        alive = set(self.dag.tree_ids)
        self.version = {t: 0 for t in alive}
        heap = [(-self.tgain[t], t, 0) for t in alive]
        heapq.heapify(heap)
        self._heap = heap
        self.order = []
        self.tree_order = []
        while alive:
            while True:                                   # lazy max-heap, key (-tgain, id) (T-1)
                ng, t, ver = heapq.heappop(heap)
                if t in alive and ver == self.version[t]:
                    break
            if on_select is not None:
                on_select(t, {x: self.tgain[x] for x in alive})
            self.tree_order.append(t)
            self._alive = alive
            self.process_ctree(t)
            alive.discard(t)
        return self.order

    def _touch(self, t):
        if hasattr(self, "_alive") and t in self._alive:
            self.version[t] += 1
            heapq.heappush(self._heap, (-self.tgain[t], t, self.version[t]))

    # Alg. 6 PROCESS-CTREE ---------------------------------------------
    def topo_members(self, t):
        """T-2: post-order DFS from the root, left operand first, AVAIL members only."""
        out = []
        seen = set()
        stack = [(self.dag.trees[t][0], 0)]
        while stack:
            u, i = stack.pop()
            if i == 0:
                if u in seen or self.state[u] != AVAIL:
                    continue
                seen.add(u)
            ch = self.dag.nodes[u].child
            if i < len(ch):
                stack.append((u, i + 1))
                stack.append((ch[i], 0))
            else:
                out.append(u)
        return out

    def process_ctree(self, t):
        for u in self.topo_members(t):
            n = self.dag.nodes[u]
            if n.child:
                for v in n.child:
                    self.process_child(u, v)
                self.order.append(u)
            self.process_node(u)

    # Alg. 7 PROCESS-CHILD ---------------------------------------------
    def process_child(self, u, x):
        size = self.dag.nodes[x].size
        for t in list(self.succ[x]):                      # T_i : x in T_i.pred
            key = (x, t)
            if u in self.members[t]:                      # cases 1.a-1.c
                if self.tau[key] == 1 and self.delta[key] == 0:
                    self.cgain[t] -= size                 # case 1.a
                    self.tgain[t] -= size
                    self._touch(t)
                self.tau[key] -= 1
                if self.tau[key] < 0:
                    raise CounterUnderflow("tau(%d,%d)" % key)
                if self.tau[key] == 0:
                    self.pred[t].discard(x)
                    self.succ[x].discard(t)
            else:                                         # cases 2.a-2.b
                if self.delta[key] == 1:
                    self.cgain[t] += size                 # case 2.a
                    self.tgain[t] += size
                    self._touch(t)
                self.delta[key] -= 1
                if self.delta[key] < 0:
                    raise CounterUnderflow("delta(%d,%d)" % key)
        self.outAv[x].discard(u)                          # G-3
        if not self.outAv[x]:
            self.state[x] = RELEASED

    # Alg. 8 PROCESS-NODE ----------------------------------------------
    def process_node(self, u):
        size = self.dag.nodes[u].size
        for t in self.ctree[u]:                           # l.1-2 individual gains
            self.tgain[t] -= self.igain[(t, u)]
            self._touch(t)
        S = []                                            # l.3-12
        in_s = set()
        n_out = len(self.outAv[u])
        for v in self.outAv[u]:
            for t in self.ctree[v]:
                key = (u, t)
                if t not in in_s:
                    self.tau[key] = 0
                    self.delta[key] = n_out
                    in_s.add(t)
                    S.append(t)
                    self.pred[t].add(u)
                    self.succ[u].add(t)
                self.delta[key] -= 1
                self.tau[key] += 1
        for t in S:                                       # l.13-16 coarse gains
            if self.delta[(u, t)] == 0:
                self.cgain[t] += size
                self.tgain[t] += size
                self._touch(t)
        self.state[u] = RELEASED if not self.outAv[u] else INMEM   # l.17-20 (G-4)

    # invariants / from-scratch gains (tests) --------------------------------------
    def check_tau_delta(self):
        """tau(u,T) + delta(u,T) = |u.outAv| for every INMEM u and T in u's successor trees."""
        for u in self.dag.nodes:
            if self.state[u] != INMEM:
                continue
            for t in self.succ[u]:
                assert self.tau[(u, t)] + self.delta[(u, t)] == len(self.outAv[u]), (u, t)
                assert self.tau[(u, t)] == sum(1 for v in self.outAv[u] if v in self.members[t])

    def recompute_gains(self, alive):
        """From scratch: gain(T) = M - M' where M' is the memory after
        contracting every AVAIL member of T on top of the current resident set."""
        dag = self.dag
        resident = {u for u in dag.nodes if self.state[u] == INMEM}
        M = sum(dag.nodes[u].size for u in resident)
        out = {}
        for t in alive:
            done = {u for u in self.members[t] if self.state[u] == AVAIL}
            processed = lambda v: self.state[v] != AVAIL or v in done  # noqa: E731
            after = set()
            for u in resident | done:
                if any(not processed(p) for p in dag.nodes[u].parents):
                    after.add(u)
            out[t] = M - sum(dag.nodes[u].size for u in after)
        return out


def schedule(dag, on_select=None):
    s = TreeScheduler(dag)
    order = s.run(on_select)
    schedule.last = s
    return order
