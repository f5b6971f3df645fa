"""RS-GS-like baseline scheduler.

TEST INFRASTRUCTURE (see oracle/__init__.py) — also the CPU reference of the C++
`CC_RSGS` scheduler.

PAPER.md §II-A describes Redstar's graph-sorting order (the paper's RS-GS
baseline) only qualitatively: "it sorts the contraction trees based on their
similarity" so "a shared tensor can be released as soon as the contraction trees that need
this tensor are processed".  Readings:
  R-1 similarity of two trees = Jaccard |A∩B| / |A∪B| of their member node sets (members =
      the closure of the root under operands, leaves included);
  R-2 the sort is a greedy chain: start from the lowest tree id, repeatedly append the
      unvisited tree most similar to the tree appended last; ties -> lowest tree id.
      Fractions are compared exactly (a/b > c/d  <=>  a*d > c*b);
  R-3 each tree in chain order contributes its not-yet-contracted non-leaf members in the
      tree scheduler's member order (T-2: post-order DFS from the root, left operand first,
      not descending into contracted nodes); leaves load lazily (G-6);
  R-4 the edge-frequency / complexity weighting of P:119-121 chooses contraction *paths*;
      here paths are fixed by the input DAG, so it has nothing to choose (out of scope).
"""


def tree_chain(dag):
    """R-1, R-2: the similarity chain of tree ids."""
    members = {t: set(dag.trees[t][1]) for t in dag.tree_ids}
    unvisited = set(dag.tree_ids)
    chain = []
    cur = min(unvisited)
    while True:
        chain.append(cur)
        unvisited.discard(cur)
        if not unvisited:
            return chain
        # |cur ∩ t| for every unvisited t sharing a node with cur
        inter = {}
        for u in members[cur]:
            for t in dag.ctree[u]:
                if t in unvisited:
                    inter[t] = inter.get(t, 0) + 1
        if not inter:
            # every similarity is 0: the lowest unvisited id wins the tie
            cur = min(unvisited)
            continue
        best = None                                   # (|A∩B|, |A∪B|, t)
        for t in sorted(inter):                       # ascending id: strict '>' keeps the lowest
            a = inter[t]
            b = len(members[cur]) + len(members[t]) - a
            if best is None or a * best[1] > best[0] * b:
                best = (a, b, t)
        cur = best[2]                                 # positive similarity beats every 0


def member_order(dag, t, done):
    """R-3 / T-2: post-order from the root of tree t, left operand first, skipping (and not
    descending into) contracted nodes; leaves are not emitted."""
    out = []
    seen = set()

    def visit(u):
        if u in seen or u in done:
            return
        seen.add(u)
        for c in dag.nodes[u].child:                  # left operand first
            visit(c)
        if dag.nodes[u].child:
            out.append(u)

    visit(dag.trees[t][0])
    return out


def schedule(dag):
    """The RS-GS-like contraction order (node ids)."""
    done = set()
    order = []
    for t in tree_chain(dag):
        for u in member_order(dag, t, done):
            done.add(u)
            order.append(u)
    return order
