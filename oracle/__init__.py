"""ORACLE — plain, slow, obviously-correct CPU implementation of the hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything under
oracle/.  The product path (paper_2511_02257_b200/) never imports it, and the
oracle never imports the product path: they share no code, headers, tables or
helpers.  The only shared module is synth/ (seeded input generators, no
method arithmetic).

Every function cites the PAPER.md passage it follows ("P:<line>" = PAPER.md
line number; SURVEY §8(c) readings "G-n / S-n / T-n / E-n / V-n" are listed in
DESIGN.md §Readings).  Parts:

  dag.py      O1  DAG formation, node types, ranks (Eq. 1), F_v/F_e
  memory.py   O2  §II-C memory model: M_i, transient, peak
  sibling.py  O3  Alg. 1-3 sibling scheduler
  tree.py     O4  Alg. 4-8 tree scheduler (+ from-scratch gains)
  lru.py      O5  capacity-limited LRU device plan
  optimum.py  O6  exact min-peak by DP / brute force
  values.py   O7  MM1/BM1/BB2/TR_MM contractions + correlators          P:54, DESIGN V-1
  partition.py    multi-GPU partition (time slices / tree chunks)       P:1053, DESIGN §Multi-GPU

Parity status of each part is in DESIGN.md §Oracle pins; every part is pinned
(no "parity unpinned" entries at present).
"""
