"""ORACLE -- test infrastructure only.

A plain, slow, obviously-correct CPU implementation (numpy, fp64 arithmetic)
of what the Adaptive SGD hot path computes (arXiv 2110.07029, /root/reference
PAPER.md).  Citations "P:N" are PAPER.md line numbers.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2110_07029_b200``) never imports it and shares no code with it; the
only shared module is ``synthgen`` (seeded inputs, no method arithmetic).

Modules
  model   forward / loss / gradients / SGD step of the sparse-input MLP
          (section 2.1, section 5.1; readings R1-R4)
  csr     batch slicing and the feature/label transposes (brute force)
  sched   stream order, replay routing, Alg. 1,
          Alg. 2 weights
  merge   replica norm, weighted merge + momentum
  train   the whole Adaptive SGD loop (mega-batches)

Parity status: every function is pinned by a test in tests/test_oracle_*.py
against something other than itself (closed forms, finite differences,
library routines, hand-worked examples under tests/golden/), except the
long-run training trajectory (time-to-accuracy), which is "parity unpinned":
the paper prints no numbers for it (figures only).
"""
