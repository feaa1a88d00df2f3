"""CPU oracle for the ReCoVer gradient-commit path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
or as the timed CPU baseline — never as the thing measured or shipped.  The
product (paper_2605_11215_b200) never imports it; its data plane fails loudly
without librcv.so.

Contents (each function cites the reference lines it restates, paths under
/root/reference/pkg/src/steadybatch/):
  fold.py      numpy data plane: the masked ascending-id fold, accumulation,
               the canonical dyadic tree, the commit scale, SGD, splitmix lanes
  protocol.py  a from-scratch numpy restatement of one replica world driven
               through run_iteration (comm / buckets / policy / trainer)

Parity pinning: tests/test_oracle_reference.py compares both modules with the
reference itself (imported from /root/reference when present, i.e. in the
build container) and tests/golden/ holds fixtures generated from the
reference by tests/golden/make_golden.py, which travel to the GPU box.
"""
