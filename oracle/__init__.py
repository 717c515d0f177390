"""HFReduce CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import, call, link or execute
anything under ``oracle/``.  The product path (``paper_2408_14158_b200``) never
does, and shares no code with it (DESIGN.md §"Oracle").

Contents
  hfr_oracle.py  numpy oracle: rank-ascending fp32 fold, bf16 RNE, scale,
                 the double binary tree construction, tree-order and
                 pair-first-order folds (the bit-exact references for
                 HFR_ALGO_DBT / HFR_ALGO_PAIR_DBT).
  fold.c         plain C twin of the rank-ascending fold (OpenMP over element
                 blocks), used for the timed CPU baseline and cross-checked
                 against hfr_oracle.py in the CPU tests.

Parity status per function (DESIGN.md §"Oracle pins"):
  fold_ascending ........ pinned (exact-rational brute force, closed forms,
                          golden worked examples, n=2 library case, invariants)
  bf16_rne .............. pinned (torch .to(bfloat16), hand-computed ties)
  build_tree / trees .... pinned (SPEC.md invariants for n=1..1024, n=4/8 tables)
  fold_tree ............. pinned (exact-rational brute force of the tree
                          expression, integer closed form, golden example,
                          n=2 reduction to a+b, Higham bound)
  fold_pairfirst ........ pinned (same kinds of pins as fold_tree)
  fold.c ................ pinned against fold_ascending (bit-exact)
"""
