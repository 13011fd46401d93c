"""ORACLE — test infrastructure only (not part of the product path).

A plain, slow, obviously-correct float64 CPU implementation of what the hot
path computes, written from the paper (arXiv 1512.04564 = PAPER.md) and the
readings in DESIGN.md:

  * `projector`  — SF forward/back projector (C, sf_oracle.c), regulariser
                   gradient/curvature (C), ctypes wrappers.
  * `alg`        — Algorithm 1 verbatim in numpy, Alg. 2
                   (PAPER.md:358-372), unrelaxed OS-LALM, OS-SQS, Eq. 37.
  * `dense`      — tiny dense-matrix tools: literal Eq. 25 iteration with
                   G^{1/2} from eigh, Eq. 33, dense PWLS solve.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with
`paper_1512_04564_b200/` and never imports it.

Parity status per function is listed in DESIGN.md "Oracle pins".  Algorithm 1
with M > 1 (P9 in SURVEY.md 8c.4) is pinned by reduction: on a scan whose
subsets are exact copies of each other (M pitch-0 turns) the ordered-subsets
gradient is exact and the M-subset iterates must equal the M = 1 iterates,
which are pinned to the literal Eq. 25 and to the dense PWLS minimiser
(tests/test_oracle_alg.py P7, P9).  No external value exists for M > 1 on
the BASELINE configs themselves.
"""
