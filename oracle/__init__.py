"""CPU oracle for the hprop matvec path -- TEST INFRASTRUCTURE ONLY.

Nothing in the product package (`paper_1403_3511_b200/`) may import, call or
link anything from this directory.  It is imported only by `tests/`, by
`__graft_entry__.smoke()` (as the checker) and by `bench.py`'s CPU-baseline
leg / `--impl reference` arm.

`hprop_oracle` restates, in numpy, the reference algorithm of the
`hprop` 0.1.0 package (/root/reference/pkg/src/hprop) for the hot path
only: index-set enumeration and neighbour tables, the matrix-free Galerkin
matvec (coordinate operator, Chebyshev sweeps, ordered term products,
oscillator diagonal, exact square sum), the Chebyshev interpolation that
produces the term list, and the Lanczos / Magnus propagation loop.  Each
function cites the reference file:line it follows.

Parity pinning: the restatement is checked against golden vectors that were
produced by importing the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`), including SHA-256
digests of the full-size cfg3/cfg5 index sets and neighbour tables.
"""
