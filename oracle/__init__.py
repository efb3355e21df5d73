"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference's per-frame deformation-tracking path
(/root/reference/pkg/src/deformtrack, arXiv 2007.08576), used to check the B200 product
(paper_2007_08576_b200) and to time the reference algorithm on the host cores.

* ``oracle.kernels``  -- the four numba kernels restated in C (oracle/csrc/oracle_kernels.c,
  built into oracle/_build/liboracle.so), same signatures, same chunked fold order, so
  they reproduce the reference kernels bit for bit (pinned by tests/test_oracle_golden.py
  against fixtures generated from the reference, tests/golden/make_golden.py).
* ``oracle.pipeline`` -- numpy restatement of the Python around those kernels: depth
  normals, basis, assembly, damped Cholesky, step, the LM frame loop, preselection,
  binding, output warp, plus the builder-defined Hamming matcher (north-star part 3a,
  which the reference does not implement: its parity is pinned only by the
  known-answer tests in tests/test_hamming.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference legs
may import this package, and only as the checker or the timed CPU baseline. The product
never imports it; nothing here runs on a GPU.
"""
