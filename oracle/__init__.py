"""CPU oracle for the TASER mini-batch-generation path -- TEST INFRASTRUCTURE.

This package restates the reference algorithm (tgadapt, /root/reference/pkg)
in numpy/numba so the CUDA path can be checked on the GPU box, where the
reference is not available.  Each function cites the reference file:line it
follows.  It is pinned against golden vectors produced by the REAL reference
(tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle_golden.py).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import it -- as the checker or the timed CPU baseline, never as the
thing measured or shipped.  The product (paper_2402_05396_b200) never imports
this package.
"""
