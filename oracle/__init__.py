"""CPU oracle for the qnsim per-timestep L-BFGS solver — TEST INFRASTRUCTURE ONLY.

This package is a numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/qnsim`, arXiv 1604.07378).  Every function cites the
reference file:line it restates.  It exists to *check* the B200 path:

* only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
  (`cpu_baseline` / `--impl reference`) may import it;
* the product package `paper_1604_07378_b200` never imports it and has no CPU
  fallback — it fails loudly when its CUDA library is missing.

Parity pinning: `tests/test_oracle_golden.py` checks this oracle against the
golden vectors written by the UNMODIFIED reference (`tests/golden/make_golden.py`,
run in the build container where `/root/reference` exists) and against the
reference's own golden trajectories `twist_lbfgs.csv` / `twist_pd_qn.csv`
(`pkg/frontend/tests/fixtures`), so the oracle is "parity pinned".
"""

from oracle.qnsim_oracle import *  # noqa: F401,F403
