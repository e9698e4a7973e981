"""CPU oracle for the PDHG hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

This package restates, in numpy/scipy, the reference package's restarted
PDHG (`hybridlp.pdhg`, /root/reference/pkg/src/hybridlp/pdhg.py:80-258) and
the KKT metrics it calls (`hybridlp.lp_core`, lp_core.py:106-142,430-485).
Every function cites the reference lines it follows.

Who may use it (and only as the checker / the CPU baseline, never as the
thing measured or shipped):
  * ``tests/``                     -- parity tests against the CUDA path;
  * ``__graft_entry__.smoke()``    -- the one-call GPU-vs-oracle smoke check;
  * ``bench.py``                   -- the ``cpu_baseline`` leg and the
                                      ``--impl reference`` arm.

Pinning: ``oracle/make_golden.py`` imports the real reference from
/root/reference (in the build container only) and writes the golden
fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
restatement against them (bit-for-bit where numpy/scipy versions match).
"""

from .pdhg_port import (  # noqa: F401
    KktPoint,
    PdhgParams,
    Residuals,
    SolveStats,
    SolveStatus,
    TerminationCheck,
    ViolationSummary,
    check_relative_termination,
    estimate_opnorm,
    extract_reduced_costs,
    initial_state,
    pdhg_step,
    residuals,
    run_pdhg,
    violation_summary,
)
from .ruiz_port import ruiz_equilibrate  # noqa: F401
