"""Result and option types of the drop-in boundary.

When the reference package ``hybridlp`` is importable, its own classes are
used (``PdhgParams`` pdhg.py:31-48, ``SolveStats`` pdhg.py:70-77, ``KktPoint``
lp_core.py:145-166, ``TerminationCheck`` lp_core.py:180-206,
``ViolationSummary`` lp_core.py:209-221, ``SolveStatus`` status.py:8-16,
``InvalidModelError`` lp_core.py:27-28, ``StandardFormMap`` lp_core.py:224-247,
``StandardLp`` lp_core.py:106-142), so callers such as the reference's
``hybrid_solve`` and its IPM warm start consume our results unchanged.
Otherwise (e.g. on a GPU box without the reference) field-for-field mirrors
are used.  ``SolveStats`` gains two defaulted fields, ``history`` (one dict
per KKT check) and ``timings`` (wall seconds of the engine's phases); every
existing field is unchanged.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field, make_dataclass
from types import SimpleNamespace

import numpy as np


class _InvalidModelError(ValueError):
    """A model (or point) violates one of its structural invariants."""


class _SolveStatus(enum.Enum):
    OPTIMAL = "Optimal"
    TIME_LIMIT = "TimeLimit"
    STALLED = "Stalled"
    ITERATION_LIMIT = "IterationLimit"
    NUMERICAL_FAILURE = "NumericalFailure"
    INFEASIBLE = "Infeasible"
    UNBOUNDED = "Unbounded"
    ERROR = "Error"


@dataclass
class _PdhgParams:
    eps_rel: float = 1e-4
    max_kkt_passes: int = 200_000
    time_limit_s: float = 10_000.0
    check_every: int = 64
    restart_beta: float = 0.2
    primal_weight_init: float = 1.0

    def __post_init__(self):
        if self.eps_rel <= 0:
            raise ValueError("eps_rel must be positive")
        if self.check_every < 1:
            raise ValueError("check_every must be at least 1")
        if not 0.0 < self.restart_beta < 1.0:
            raise ValueError("restart_beta must lie in (0, 1)")
        if self.primal_weight_init <= 0:
            raise ValueError("primal_weight_init must be positive")


@dataclass
class _KktPoint:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray

    def __post_init__(self):
        self.x = np.asarray(self.x, dtype=float).ravel()
        self.y = np.asarray(self.y, dtype=float).ravel()
        self.z = np.asarray(self.z, dtype=float).ravel()

    def copy(self):
        return _KktPoint(self.x.copy(), self.y.copy(), self.z.copy())

    def is_finite(self) -> bool:
        return bool(np.all(np.isfinite(self.x)) and np.all(np.isfinite(self.y))
                    and np.all(np.isfinite(self.z)))


@dataclass
class _TerminationCheck:
    ok: bool
    primal_lhs: float
    primal_rhs: float
    dual_lhs: float
    dual_rhs: float
    gap_lhs: float
    gap_rhs: float

    @property
    def primal_ok(self) -> bool:
        return self.primal_lhs <= self.primal_rhs

    @property
    def dual_ok(self) -> bool:
        return self.dual_lhs <= self.dual_rhs

    @property
    def gap_ok(self) -> bool:
        return self.gap_lhs <= self.gap_rhs


@dataclass
class _ViolationSummary:
    primal_inf: float
    dual_inf: float
    rel_gap: float
    max_violation: float
    comp_negative: bool = False


@dataclass
class _SolveStats:
    status: _SolveStatus
    iterations: int
    restarts: int
    wall_seconds: float
    termination: _TerminationCheck | None
    max_violation: float


@dataclass
class _StandardFormMap:
    n_general: int
    m_general: int
    n_std: int
    m_std: int
    obj_shift: float
    shifts: np.ndarray
    pos_col: np.ndarray
    neg_col: np.ndarray
    slack_of_row: np.ndarray
    slack_coef: np.ndarray
    bound_var: np.ndarray

    def slack_columns(self) -> np.ndarray:
        return self.slack_of_row[self.slack_of_row >= 0]


def _standard_lp(A, b, c):
    from .instances import Instance

    return Instance("standard", A, np.asarray(b, dtype=float), np.asarray(c, dtype=float))


_cache = None


def resolve() -> SimpleNamespace:
    """The type namespace: the reference's classes if importable, else mirrors."""
    global _cache
    if _cache is not None:
        return _cache
    try:
        from hybridlp import lp_core as L, pdhg as Pm, status as S  # type: ignore

        ns = SimpleNamespace(
            PdhgParams=Pm.PdhgParams, BaseSolveStats=Pm.SolveStats, KktPoint=L.KktPoint,
            TerminationCheck=L.TerminationCheck, ViolationSummary=L.ViolationSummary,
            SolveStatus=S.SolveStatus, InvalidModelError=L.InvalidModelError,
            StandardFormMap=L.StandardFormMap, StandardLp=L.StandardLp,
            reference=True,
        )
    except ImportError:
        ns = SimpleNamespace(
            PdhgParams=_PdhgParams, BaseSolveStats=_SolveStats, KktPoint=_KktPoint,
            TerminationCheck=_TerminationCheck, ViolationSummary=_ViolationSummary,
            SolveStatus=_SolveStatus, InvalidModelError=_InvalidModelError,
            StandardFormMap=_StandardFormMap, StandardLp=_standard_lp,
            reference=False,
        )
    ns.SolveStats = make_dataclass(
        "SolveStats", [("history", list, field(default_factory=list)),
                       ("timings", dict, field(default_factory=dict))],
        bases=(ns.BaseSolveStats,),
    )
    ns.SolveStats.__doc__ = ("SolveStats (pdhg.py:70-77) plus `history`: one dict per "
                             "KKT check (iteration, scores, termination sides, omega, restart), "
                             "and `timings`: wall seconds of the layout build, power "
                             "iteration, iterations and result download.")
    _cache = ns
    return ns


def reset_cache() -> None:
    global _cache
    _cache = None
