"""Configuration objects with the reference's names, fields and defaults.

Mirrors linesearch.Bracket (linesearch.py:80-97), ccd.CcdConfig
(ccd.py:45-67) and locus.LocusConfig (locus.py:41-71).  The solver also
accepts the reference's own config objects unchanged (duck-typed by field).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .errors import InvalidInputError

LINE_SEARCHES = ("exact_median", "ternary", "quadrature")
OUTER_SEARCHES = ("ternary", "quadrature")
DEFAULT_LAMBDA_FLOOR = 1e-9


@dataclass(frozen=True)
class Bracket:
    lo: float
    hi: float

    def __post_init__(self):
        if not (math.isfinite(self.lo) and math.isfinite(self.hi)):
            raise InvalidInputError("bracket endpoints must be finite")
        if not self.lo < self.hi:
            raise InvalidInputError(f"bracket needs lo < hi, got [{self.lo}, {self.hi}]")

    @property
    def width(self) -> float:
        return self.hi - self.lo

    @property
    def mid(self) -> float:
        return 0.5 * (self.lo + self.hi)


@dataclass(frozen=True)
class CcdConfig:
    line_search: str = "exact_median"
    sweep_tolerance: float = 1e-10
    max_sweeps: int = 500
    frozen_axis: int | None = None

    def __post_init__(self):
        if self.line_search not in LINE_SEARCHES:
            raise InvalidInputError(f"unknown line search {self.line_search!r}")
        if self.sweep_tolerance <= 0:
            raise InvalidInputError("sweep_tolerance must be positive")
        if self.max_sweeps < 1:
            raise InvalidInputError("max_sweeps must be at least 1")


@dataclass(frozen=True)
class LocusConfig:
    outer_axis: int | None = None
    outer_search: str = "ternary"
    outer_tolerance: float = 1e-9
    inner: CcdConfig = field(default_factory=CcdConfig)
    initial_bracket: Bracket | None = None
    outer_probes: int = 8
    outer_max_iterations: int = 200

    def __post_init__(self):
        if self.outer_search not in OUTER_SEARCHES:
            raise InvalidInputError(f"unknown outer search {self.outer_search!r}")
        if self.outer_tolerance <= 0:
            raise InvalidInputError("outer_tolerance must be positive")


def locus_params(cfg, lambda_floor: float = DEFAULT_LAMBDA_FLOOR, d: int | None = None):
    """Translate a (reference or local) LocusConfig into the C ABI struct."""
    from ._lib import LocusParams

    cfg = cfg if cfg is not None else LocusConfig()
    inner = getattr(cfg, "inner", None) or CcdConfig()
    if getattr(inner, "line_search", "exact_median") != "exact_median":
        raise InvalidInputError("the CUDA path implements the exact weighted-median inner step only "
                                "(CcdConfig.line_search='exact_median', the reference default)")
    if cfg.outer_search not in OUTER_SEARCHES:
        raise InvalidInputError(f"unknown outer search {cfg.outer_search!r}")
    if cfg.outer_tolerance <= 0:
        raise InvalidInputError("outer_tolerance must be positive")
    if cfg.outer_probes < 3:
        raise InvalidInputError("probes must be at least 3")
    if cfg.outer_max_iterations < 1:
        raise InvalidInputError("max_iterations must be at least 1")
    if d is not None and cfg.outer_axis is not None and not 0 <= cfg.outer_axis < d:
        raise InvalidInputError(f"axis {cfg.outer_axis} out of range for d={d}")
    p = LocusParams()
    p.outer_axis = -1 if cfg.outer_axis is None else int(cfg.outer_axis)
    p.outer_search = OUTER_SEARCHES.index(cfg.outer_search)
    p.outer_tolerance = float(cfg.outer_tolerance)
    p.outer_probes = int(cfg.outer_probes)
    p.outer_max_iterations = int(cfg.outer_max_iterations)
    br = cfg.initial_bracket
    if br is not None:
        p.has_bracket = 1
        p.bracket_lo, p.bracket_hi = float(br.lo), float(br.hi)
    else:
        p.bracket_lo, p.bracket_hi = -1.0, 1.0
    p.inner_sweep_tol = float(inner.sweep_tolerance)
    p.inner_max_sweeps = int(inner.max_sweeps)
    if not (math.isfinite(lambda_floor) and lambda_floor > 0):
        raise InvalidInputError("lambda_floor must be finite and > 0")
    p.lambda_floor = float(lambda_floor)
    return p
