"""B200-native batched LAD-LASSO solver (drop-in for arxiv/paper_2510_15649's ladlasso hot path).

The reference's public names are mirrored here with the same signatures and results
(bit-identical); the solvers run on the GPU.  Not mirrored: the generic 1-D line searches
over Python callables (``linesearch.PiecewiseLinear1D``, ``SearchConfig``/``SearchResult``,
``expand_bracket``, ``ternary_min``, ``quadrature_min``, ``weighted_median_min``,
``model.axis_restriction``) and the brute-force helpers ``enumerate_vertices`` /
``solve_linear_system`` -- their GPU counterparts live inside the batched kernels.

The reference's solver entry points -- ``solve_locus`` (ternary-chop and
quadrature), ``ccd_descend`` and ``solve_brute`` -- run as hand-written sm_100a
CUDA kernels behind the C ABI in include/ladlasso_b200.h, batched over
(B, n, p) problems.  See DESIGN.md.
"""

from .config import Bracket, CcdConfig, LocusConfig
from .errors import (DegenerateInputError, DeviceError, DimensionMismatchError, InvalidInputError,
                     ProblemTooLargeError, SimplexError, UnboundedDirectionError)
from .solver import (validate_result, BatchedSolveResult, Coefficients, Dataset, ProblemSpec, SolveResult, axiswise_minimum_batched,
                     ccd_descend, ccd_descend_batched, evaluate_objective, evaluate_objective_batched,
                     is_axiswise_minimum, solve_brute, solve_brute_batched, solve_ccd, solve_locus,
                     solve_locus_batched)
from .lp import (LpStandardForm, SimplexConfig, SimplexSolution, dump_lp, formulate, simplex_minimize, simplex_solve,
                 solve_lp, solve_lp_batched)
from .path import solve_lambda_path_batched
from .synth import GenSpec, generate, read_dataset_csv, write_dataset_csv
from .curve import (LocusPoint, axes_by_influence, default_bracket, default_outer_axis, locus_value,
                    perturb_restart, sample_locus, sample_locus_batched)

__version__ = "0.1.0"

__all__ = [
    "BatchedSolveResult", "Bracket", "CcdConfig", "Coefficients", "Dataset", "DegenerateInputError", "DeviceError",
    "DimensionMismatchError", "InvalidInputError", "LocusConfig", "ProblemSpec", "ProblemTooLargeError",
    "SolveResult", "UnboundedDirectionError", "ccd_descend", "ccd_descend_batched", "evaluate_objective",
    "evaluate_objective_batched", "solve_brute", "solve_brute_batched", "solve_ccd", "solve_locus",
    "solve_locus_batched", "axiswise_minimum_batched", "is_axiswise_minimum", "LocusPoint", "axes_by_influence",
    "default_bracket", "default_outer_axis", "locus_value", "perturb_restart", "sample_locus", "sample_locus_batched",
    "SimplexConfig", "SimplexSolution", "SimplexError", "solve_lp", "solve_lp_batched",
    "LpStandardForm", "dump_lp", "formulate", "simplex_minimize", "simplex_solve", "GenSpec", "generate",
    "read_dataset_csv", "write_dataset_csv", "validate_result", "solve_lambda_path_batched",
]
