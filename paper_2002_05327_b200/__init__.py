"""B200-native diagonal-sweeping DDM hot path (drop-in for `diagsweep`).

Public names follow `diagsweep/__init__.py:26-54` for the hot path
(SURVEY §8): geometry and partition metadata, PML operators, the GPU
factorization cache, `diagonal_sweep_solve` and `gmres`, each additionally
batched over right-hand sides.  The drivers around it (SURVEY §8(f) rank
4: config loader, `solve` / `decay` / `precond-study` commands and their
file artifacts) are in `runconfig`, `drivers`, `artifacts` and `cli`
(`python -m paper_2002_05327_b200`).  Out of scope: the pipeline timing
model and the semi-analytic reference solution (convergence study).
"""

from .ddm import (
    DdmReport,
    SweepPlan,
    build_global_operator,
    build_operators,
    content_cuts,
    additive_ddm_solve,
    diagonal_sweep_solve,
    emits,
    octant_exactness_check,
    restrict_source,
    solve_cuts,
    source_directions,
)
from .artifacts import dump_field, load_field, load_velocity, save_velocity, write_pgm
from .drivers import decay_history, fit_decay_rate, solve_once
from .errors import ConfigurationError, ModelError, SolverError
from .grid import ComplexField, Grid, Window, make_grid
from .krylov import SolveReport, gmres, gmres_batched
from .media import (
    ConstantModel,
    LayeredModel,
    RasterModel,
    constant_model,
    gaussian_source,
    layered_model,
    point_shots,
    raster_model,
)
from .partition import Partition, beta_hat, make_partition, steps_per_sweep, sweep_step_of
from .pml import DiscreteOperator, PmlProfile, assemble_operator, tuned_sigma_max
from .runconfig import RunConfig, load_config
from .subdomain import FactorizationCache, factorize
from .transfer import next_usable_sweep, rule_allows, similar_direction, transfer_geometry

__version__ = "0.1.0"

__all__ = [
    "ComplexField", "ConfigurationError", "ConstantModel", "DdmReport", "DiscreteOperator",
    "FactorizationCache", "Grid", "LayeredModel", "ModelError", "Partition", "PmlProfile",
    "RasterModel", "SolveReport", "SolverError", "SweepPlan", "Window", "assemble_operator",
    "beta_hat", "build_global_operator", "build_operators", "constant_model", "content_cuts",
    "additive_ddm_solve", "diagonal_sweep_solve", "emits", "factorize", "gaussian_source", "gmres", "gmres_batched",
    "layered_model", "make_grid", "make_partition", "next_usable_sweep",
    "octant_exactness_check", "point_shots", "raster_model", "restrict_source", "rule_allows",
    "similar_direction", "solve_cuts", "source_directions", "steps_per_sweep", "sweep_step_of",
    "transfer_geometry", "tuned_sigma_max",
    "RunConfig", "load_config", "solve_once", "decay_history", "fit_decay_rate",
    "dump_field", "load_field", "write_pgm", "save_velocity", "load_velocity",
]
