"""B200-native scenario-tree stochastic MPC solver (arXiv:1604.01074).

Drop-in for the accelerated dual proximal gradient path of the reference
``treesmpc`` package: same entry points and data layout, with every APG
iteration executed on the GPU by hand-written sm_100a kernels (``csrc/``)
behind the C ABI of ``include/tsmpc.h``.
"""

from .errors import DeviceError, DimensionError, ParseError, TreeSmpcError, ValidationError
from .model import NetworkModel, check_model, validate_model
from .tree import DemandForecast, ScenarioTree, node_demands
from .points import DualPoint, PrimalPoint, SplitPoint
from .precompute import (DualScaling, EliminationBasis, FactorCache, StageCache,
                         build_stage_cache, compute_basis, compute_preconditioner,
                         factor_step, lift_controls, particular_solution, theta_schedule,
                         theta_update)
from .engine import (SolverConfig, SolveReport, adjoint_H, apply_H, compute_lambda,
                     extrapolate, prox_g, smooth_cost, solve)
from .factor import SolveContext, solve_step

__version__ = "0.1.0"
