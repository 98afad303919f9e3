"""Drop-in ``elimination`` module (reference ``pkg/src/treesmpc/elimination.py``)."""

from .precompute import (EliminationBasis, StageCache, build_stage_cache, compute_basis,
                         lift_controls, particular_solution)

__all__ = ["EliminationBasis", "StageCache", "compute_basis", "particular_solution",
           "build_stage_cache", "lift_controls"]
