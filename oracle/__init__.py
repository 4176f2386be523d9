"""FP64 CPU oracle for LSG-CPD (arXiv 2103.15039) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import, call, link or execute anything under oracle/.  The CUDA product path
(paper_2103_15039_b200/) shares no code with it and never imports it.

Parity status per function: every function below is pinned by a
`-m "not gpu"` test against the paper, closed forms, brute force or textbook special cases, except
the EM *trajectory choice* among stationary points, which is "parity unpinned" beyond the shared
readings (SURVEY §8(c).5 last row).
"""
from ._lib import build  # noqa: F401
from .estep import estep, estep_cf, posterior, sym6, REC  # noqa: F401
from .model import (knn, alpha_from_kappa, local_surface, prepare_target, working_volume,  # noqa: F401
                    sigma2_init, sum_sq_pairs, mean_nn_spacing)
from .mstep import PointStats, newton, mstep, grad_hess_literal  # noqa: F401
from .em import register, register_workload  # noqa: F401
from . import se3, matrix_form, outlier, affine  # noqa: F401
