"""paper_2405_03584_b200 — B200-native (sm_100a) hot path of the GPU interior point method
of arxiv 2405.03584: Jacobi-PCG on the condensed IPM Newton system plus the per-iteration
vector kernels, behind the C ABI of include/ipm.h (libipm.so); the closed-loop SQP driver
of include/sqp.h on top."""
from . import _lib
from .qp import QP, make_options
from .sqp import SQP, make_sqp_options

__all__ = ["QP", "make_options", "SQP", "make_sqp_options", "_lib"]
