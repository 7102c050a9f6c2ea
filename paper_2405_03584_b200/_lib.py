"""ctypes binding of libipm.so — argument marshalling only (include/ipm.h is the contract).

Every function here has the C name of the entry point it wraps and forwards plain
pointers; all arithmetic runs in the library's CUDA kernels.  There is no fallback:
if the shared library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPM_LIB") or os.path.join(_HERE, "libipm.so")   # IPM_LIB: diagnostic builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA extension is required; there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

IPM_OK, IPM_NOT_CONVERGED, IPM_ERR_INVALID, IPM_ERR_PCG_BREAKDOWN, IPM_ERR_NONFINITE, IPM_ERR_CUDA, \
    IPM_ERR_OOM, IPM_ERR_NCCL, IPM_ERR_STATE = range(9)
STATUS_NAMES = {0: "ok", 1: "not_converged", 2: "invalid", 3: "pcg_breakdown", 4: "nonfinite", 5: "cuda",
                6: "oom", 7: "nccl", 8: "state"}


class ipm_options(C.Structure):
    _fields_ = [("size", C.c_int32), ("mu_tol", C.c_double), ("mu0_scale", C.c_double),
                ("mu_divisor", C.c_double), ("tau", C.c_double), ("max_ipm_iter", C.c_int32),
                ("pcg_schedule", C.c_int32), ("pcg_rtol_max", C.c_double), ("pcg_rtol_mu_factor", C.c_double),
                ("pcg_rtol_floor", C.c_double), ("pcg_atol", C.c_double), ("pcg_max_iter", C.c_int32),
                ("predictor_corrector", C.c_int32), ("trace", C.c_int32), ("use_graph", C.c_int32),
                ("warm_shift", C.c_double), ("gemv_kernel", C.c_int32), ("pcg_warm_start", C.c_int32),
                ("pcg_system", C.c_int32), ("a_row_split", C.c_int32), ("pcg_single_reduction", C.c_int32),
                ("kernel_timer", C.c_int32)]


class ipm_problem(C.Structure):
    _fields_ = [("n", C.c_int64), ("m", C.c_int64), ("nnz", C.c_int64), ("H", C.c_void_p), ("ldh", C.c_int64),
                ("g", C.c_void_p), ("A_rowptr", C.c_void_p), ("A_col", C.c_void_p), ("A_val", C.c_void_p),
                ("l", C.c_void_p), ("u", C.c_void_p), ("xl", C.c_void_p), ("xu", C.c_void_p),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("comm_kind", C.c_int32), ("comm_handle_host", C.c_void_p),
                ("hess_kind", C.c_int32), ("k", C.c_int32), ("ldu", C.c_int64), ("h0", C.c_void_p),
                ("U", C.c_void_p), ("w", C.c_void_p)]


# comm_kind 3 (include/ipm.h ipm_host_comm): the caller's host allgather, used only at create
IPM_HOST_ALLGATHER = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class ipm_host_comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("allgather", IPM_HOST_ALLGATHER), ("user", C.c_void_p)]


class ipm_stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("ipm_iters", C.c_int32), ("pcg_iters_total", C.c_int64),
                ("pcg_iters_max", C.c_int32), ("pcg_stalls", C.c_int32), ("pcg_restarts", C.c_int32),
                ("mu_final", C.c_double), ("kkt_inf", C.c_double), ("obj", C.c_double),
                ("t_solve_ms", C.c_double), ("t_pcg_ms", C.c_double)]


class ipm_trace_rec(C.Structure):
    _fields_ = [("it", C.c_int32), ("pcg_iters", C.c_int32), ("mu", C.c_double), ("kkt_inf", C.c_double),
                ("alpha_x", C.c_double), ("alpha_lam", C.c_double), ("pcg_relres", C.c_double),
                ("obj", C.c_double)]


class ipm_info(C.Structure):
    _fields_ = [("gemv_kernel", C.c_int32), ("ncb", C.c_int32), ("group_lanes", C.c_int32),
                ("sharded", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("row_begin", C.c_int64), ("row_end", C.c_int64)]


# include/sqp.h
class ipm_dose_nlp(C.Structure):
    _fields_ = [("nd", C.c_int64), ("nnz", C.c_int64), ("D_rowptr", C.c_void_p), ("D_col", C.c_void_p),
                ("D_val", C.c_void_p), ("w", C.c_void_p), ("p", C.c_void_p), ("dmax", C.c_void_p),
                ("kappa", C.c_void_p), ("beta", C.c_double)]


class ipm_sqp_options(C.Structure):
    _fields_ = [("size", C.c_int32), ("max_iter", C.c_int32), ("tol_d", C.c_double), ("armijo_c1", C.c_double),
                ("max_backtrack", C.c_int32), ("powell", C.c_double), ("warm_start", C.c_int32),
                ("hess_kind", C.c_int32), ("max_cols", C.c_int32), ("h0_floor", C.c_double)]


class ipm_sqp_stats(C.Structure):
    _fields_ = [("status", C.c_int32), ("iters", C.c_int32), ("f", C.c_double), ("d_inf", C.c_double),
                ("ipm_iters_total", C.c_int64), ("pcg_iters_total", C.c_int64), ("updates_skipped", C.c_int32),
                ("backtracks", C.c_int32), ("t_total_ms", C.c_double), ("t_qp_ms", C.c_double)]


class ipm_sqp_trace_rec(C.Structure):
    _fields_ = [("it", C.c_int32), ("ipm_iters", C.c_int32), ("pcg_iters", C.c_int64), ("f", C.c_double),
                ("d_inf", C.c_double), ("step", C.c_double), ("theta", C.c_double), ("qp_ms", C.c_double),
                ("updated", C.c_int32), ("ncols", C.c_int32)]


_P = C.c_void_p
_D = C.c_double
_S = C.c_int32
_sigs = {
    "ipm_abi_version": ([], C.c_int32),
    "ipm_options_default": ([C.POINTER(ipm_options)], None),
    "ipm_nccl_unique_id": ([_P, C.c_size_t], _S),
    "ipm_group_create": ([C.c_int32, C.POINTER(_P)], _S),
    "ipm_group_destroy": ([_P], None),
    "ipm_workspace_size": ([C.POINTER(ipm_problem), C.POINTER(ipm_options), C.POINTER(C.c_size_t)], _S),
    "ipm_create": ([C.POINTER(_P), C.POINTER(ipm_problem), C.POINTER(ipm_options), _P, C.c_size_t, _P], _S),
    "ipm_solve": ([_P], _S),
    "ipm_get_solution": ([_P, _P, _P, _P, _P, _P, C.POINTER(_D)], _S),
    "ipm_get_stats": ([_P, C.POINTER(ipm_stats)], _S),
    "ipm_get_info": ([_P, C.POINTER(ipm_info)], _S),
    "ipm_get_trace": ([_P, C.POINTER(ipm_trace_rec), C.c_int32, C.POINTER(C.c_int32)], _S),
    "ipm_set_linear_term": ([_P, _P], _S),
    "ipm_update_hessian_rank2": ([_P, _P, _D, _P, _D], _S),
    "ipm_warm_start": ([_P], _S),
    "ipm_set_iterate": ([_P, _P, C.POINTER(_P), C.POINTER(_P), _D], _S),
    "ipm_get_iterate": ([_P, _P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_D)], _S),
    "ipm_op_apply": ([_P, _P, _P, _P, _P], _S),
    "ipm_op_diag": ([_P, _P, _P, _P], _S),
    "ipm_pcg": ([_P, _P, _P, _P, _P, _D, C.POINTER(C.c_int32)], _S),
    "ipm_set_bounds": ([_P, _P, _P, _P, _P], _S),
    "ipm_pcg_iterate": ([_P, _P, _P, _P, C.c_int32, _P, _P, _P, _P, C.POINTER(_D)], _S),
    "ipm_profile": ([_P, C.c_int32, C.c_int32, C.POINTER(_D)], _S),
    "ipm_kernel_launches": ([_P], C.c_int64),
    "ipm_kernel_timer": ([_P, C.POINTER(_D), C.POINTER(C.c_int64)], _S),
    "ipm_sym_plan": ([C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int32, C.POINTER(C.c_int32), _P,
                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)], _S),
    "ipm_last_error": ([_P], C.c_char_p),
    "ipm_destroy": ([_P], None),
    "ipm_sqp_options_default": ([C.POINTER(ipm_sqp_options)], None),
    "ipm_sqp_workspace_size": ([C.POINTER(ipm_problem), C.POINTER(ipm_dose_nlp), C.POINTER(ipm_sqp_options),
                                C.POINTER(ipm_options), C.POINTER(C.c_size_t)], _S),
    "ipm_sqp_create": ([C.POINTER(_P), C.POINTER(ipm_problem), C.POINTER(ipm_dose_nlp), C.POINTER(ipm_sqp_options),
                        C.POINTER(ipm_options), _P, C.c_size_t, _P], _S),
    "ipm_sqp_solve": ([_P, _P], _S),
    "ipm_sqp_get_x": ([_P, _P], _S),
    "ipm_sqp_get_stats": ([_P, C.POINTER(ipm_sqp_stats)], _S),
    "ipm_sqp_get_trace": ([_P, C.POINTER(ipm_sqp_trace_rec), C.c_int32, C.POINTER(C.c_int32)], _S),
    "ipm_sqp_eval": ([_P, _P, C.POINTER(_D), _P], _S),
    "ipm_sqp_qp": ([_P], _P),
    "ipm_sqp_kernel_launches": ([_P], C.c_int64),
    "ipm_sqp_last_error": ([_P], C.c_char_p),
    "ipm_sqp_destroy": ([_P], None),
}
EXPORTED = tuple(_sigs)

for _name, (_args, _res) in _sigs.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res
    globals()[_name] = _f


class IpmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ipm status {status} ({STATUS_NAMES.get(status, '?')}): {msg}")
        self.status = status


def check(status: int, ctx=None, allow=(IPM_OK,)) -> int:
    if status not in allow:
        raise IpmError(status, (ipm_last_error(ctx) or b"").decode(errors="replace"))
    return status
