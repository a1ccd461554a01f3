"""ctypes binding of the C ABI declared in include/lipsub_b200.h.

The shared library is built in-tree (paper_2409_03807_b200/_lib/liblipsub_b200.so,
see __graft_entry__.build()).  There is no CPU fallback: if the library or a
CUDA device is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "liblipsub_b200.so")

LSB_OK, LSB_EINVAL, LSB_ENONFINITE, LSB_ECUDA, LSB_EMESH, LSB_ESTATE = range(6)
LSB_FP64, LSB_FP32 = 0, 1


class lsb_mesh_desc(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_int),
        ("rest_positions", C.POINTER(C.c_double)),
        ("num_tets", C.c_int),
        ("tets", C.POINTER(C.c_int32)),
        ("num_pinned", C.c_int),
        ("pinned", C.POINTER(C.c_int32)),
        ("mu", C.POINTER(C.c_double)),
        ("lam", C.POINTER(C.c_double)),
        ("density", C.c_double),
    ]


class lsb_decoder_desc(C.Structure):
    _fields_ = [
        ("latent_dim", C.c_int),
        ("num_layers", C.c_int),
        ("rows", C.POINTER(C.c_int)),
        ("cols", C.POINTER(C.c_int)),
        ("activations", C.POINTER(C.c_int)),
        ("weights", C.POINTER(C.POINTER(C.c_double))),
        ("biases", C.POINTER(C.POINTER(C.c_double))),
        ("norm_shift", C.POINTER(C.c_double)),
        ("norm_scale", C.POINTER(C.c_double)),
    ]


class lsb_solver_config(C.Structure):
    _fields_ = [
        ("epsilon", C.c_double),
        ("max_iters", C.c_int),
        ("max_linesearch", C.c_int),
        ("lbfgs_history", C.c_int),
        ("dt", C.c_double),
    ]


class lsb_exit_report(C.Structure):
    _fields_ = [
        ("code", C.c_int),
        ("iterations", C.c_int),
        ("final_grad_inf_norm", C.c_double),
        ("wall_time_ms", C.c_double),
        ("value_evals", C.c_int),
        ("grad_evals", C.c_int),
    ]


# (name, restype, argtypes) for every symbol the header declares.
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)
_CTX = C.c_void_p
SIGNATURES = [
    ("lsb_last_error", C.c_char_p, []),
    ("lsb_version", C.c_char_p, []),
    ("lsb_bar_mesh_size", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("lsb_make_bar_mesh", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_uint64, C.c_int, _D, _I, _I]),
    ("lsb_make_bar_decoder", C.c_int, [C.c_int, _D, C.c_int, _I, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                       C.c_double, _D, _D, _D]),
    ("lsb_lame_from_young", C.c_int, [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64, _D, _D]),
    ("lsb_gaussian_stream", C.c_int, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, _D]),
    ("lsb_create", C.c_int, [C.POINTER(lsb_mesh_desc), C.POINTER(lsb_decoder_desc), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    ("lsb_destroy", None, [_CTX]),
    ("lsb_get_info", C.c_int, [_CTX] + [C.POINTER(C.c_int)] * 6),
    ("lsb_get_mass", C.c_int, [_CTX, _D, _D]),
    ("lsb_set_pin_positions", C.c_int, [_CTX, _D]),
    ("lsb_set_inertia", C.c_int, [_CTX, _D, C.c_double]),
    ("lsb_eval", C.c_int, [_CTX, _D, _D, _D]),
    ("lsb_decode", C.c_int, [_CTX, _D, _D]),
    ("lsb_lbfgs", C.c_int, [_CTX, _D, C.POINTER(lsb_solver_config), C.POINTER(lsb_exit_report)]),
    ("lsb_set_state", C.c_int, [_CTX, _D, _D, _D]),
    ("lsb_get_state", C.c_int, [_CTX, _D, _D, _D, _D]),
    ("lsb_set_external_force", C.c_int, [_CTX, _D]),
    ("lsb_step", C.c_int, [_CTX, C.POINTER(lsb_solver_config), C.c_int, C.POINTER(lsb_exit_report)]),
    ("lsb_simulate", C.c_int, [_CTX, C.c_int, C.POINTER(lsb_solver_config), C.c_int, C.POINTER(lsb_exit_report), _D]),
    ("lsb_eval_batched", C.c_int, [_CTX, C.c_int, _D, _D, _D]),
    ("lsb_assemble", C.c_int, [_CTX, _D, _D, _D]),
    ("lsb_element_snh", C.c_int, [_CTX, C.c_int, C.POINTER(C.c_int), _D, _D, _D, _D]),
    ("lsb_elastic_hessian_apply", C.c_int, [_CTX, _D, C.c_int, _D, _D]),
    ("lsb_decode_jacobian", C.c_int, [_CTX, _D, _D]),
    ("lsb_decode_second_directional", C.c_int, [_CTX, _D, _D, _D, _D]),
    ("lsb_hessian_batched", C.c_int, [_CTX, C.c_int, _D, _D]),
    ("lsb_objective_hessian", C.c_int, [_CTX, C.c_int, _D, _D]),
    ("lsb_set_cubature", C.c_int, [_CTX, C.c_int, C.POINTER(C.c_int), _D]),
    ("lsb_projective_newton", C.c_int, [_CTX, _D, C.POINTER(lsb_solver_config), C.POINTER(lsb_exit_report)]),
    ("lsb_lipschitz_loss", C.c_int, [_CTX, C.c_int, _D, _D, _D]),
    ("lsb_lipschitz_loss_grad", C.c_int, [_CTX, C.c_int, _D, _D, _D, _D]),
    ("lsb_bench_evals", C.c_int, [_CTX, C.c_int, _D, C.c_size_t, _D, _D, _D]),
    ("lsb_bench_e2e", C.c_int, [_CTX, C.c_int, _D, _D, _D, _D]),
    ("lsb_bench_evals_ex", C.c_int, [_CTX, C.c_int, _D, C.c_size_t, C.c_int, _D, _D, _D]),
    ("lsb_bench_batched", C.c_int, [_CTX, C.c_int, C.c_int, _D, _D, C.c_int, C.c_size_t, _D, _D, _D, _D]),
    ("lsb_bench_steps", C.c_int, [_CTX, C.c_int, C.POINTER(lsb_solver_config), C.c_int, C.c_size_t, _D,
                                  C.POINTER(lsb_exit_report)]),
    ("lsb_get_solve_info", C.c_int, [_CTX, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("lsb_set_solve_kernel", C.c_int, [_CTX, C.c_int]),
    ("lsb_get_trace", C.c_int, [_CTX, C.POINTER(C.c_ulonglong), C.c_int, C.POINTER(C.c_int)]),
    ("lsb_get_trace_raw", C.c_int, [_CTX, C.POINTER(C.c_ulonglong)]),
    ("lsb_get_sweep_trace", C.c_int, [_CTX, C.POINTER(C.c_ulonglong), C.c_int, C.POINTER(C.c_int)]),
    ("lsb_get_launch_count", C.c_int, [_CTX, C.POINTER(C.c_longlong)]),
    ("lsb_get_dev_flags", C.c_int, [_CTX, C.c_char_p, C.c_int]),
    ("lsb_profile_eval", C.c_int, [_CTX, _D, C.c_int, _D, _D, _D, _D]),
]

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load (once) the in-tree CUDA library; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise LibraryMissing(
                f"{_LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
        L = C.CDLL(_LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class LsbError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def check(status):
    if status != LSB_OK:
        msg = lib().lsb_last_error().decode()
        if status == LSB_EINVAL:
            raise ValueError(msg)  # reference std::invalid_argument
        raise LsbError(status, msg)  # reference std::runtime_error family


def dptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous, "expected C-contiguous float64"
    return a.ctypes.data_as(_D)


def iptr(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous, "expected C-contiguous int32"
    return a.ctypes.data_as(_I)
