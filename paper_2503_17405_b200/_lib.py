"""ctypes binding of ``libfsmc.so`` (C ABI: ``include/fsmc.h``).

This is the only place the Python host touches native code.  There is no
fallback: if the library is missing or no CUDA device is present, every
compute entry point raises :class:`EngineUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSMC_LIB", os.path.join(HERE, "libfsmc.so"))

ABI_VERSION = 7    # fsmc.h FSMC_ABI_VERSION
WORK_WORDS = 256   # fsmc.h FSMC_WORK_WORDS
FSMC_NINT = 32
MAX_MODES = 8

# families / variants / targets / priors (fsmc.h)
DRMH, ESS, NUTS, SLICE = 1, 2, 3, 4
PLAIN, BUNDLED, AMORTIZED = 0, 1, 2
T_GAUSS_DIAG, T_GAUSS_DENSE, T_GAUSS_EQUICORR, T_MOG, T_FUNNEL, T_NANBAND, T_LOGISTIC, T_FLAT, \
    T_LOGREG, T_BOX, T_GP_HYPER, T_EXTERNAL = range(1, 13)
PRIOR_NONE, PRIOR_IDENTITY, PRIOR_DENSE = 0, 1, 2

# per-chain int slots
I_COUNTER, I_STREAM, I_STATE, I_TICK, I_COUNT = 0, 1, 2, 3, 4
I_ERR_KIND, I_ERR_LABEL, I_ERR_TICK, I_ERR_ITER = 5, 6, 7, 8
I_SHARED, I_BLOCKS, I_PEND, I_FAMILY, I_DRAW0, I_RESUME = 9, 10, 16, 20, 30, 31
SLICE_LABEL = 7   # device label of check_log_density(.., "slice")
E_NONE, E_BLOCK, E_ZERO_START, E_GRAD, E_INIT, E_TARGET = 0, 1, 2, 3, 4, 5

_D = ctypes.c_double
_P = ctypes.c_void_p


class EngineUnavailable(RuntimeError):
    """libfsmc.so could not be loaded or no CUDA device is visible."""


class EngineError(RuntimeError):
    """A C-ABI entry point returned a non-OK status."""


class Kernel(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("max_tries", ctypes.c_int32),
                ("proposal_scale", _D), ("step_size", _D), ("max_depth", ctypes.c_int32),
                ("split_body", ctypes.c_int32), ("divergence_threshold", _D),
                ("slice_width", _D), ("max_expansions", ctypes.c_int32), ("precision", ctypes.c_int32)]


class Target(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32), ("n_modes", ctypes.c_int32),
                ("prior_kind", ctypes.c_int32), ("log_norm", _D), ("a", _D), ("b", _D),
                ("full", ctypes.c_int32), ("scratch", ctypes.c_int32), ("offsets", _D * MAX_MODES), ("mean", _P), ("diag", _P),
                ("diag2", _P), ("mat_t", _P), ("mat2_t", _P), ("yvec", _P), ("prior_t", _P),
                ("data", _P), ("n_rows", ctypes.c_int64)]


class State(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("dim", ctypes.c_int64), ("n_vec", ctypes.c_int32),
                ("n_scal", ctypes.c_int32), ("vec", _P), ("scal", _P), ("ints", _P),
                ("seed", ctypes.c_uint64), ("err_key", _P), ("work", _P)]


class Outputs(ctypes.Structure):
    _fields_ = [("samples", _P), ("loop_counts", _P), ("sample_ticks", _P), ("loop_counts64", _P)]


class Egress(ctypes.Structure):
    _fields_ = [("samples", _P), ("loop_counts", _P), ("iter_counts", _P), ("iter_loop", ctypes.c_int32),
                ("n_loops", ctypes.c_int32)]


_lib = None


def lib():
    """Load libfsmc.so once; raise loudly when the native engine is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailable(
            f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()). "
            "There is no CPU fallback.")
    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device visible; the FSM engine runs only on the GPU")
    L = ctypes.CDLL(LIB_PATH)
    S = ctypes.c_int
    L.fsmc_abi_version.restype = ctypes.c_int32
    L.fsmc_launch_count.restype = ctypes.c_int64
    L.fsmc_last_error.restype = ctypes.c_char_p
    L.fsmc_state_layout.restype = S
    L.fsmc_state_layout.argtypes = [ctypes.POINTER(Kernel), ctypes.c_int64] + \
        [ctypes.POINTER(ctypes.c_int32)] * 4
    L.fsmc_prng_fill.restype = S
    L.fsmc_prng_fill.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int64, ctypes.c_int32, _P, _P]
    L.fsmc_init.restype = S
    L.fsmc_init.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target), ctypes.POINTER(State),
                            ctypes.c_uint64, ctypes.c_int64, _P, _D, _P]
    L.fsmc_run.restype = S
    L.fsmc_run.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target), ctypes.POINTER(State),
                           ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                           ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(Outputs),
                           ctypes.c_int32, _P]
    L.fsmc_run_egress.restype = S
    L.fsmc_run_egress.argtypes = list(L.fsmc_run.argtypes[:-1]) + [ctypes.c_int32,
                                                                   ctypes.POINTER(Egress), _P]
    L.fsmc_dmath_eval.restype = S
    L.fsmc_dmath_eval.argtypes = [ctypes.c_int32, _P, ctypes.c_int64, _P, _P]
    L.fsmc_copy_to_host_2d.restype = S
    L.fsmc_copy_to_host_2d.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P]
    L.fsmc_advance.restype = S
    L.fsmc_advance.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target), ctypes.POINTER(State),
                               ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                               ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(Outputs),
                               _P, _P, _P, _P, _P, ctypes.c_int32, _P]
    L.fsmc_init_deferred.restype = S
    L.fsmc_init_deferred.argtypes = list(L.fsmc_init.argtypes)
    L.fsmc_init_finish.restype = S
    L.fsmc_init_finish.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                   ctypes.POINTER(State), _P, _P]
    L.fsmc_gp_lml.restype = S
    L.fsmc_gp_lml.argtypes = [_P, ctypes.c_int64, _P, _P, ctypes.c_int64, _D, ctypes.c_int32, _P,
                              ctypes.c_int64, _P, _P]
    L.fsmc_gp_lml_grad.restype = S
    L.fsmc_gp_lml_grad.argtypes = [_P, ctypes.c_int64, _P, _P, ctypes.c_int64, _D, ctypes.c_int32, _P,
                                   ctypes.c_int64, _P, _P, _P]
    L.fsmc_gp_last_error.restype = ctypes.c_char_p
    L.fsmc_gp_lml_max_rows.restype = ctypes.c_int64
    L.fsmc_advance_lockstep.restype = S
    L.fsmc_advance_lockstep.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                        ctypes.POINTER(State), ctypes.c_int64,
                                        ctypes.POINTER(Outputs), _P, _P, _P, _P, _P, _P,
                                        ctypes.c_int32, _P]
    L.fsmc_advance_prior.restype = S
    L.fsmc_advance_prior.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                     ctypes.POINTER(State), ctypes.c_int64, ctypes.c_int32,
                                     ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, ctypes.c_int32,
                                     ctypes.POINTER(Outputs), _P, _P, _P, ctypes.c_int32, _P]
    L.fsmc_advance_prior_part.restype = S
    L.fsmc_advance_prior_part.argtypes = list(L.fsmc_advance_prior.argtypes[:-1]) + \
        [ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, _P]
    L.fsmc_prior_apply.restype = S
    L.fsmc_prior_apply.argtypes = [ctypes.POINTER(Target), _P, ctypes.c_int64, _P]
    L.fsmc_prior_trmm.restype = S
    L.fsmc_prior_trmm.argtypes = [ctypes.POINTER(Target), _P, _P, ctypes.c_int64, _P]
    L.fsmc_prior_trmm_last_error.restype = ctypes.c_char_p
    L.fsmc_lockstep_run.restype = S
    L.fsmc_lockstep_run.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                    ctypes.POINTER(State), ctypes.c_int64,
                                    ctypes.POINTER(Outputs), ctypes.c_int32, _P]
    L.fsmc_lockstep_barrier_probe.restype = S
    L.fsmc_lockstep_barrier_probe.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                              ctypes.POINTER(State), ctypes.c_int64, ctypes.c_int32,
                                              _P]
    L.fsmc_run_windowed.restype = S
    L.fsmc_run_windowed.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                    ctypes.POINTER(State), ctypes.c_int64, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, ctypes.c_int32,
                                    ctypes.POINTER(Outputs), ctypes.c_int64, _P, ctypes.c_int32, _P]
    L.fsmc_run_windowed_overlap.restype = S
    L.fsmc_run_windowed_overlap.argtypes = list(L.fsmc_run_windowed.argtypes[:-1]) + [ctypes.c_int32, _P]
    L.fsmc_run_windowed_egress.restype = S
    L.fsmc_run_windowed_egress.argtypes = list(L.fsmc_run_windowed.argtypes[:-1]) + \
        [ctypes.c_int32, ctypes.POINTER(Egress), _P]
    L.fsmc_profile_blocks.restype = S
    L.fsmc_profile_blocks.argtypes = [ctypes.POINTER(Kernel), ctypes.POINTER(Target),
                                      ctypes.POINTER(State), ctypes.c_int64, _P, _P]
    L.fsmc_target_eval.restype = S
    L.fsmc_target_eval.argtypes = [ctypes.POINTER(Target), _P, ctypes.c_int64, _P, _P,
                                   ctypes.c_int32, ctypes.c_int32, _P]
    L.fsmc_logreg_epilogue.restype = S
    L.fsmc_logreg_epilogue.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int64, _P, _P, _P]
    L.fsmc_logreg_tc_eval.restype = S
    L.fsmc_logreg_tc_eval.argtypes = [_P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64,
                                      ctypes.c_int64, _P, _P, _P]
    L.fsmc_logreg_tc_eval2.restype = S
    L.fsmc_logreg_tc_eval2.argtypes = [_P, ctypes.c_int64, _P, _P, _P, _P, ctypes.c_int64,
                                       ctypes.c_int64, _P, _P, ctypes.c_int32, _P]
    L.fsmc_logreg_tc_last_error.restype = ctypes.c_char_p
    L.fsmc_diag_partials.restype = S
    L.fsmc_diag_partials.argtypes = [_P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P]
    if L.fsmc_abi_version() != ABI_VERSION:
        raise EngineUnavailable("libfsmc.so ABI version mismatch")
    _lib = L
    return L


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().fsmc_last_error().decode(errors="replace")
        if status == 1:
            raise ValueError(f"{what}: {msg}")
        raise EngineError(f"{what} failed (status {status}): {msg}")


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()
