"""ctypes binding of libflowrec_b200.so (the C ABI in include/flowrec_b200.h).

The library is the only compute path: there is no CPU fallback.  Importing
this module never touches the GPU; `lib()` raises if the shared object has not
been built, and every call raises `FlowrecError` with the library's message on
a non-zero status.
"""

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FLOWREC_B200_LIB") or os.path.join(HERE, "_lib", "libflowrec_b200.so")

ACT_TANH, ACT_SIN = 0, 1
STEADY2D, UNSTEADY2D, UNSTEADY3D = 0, 1, 2
F32, F64 = 0, 1
MODE_PDE, MODE_MSE, MODE_VALUE, MODE_JET, MODE_GJ = 0, 1, 2, 3, 4
FLAG_NONFINITE_LOSS, FLAG_NONFINITE_GRAD, FLAG_EXCHANGE_TIMEOUT = 1, 2, 4

REGIME_CODES = {"steady2d": STEADY2D, "unsteady2d": UNSTEADY2D, "unsteady3d": UNSTEADY3D}
ACT_CODES = {"tanh": ACT_TANH, "sin": ACT_SIN}


class FlowrecError(RuntimeError):
    pass


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_in", C.c_int), ("n_out", C.c_int), ("n_vel", C.c_int),
        ("hidden_layers", C.c_int), ("width", C.c_int), ("width_pad", C.c_int),
        ("n_params", C.c_int), ("np_pad", C.c_int), ("kp_elems", C.c_int),
        ("dtype", C.c_int), ("act", C.c_int), ("regime", C.c_int), ("num_sms", C.c_int),
        ("inv_re", C.c_double), ("math", C.c_int), ("tc_width", C.c_int),
    ]


class Workspace(C.Structure):
    _fields_ = [
        ("grid", C.c_int), ("threads", C.c_int), ("points_per_tile", C.c_int),
        ("jet_streams", C.c_int),
        ("gpart_elems", C.c_longlong), ("lpart_elems", C.c_longlong),
        ("scratch_bytes", C.c_longlong), ("smem_bytes", C.c_size_t),
        ("loss_rows", C.c_int), ("wide", C.c_int), ("tiles", C.c_longlong),
    ]


class AdamArgs(C.Structure):
    _fields_ = [
        ("n", C.c_longlong),
        ("params", C.c_void_p), ("grad", C.c_void_p), ("m", C.c_void_p), ("v", C.c_void_p),
        ("step", C.c_void_p), ("sched", C.c_void_p), ("row_base", C.c_longlong),
        ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double), ("clip_norm", C.c_double),
        ("norm_parts", C.c_void_p), ("n_norm_parts", C.c_int),
        ("lpart", C.c_void_p), ("seg_rows", C.c_int * 4),
        ("n_obs", C.c_double), ("n_colloc", C.c_double), ("n_ghost_total", C.c_double),
        ("n_ghost_space", C.c_double), ("n_ghost_time", C.c_double),
        ("w_obs", C.c_double), ("w_pde", C.c_double), ("w_ghost_u", C.c_double),
        ("w_ghost_p_space", C.c_double), ("w_ghost_p_time", C.c_double),
        ("history", C.c_void_p), ("flags", C.c_void_p), ("grad_norm", C.c_void_p),
        ("kparams", C.c_void_p), ("sync_counter", C.c_void_p),
    ]


class EpochGate(C.Structure):
    _fields_ = [("gate", C.c_void_p), ("first_gated_set", C.c_int), ("max_ctas", C.c_int),
                ("flags", C.c_void_p), ("timeout_ms", C.c_uint), ("gate_round", C.c_void_p),
                ("gate_mult", C.c_uint)]


class GhostEdge(C.Structure):
    _fields_ = [("y_row", C.c_longlong), ("anchor_row", C.c_longlong), ("n", C.c_longlong),
                ("u", C.c_void_p), ("p", C.c_void_p), ("du", C.c_void_p),
                ("ready", C.c_void_p), ("epochs", C.c_void_p)]


MAX_GHOST_EDGES = 16
IPC_HANDLE_BYTES = 64


class MseSet(C.Structure):
    _fields_ = [("pts", C.c_void_p), ("target_u", C.c_void_p), ("target_p", C.c_void_p),
                ("n", C.c_longlong), ("vel_coef", C.c_double), ("p_coef", C.c_double)]


# name -> (restype, argtypes); every function returns int status unless noted
_P = C.c_void_p
_SIGS = {
    "fr_plan_create": [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.POINTER(_P)],
    "fr_plan_destroy": [_P],
    "fr_plan_get_info": [_P, C.POINTER(PlanInfo)],
    "fr_plan_set_math": [_P, C.c_int],
    "fr_plan_workspace": [_P, C.c_int, C.c_longlong, C.POINTER(Workspace)],
    "fr_prepare_params": [_P, _P, _P, _P],
    "fr_pde_fwd_bwd": [_P, _P, _P, C.c_longlong, C.c_double, _P, _P, _P, _P],
    "fr_mse_fwd_bwd": [_P, _P, _P, _P, _P, C.c_longlong, _P, C.c_double, C.c_double, _P, _P, _P, _P],
    "fr_epoch_workspace": [_P, C.c_longlong, C.POINTER(C.c_longlong), C.c_int, C.POINTER(Workspace)],
    "fr_epoch_fwd_bwd": [_P, _P, _P, C.c_longlong, C.c_double, C.POINTER(MseSet), C.c_int, _P, _P,
                         C.POINTER(C.c_void_p), _P, _P],
    "fr_epoch_workspace_capped": [_P, C.c_longlong, C.POINTER(C.c_longlong), C.c_int, C.c_int,
                                  C.POINTER(Workspace)],
    "fr_epoch_fwd_bwd_gated": [_P, _P, _P, C.c_longlong, C.c_double, C.POINTER(MseSet), C.c_int, _P, _P,
                               C.POINTER(C.c_void_p), _P, C.POINTER(EpochGate), _P],
    "fr_signal": [_P, C.c_uint, C.c_uint, _P],
    "fr_ghost_jet_fwd_bwd": [_P, _P, _P, _P, C.c_longlong, _P, C.c_double, _P, _P, _P, _P],
    "fr_nccl_get_unique_id": [_P],
    "fr_nccl_init": [_P, C.c_int, C.c_int, C.POINTER(_P)],
    "fr_nccl_destroy": [_P],
    "fr_exchange": [_P, C.c_int, C.POINTER(C.c_int), C.POINTER(_P), C.POINTER(C.c_longlong), C.c_int,
                    C.POINTER(C.c_int), C.POINTER(_P), C.POINTER(C.c_longlong), C.c_int, _P],
    "fr_ipc_alloc": [C.c_size_t, C.POINTER(_P), _P],
    "fr_ipc_open": [_P, C.POINTER(_P)],
    "fr_ipc_close": [_P],
    "fr_ipc_free": [_P],
    "fr_ghost_put": [_P, _P, _P, C.c_int, C.POINTER(GhostEdge), _P, C.c_uint, _P, _P],
    "fr_counter_add": [_P, C.c_uint, _P],
    "fr_pcg64_uniform": [C.POINTER(C.c_ulonglong), C.c_ulonglong, C.c_longlong, C.c_int, C.POINTER(C.c_double),
                         C.POINTER(C.c_double), _P, _P, _P],
    "fr_value_fwd": [_P, _P, _P, C.c_longlong, _P, _P],
    "fr_jet_fwd": [_P, _P, _P, C.c_longlong, _P, _P],
    "fr_reduce_grad": [_P, _P, C.c_int, _P, C.c_int, _P, _P],
    "fr_reduce_grad_parts": [_P],
    "fr_reduce_loss": [_P, C.POINTER(C.c_int), C.c_int, _P, _P],
    "fr_adam_step": [_P, C.POINTER(AdamArgs), _P],
    "fr_pack_ghost": [_P, _P, _P, C.c_longlong, _P, _P, _P],
    "fr_jet_act_forward": [C.c_int, _P, _P, _P, _P, _P, C.c_longlong, C.c_int, C.c_int, _P],
    "fr_jet_act_backward": [C.c_int, _P, _P, _P, _P, _P, C.c_longlong, C.c_int, C.c_int, C.c_int, _P],
    "fr_bench_ffma": [C.c_int, C.c_int, C.c_int, _P, _P],
    "fr_debug_tc_gemm_tf32": [_P, _P, _P, C.c_int, C.c_int, C.c_int, _P],
    "fr_debug_tc_raw": [_P, C.c_int, C.c_int, C.c_int, C.c_int, _P],
    "fr_debug_tc_raw2": [_P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _P],
    "fr_debug_tma_kquad": [_P, _P, C.c_int, C.c_int, C.c_int, C.c_int, _P],
}
EXPORTS = tuple(_SIGS) + ("fr_last_error", "fr_version", "fr_kernel_launches")

_lib = None


def lib():
    """Load (once) and return the shared library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FlowrecError(
            f"{LIB_PATH} is not built; run `python -m paper_2602_15883_b200.build` "
            "(there is no CPU fallback)"
        )
    L = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        f = getattr(L, name)
        f.restype = C.c_int
        f.argtypes = args
    L.fr_last_error.restype = C.c_char_p
    L.fr_last_error.argtypes = []
    L.fr_version.restype = C.c_char_p
    L.fr_version.argtypes = []
    L.fr_kernel_launches.restype = C.c_longlong
    L.fr_kernel_launches.argtypes = []
    _lib = L
    return L


# functions that enqueue kernels (counted for the bench's gpu_launches claim)
LAUNCHERS = frozenset({
    "fr_prepare_params", "fr_pde_fwd_bwd", "fr_mse_fwd_bwd", "fr_epoch_fwd_bwd", "fr_epoch_fwd_bwd_gated",
    "fr_signal", "fr_ghost_jet_fwd_bwd", "fr_value_fwd", "fr_jet_fwd",
    "fr_reduce_grad", "fr_reduce_loss", "fr_adam_step", "fr_pack_ghost", "fr_ghost_put", "fr_counter_add",
    "fr_pcg64_uniform",
    "fr_jet_act_forward",
    "fr_jet_act_backward", "fr_bench_ffma", "fr_debug_tc_gemm_tf32", "fr_debug_tma_kquad",
})
launch_count = 0


def call(name, *args):
    """Invoke an exported function and raise FlowrecError on failure."""
    global launch_count
    L = lib()
    if name in LAUNCHERS:
        launch_count += 1
    rc = getattr(L, name)(*args)
    if rc != 0:
        msg = L.fr_last_error().decode(errors="replace")
        raise FlowrecError(f"{name}: {msg}")
    return rc


def kernel_launches():
    """Kernels enqueued by the library so far (for launch accounting)."""
    return int(lib().fr_kernel_launches())


def version():
    return lib().fr_version().decode()


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)
