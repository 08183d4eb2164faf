"""ctypes binding of the C-ABI declared in include/tlora.h.

This is the Python view of the drop-in boundary: the same entry points a cgo / JNI /
N-API stub would bind.  There is no CPU fallback: if the shared
library is missing, loading fails loudly; if there is no sm_100 device, every compute
entry point returns TLORA_ERR_NO_DEVICE and this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("TLORA_LIB", _PKG_DIR / "libtlora.so"))

OK, ERR_ARG, ERR_SHAPE, ERR_REGISTRY, ERR_PLAN, ERR_CUDA, ERR_NO_DEVICE, ERR_NCCL = range(8)
GROUP_WORLD, GROUP_TP, GROUP_DP = range(3)
UNIQUE_ID_BYTES = 128
F64, F32, BF16 = 0, 1, 2
HOST, DEVICE = 0, 1
L_SHRINK, L_FWD, L_DH, L_DX, L_DB, L_DA, L_SHRINK2, L_DH2 = range(8)
LAUNCH_NAMES = ("shrink", "fwd", "dH", "dX", "dB", "dA")


class TileC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("m0", "n0", "kb0", "ke0", "kb1", "ke1", "split", "pad")]


class PlanInfoC(C.Structure):
    _fields_ = [
        ("tokens", C.c_int64),
        ("d", C.c_int64),
        ("k", C.c_int64),
        ("num_slots", C.c_int32),
        ("rank_pad_total", C.c_int32),
        ("num_tiles", C.c_int32 * 8),
        ("splits_db", C.c_int32),
        ("splits_da", C.c_int32),
        ("useful_ext_cols", C.c_int64),
        ("packed_ext_cols", C.c_int64),
    ]


class StepDescC(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("num_layers", C.c_int32), ("num_projections", C.c_int32),
        ("proj_d", C.POINTER(C.c_int64)), ("proj_k", C.POINTER(C.c_int64)),
        ("proj_input", C.POINTER(C.c_int32)), ("num_slots", C.c_int32),
        ("ranks", C.POINTER(C.c_int32)), ("batch", C.POINTER(C.c_int32)),
        ("seq_len", C.POINTER(C.c_int32)), ("y_dtype", C.c_int32), ("flags", C.c_int32),
        ("dh_ring", C.c_int32), ("input_sets", C.c_int32), ("nano_init", C.c_int32),
        ("nano_fixed", C.c_int32), ("aimd_alpha", C.c_int32), ("aimd_beta", C.c_double),
        ("aimd_tau_rel", C.c_double),
    ]


class StepStatsC(C.Structure):
    _fields_ = [("nano_used", C.c_int32), ("next_nano", C.c_int32), ("ms", C.c_double),
                ("replayed_graph", C.c_int32), ("launches", C.c_longlong), ("tokens", C.c_int64)]


class StepOpC(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("kind", "stream", "key", "nano", "slot", "sec_kind",
                                         "sec_key", "sec_nano", "sec_slot", "beta", "wait0",
                                         "wait1")]


STEP_SIDE_GRADS, STEP_GRAPH, STEP_EARLY_GRADS, STEP_SHARDED_OPT = 1, 2, 4, 8
RUN_EAGER, RUN_TRACE = 1, 2
BUF_X, BUF_DY, BUF_Y, BUF_DX, BUF_H = range(5)
OP_SHRINK, OP_FWD, OP_DH, OP_DX, OP_GRADS, OP_ALLREDUCE, OP_ADAMW, OP_REDUCE_SCATTER, OP_ALLGATHER = range(9)
STREAM_MAIN, STREAM_SIDE, STREAM_COMM = range(3)

# exported symbol -> (restype, argtypes); also the list the CPU test checks against the header
SIGNATURES = {
    "tlora_last_error": (C.c_char_p, []),
    "tlora_abi_version": (C.c_int, []),
    "tlora_device_check": (C.c_int, [C.c_int, C.POINTER(C.c_int)]),
    "tlora_buffer_alloc": (C.c_int, [C.c_int, C.c_size_t, C.POINTER(C.c_void_p)]),
    "tlora_buffer_free": (C.c_int, [C.c_int, C.c_void_p]),
    "tlora_copy_to_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                       C.c_void_p]),
    "tlora_copy_to_host": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int64,
                                     C.c_void_p]),
    "tlora_stream_sync": (C.c_int, [C.c_void_p]),
    "tlora_copy_async": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "tlora_stream_write_u32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "tlora_stream_wait_u32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "tlora_layer_create": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int32,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_void_p)]),
    "tlora_layer_destroy": (C.c_int, [C.c_void_p]),
    "tlora_layer_set_base": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "tlora_layer_set_adapter": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_int, C.c_void_p]),
    "tlora_layer_layout": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "tlora_layer_zero_grad": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tlora_layer_grad_ptrs": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "tlora_layer_read_grad": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int,
                                        C.c_void_p]),
    "tlora_layer_set_optimizer": (C.c_int, [C.c_void_p, C.POINTER(C.c_float),
                                            C.POINTER(C.c_float), C.c_float, C.c_float,
                                            C.c_float]),
    "tlora_layer_optimizer_step": (C.c_int, [C.c_void_p, C.c_float, C.c_void_p]),
    "tlora_layer_optimizer_step_masked": (C.c_int, [C.c_void_p, C.c_void_p, C.c_float,
                                                    C.c_void_p]),
    "tlora_plan_present_mask": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "tlora_layer_optimizer_step_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_float, C.c_int64,
                                                  C.c_int64, C.c_void_p]),
    "tlora_layer_dp_shard": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int64)]),
    "tlora_layer_reduce_scatter_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "tlora_layer_allgather_operands": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "tlora_layer_read_adapter": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int,
                                           C.c_void_p]),
    "tlora_plan_create": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_void_p)]),
    "tlora_plan_create_gathered": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_void_p)]),
    "tlora_plan_row_map": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "tlora_gather_rows": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_void_p]),
    "tlora_plan_grad_schedule_host": (C.c_int, [C.c_int64, C.c_int64, C.c_int32,
                                                C.POINTER(C.c_int32), C.c_int64,
                                                C.POINTER(C.c_int32), C.c_int32,
                                                C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                                C.c_int32, C.POINTER(C.c_int32)]),
    "tlora_plan_destroy": (C.c_int, [C.c_void_p]),
    "tlora_plan_get_info": (C.c_int, [C.c_void_p, C.POINTER(PlanInfoC)]),
    "tlora_plan_get_tiles": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(TileC), C.c_int32,
                                       C.POINTER(C.c_int32)]),
    "tlora_plan_tiles_host": (C.c_int, [C.c_int64, C.c_int64, C.c_int32, C.POINTER(C.c_int32),
                                        C.c_int64, C.POINTER(C.c_int32), C.c_int,
                                        C.POINTER(TileC), C.c_int32, C.POINTER(C.c_int32)]),
    "tlora_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_void_p, C.c_void_p]),
    "tlora_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_float, C.c_void_p]),
    "tlora_forward_shrink": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_void_p]),
    "tlora_forward_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_int, C.c_void_p]),
    "tlora_forward_gemm_shrink": (C.c_int, [C.c_void_p] * 5 + [C.c_int] + [C.c_void_p] * 4
                                  + [C.c_int, C.c_void_p]),
    "tlora_forward_gemm_dh": (C.c_int, [C.c_void_p] * 5 + [C.c_int] + [C.c_void_p] * 4
                              + [C.c_int, C.c_void_p]),
    "tlora_forward_gemm_rs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_int64,
                                        C.c_int64, C.c_void_p]),
    "tlora_reduce_slots": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_void_p, C.c_void_p]),
    "tlora_backward_dh": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "tlora_backward_dx": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_float, C.c_void_p]),
    "tlora_backward_dx_dh": (C.c_int, [C.c_void_p] * 5 + [C.c_float] + [C.c_void_p] * 4
                             + [C.c_int, C.c_void_p]),
    "tlora_plan_read_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int32,
                                         C.POINTER(C.c_int32), C.c_void_p]),
    "tlora_segments": (C.c_int, [C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "tlora_comm_get_unique_id": (C.c_int, [C.c_void_p]),
    "tlora_comm_create": (C.c_int, [C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_void_p)]),
    "tlora_comm_destroy": (C.c_int, [C.c_void_p]),
    "tlora_comm_info": (C.c_int, [C.c_void_p] + [C.POINTER(C.c_int32)] * 4),
    "tlora_comm_all_gather": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t,
                                        C.c_int, C.c_void_p]),
    "tlora_comm_reduce_scatter": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_size_t, C.c_int, C.c_void_p]),
    "tlora_comm_all_reduce": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t,
                                        C.c_int, C.c_int, C.c_void_p]),
    "tlora_layer_allreduce_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                              C.c_void_p]),
    "tlora_backward_grads": (C.c_int, [C.c_void_p] * 6 + [C.c_float, C.c_void_p]),
    "tlora_backward_grad_b": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_float, C.c_void_p]),
    "tlora_backward_grad_a": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_float, C.c_void_p]),
    "tlora_set_sm_budget": (C.c_int, [C.c_int, C.c_int32, C.c_int32]),
    "tlora_set_tile_scheduler": (C.c_int, [C.c_int, C.c_int]),
    "tlora_profile_begin": (C.c_int, []),
    "tlora_launch_count": (C.c_longlong, []),
    "tlora_profile_end": (C.c_int, [C.POINTER(C.c_int32), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]),
    "tlora_op_cost": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.c_int,
                                C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_longlong)]),
    "tlora_partition": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]),
    "tlora_backward_dx_shrink": (C.c_int, [C.c_void_p] * 5 + [C.c_float] + [C.c_void_p] * 4
                                 + [C.c_int, C.c_void_p]),
    "tlora_fill_normal": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_float,
                                    C.c_void_p]),
    "tlora_nano_assign": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.POINTER(C.c_int32), C.c_void_p, C.c_void_p, C.c_void_p]),
    "tlora_step_create": (C.c_int, [C.POINTER(StepDescC), C.c_void_p, C.POINTER(C.c_void_p)]),
    "tlora_step_destroy": (C.c_int, [C.c_void_p]),
    "tlora_step_layer": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "tlora_step_buffer": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64)]),
    "tlora_step_layout": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p,
                                    C.c_void_p, C.c_void_p]),
    "tlora_step_next_n": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "tlora_step_set_controller": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                            C.c_double, C.c_double]),
    "tlora_step_run": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                 C.POINTER(StepStatsC)]),
    "tlora_step_trace": (C.c_int, [C.c_void_p, C.POINTER(StepOpC), C.POINTER(C.c_double),
                                   C.c_int32, C.POINTER(C.c_int32)]),
    "tlora_step_schedule_host": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.POINTER(StepOpC), C.c_int32, C.POINTER(C.c_int32)]),
    "tlora_tp_create": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tlora_tp_destroy": (C.c_int, [C.c_void_p]),
    "tlora_tp_layer": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "tlora_tp_buffer": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tlora_tp_layout": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p,
                                  C.c_void_p]),
    "tlora_tp_run": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(StepStatsC)]),
    "tlora_tp_trace": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                 C.c_int32, C.POINTER(C.c_int32)]),
    "tlora_aimd_step": (C.c_int, [C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_double,
                                  C.c_double]),
}


class TloraError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tlora status {code}] {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load libtlora.so (built in-tree by `make` / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run `make` (there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(code: int) -> None:
    if code != OK:
        msg = lib().tlora_last_error().decode(errors="replace")
        raise TloraError(code, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
