"""ctypes binding of include/oea_cuda.h (liboea_cuda.so, built in-tree).

The library is the only compute path: if it is missing or no sm_100 GPU is
present, calls raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OEA_LIB") or os.path.join(_HERE, "lib", "liboea_cuda.so")

OEA_OK = 0
OEA_ERR_INVALID_ARGUMENT = 1
OEA_ERR_DOMAIN = 2
OEA_ERR_CUDA = 3

DTYPES = {"f64": 0, "f32": 1, "bf16": 2}


class OeaError(RuntimeError):
    """CUDA / internal failure of the oea library."""


class InvalidArgument(ValueError):
    """Reference std::invalid_argument."""


class DomainError(ArithmeticError):
    """Reference std::domain_error."""


class RoutingCfgC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("k", C.c_int32), ("k0", C.c_int32), ("p", C.c_double),
                ("k_max", C.c_int32), ("max_p", C.c_int32), ("cap", C.c_int32)]


class ScoreGenCfgC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_experts", C.c_int32), ("batch", C.c_int32),
                ("steps", C.c_int32), ("layers", C.c_int32), ("seed", C.c_uint64),
                ("alpha", C.c_double), ("groups", C.c_int32),
                ("within_group_concentration", C.c_double), ("between_group_spread", C.c_double)]


class PlanViewC(C.Structure):
    _fields_ = [("set_stride", C.c_int32)] + [
        (name, C.c_void_p) for name in (
            "sets", "set_len", "weights", "weights_f32", "loads", "active_union",
            "active_count", "total_load", "order", "phase1_t", "phase1_n", "base_union",
            "base_union_count")]


_lib = None
_lib_lock = threading.Lock()


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise OeaError(
                    f"{LIB_PATH} is not built (run `python -c 'import __graft_entry__ as g; "
                    "g.build()'` or `make -C paper_2511_02237_b200/csrc`); oea has no CPU path")
            L = C.CDLL(LIB_PATH)
            vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
            L.oea_last_error.restype = C.c_char_p
            L.oea_last_error.argtypes = [vp]
            L.oea_ctx_kernel_launches.restype = i64
            L.oea_ctx_kernel_launches.argtypes = [vp]
            L.oea_plan_set_stride.restype = i32
            sigs = {
                "oea_abi_version": [],
                "oea_ctx_create": [i32, vp],
                "oea_ctx_destroy": [vp],
                "oea_ctx_stream": [vp, vp],
                "oea_ctx_synchronize": [vp],
                "oea_config_resolve": [vp, i32, vp],
                "oea_route_f64_host": [vp, vp, vp, i32, i32, vp, vp],
                "oea_route_f64": [vp, vp, vp, i32, i32, vp, vp, vp],
                "oea_route_f64_batched_host": [vp, vp, vp, vp, i32, i32, vp, vp],
                "oea_gen_scores": [vp, vp, i32, i32, vp, vp],
                "oea_residual_rmsnorm": [vp, vp, vp, vp, i32, i32, C.c_double, vp],
                "oea_moe_decode_ep_partial": [vp, vp, vp, i32, vp, i32, i32, vp, vp, vp],
                "oea_ep_combine": [vp, vp, vp, i32, i32, i32, vp, vp],
                "oea_device_alloc": [vp, C.c_uint64, vp],
                "oea_device_free": [vp, vp],
                "oea_ipc_get_handle": [vp, vp, vp],
                "oea_ipc_open_handle": [vp, vp, vp],
                "oea_ipc_close_handle": [vp, vp],
                "oea_gen_scores_host": [vp, vp, i32, i32, vp],
                "oea_sort_experts_f64_host": [vp, vp, i32, i32, vp],
                "oea_phase1_f64_host": [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp],
                "oea_phase2_f64_host": [vp, vp, i32, i32, vp, vp, vp, i32, vp, vp],
                "oea_layer_create": [vp, i32, i32, i32, i32, vp],
                "oea_layer_create_shard": [vp, i32, i32, i32, i32, i32, i32, vp],
                "oea_layer_destroy": [vp],
                "oea_layer_upload_router": [vp, vp, i32, i32],
                "oea_layer_upload_expert": [vp, i32, vp, vp, vp, i32, i32],
                "oea_layer_init_random": [vp, C.c_uint64],
                "oea_layer_download_router": [vp, vp, i32],
                "oea_layer_download_expert": [vp, i32, vp, vp, vp, i32],
                "oea_layer_info": [vp, vp, vp, vp, vp, vp, vp],
                "oea_moe_decode": [vp, vp, vp, vp, i32, vp, vp, vp],
                "oea_moe_decode_host": [vp, vp, vp, vp, i32, vp, vp],
                "oea_last_plan_host": [vp, vp, vp, vp],
                "oea_decode_graph_create": [vp, vp, vp, vp, i32, vp, vp, vp],
                "oea_graph_launch": [vp, vp],
                "oea_decode_chain_graph_create": [vp, i32, vp, vp, vp, i32, vp, vp, vp],
                "oea_decode_stage_graphs_create": [vp, vp, vp, vp, i32, vp, vp, vp, vp],
                "oea_graph_destroy": [vp],
                "oea_moe_forward_plan_host": [vp, vp, vp, i32, vp, vp, vp, i32, vp, vp],
                "oea_router_scores_host": [vp, vp, vp, i32, vp],
                "oea_ep_owner": [i32, i32, i32],
                "oea_debug_ffn_trace": [vp, vp, i32],
            }
            for name, args in sigs.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = C.c_int
            _lib = L
    return _lib


# Exported symbols of the C ABI (checked by the CPU test-suite against
# include/oea_cuda.h).
EXPORTED = (
    "oea_abi_version", "oea_ctx_create", "oea_ctx_destroy", "oea_last_error", "oea_ctx_stream",
    "oea_ctx_synchronize", "oea_ctx_kernel_launches", "oea_config_resolve",
    "oea_plan_set_stride", "oea_route_f64_host", "oea_route_f64", "oea_route_f64_batched_host",
    "oea_gen_scores", "oea_gen_scores_host", "oea_residual_rmsnorm",
    "oea_moe_decode_ep_partial", "oea_ep_combine", "oea_device_alloc",
    "oea_device_free", "oea_ipc_get_handle", "oea_ipc_open_handle", "oea_ipc_close_handle",
    "oea_sort_experts_f64_host",
    "oea_phase1_f64_host", "oea_phase2_f64_host", "oea_layer_create", "oea_layer_destroy",
    "oea_layer_upload_router", "oea_layer_upload_expert", "oea_layer_init_random",
    "oea_layer_download_router", "oea_layer_download_expert", "oea_layer_info",
    "oea_moe_decode", "oea_moe_decode_host", "oea_last_plan_host", "oea_decode_graph_create",
    "oea_graph_launch", "oea_decode_stage_graphs_create", "oea_graph_destroy", "oea_moe_forward_plan_host",
    "oea_router_scores_host", "oea_ep_owner", "oea_debug_ffn_trace", "oea_layer_create_shard",
    "oea_decode_chain_graph_create")


def check(rc: int, ctx=None):
    if rc == OEA_OK:
        return
    msg = lib().oea_last_error(ctx).decode(errors="replace")
    if rc == OEA_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == OEA_ERR_DOMAIN:
        raise DomainError(msg)
    raise OeaError(msg)


class Context:
    """An oea context: one CUDA stream + workspace on one device."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib().oea_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if getattr(self, "h", None) and self.h:
            lib().oea_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        check(rc, self.h)

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        self.check(lib().oea_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        self.check(lib().oea_ctx_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(lib().oea_ctx_kernel_launches(self.h))


_tls = threading.local()


def default_context() -> Context:
    """One context per host thread (the reference's functions are reentrant,
    simulate.cpp:142-150)."""
    ctx = getattr(_tls, "ctx", None)
    if ctx is None:
        ctx = Context(int(os.environ.get("OEA_DEVICE", "0")))
        _tls.ctx = ctx
    return ctx
