"""ctypes binding of libharmony_b200.so (declared in include/harmony_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` /
``python -m paper_2202_01306_b200.build``.  There is no fallback: if the
library is missing every entry point raises, so nothing silently runs on the
CPU instead of the native runtime.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import WrapschedError, raise_for_status

LIB_NAME = "libharmony_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)


class hm_entry(C.Structure):
    _fields_ = [("tensor", C.c_int32), ("layer", C.c_int32), ("channel", C.c_int32),
                ("peer_task", C.c_int32), ("src_layer", C.c_int32)]


class hm_task(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "index", "type", "lo", "hi", "dev_kind", "dev_id", "recompute",
        "group_off", "group_len", "in_off", "in_len", "out_off", "out_len")]


class hm_machine(C.Structure):
    _fields_ = [("gpu_count", C.c_int32), ("cpu_offload_update", C.c_int32),
                ("pcie_bandwidth", C.c_int64), ("root_link_bandwidth", C.c_int64),
                ("p2p_bandwidth", C.c_int64), ("update_cpu_rate", C.c_int64),
                ("p2p_group_of", C.POINTER(C.c_int32)), ("dp_sharded_update", C.c_int32)]


class hm_profile(C.Structure):
    _fields_ = [("layers", C.c_int32), ("u_top", C.c_int32)] + [
        (n, C.POINTER(C.c_int64)) for n in ("x", "y", "w", "dw", "k", "t_f", "t_b", "t_u", "w_f")]


ITEM_DTYPE = np.dtype([
    ("task", np.int32), ("stage", np.int32), ("member", np.int32), ("seq", np.int32),
    ("is_compute", np.int32), ("tensor", np.int32), ("channel", np.int32), ("gpu", np.int32),
    ("layer", np.int32), ("peer_task", np.int32), ("peer_member", np.int32), ("n_res", np.int32),
    ("res", np.int32, (4,)), ("nbytes", np.int64), ("duration_ns", np.int64),
    ("start_ns", np.int64), ("end_ns", np.int64)])


class hm_model(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_layer", "d_model", "n_head", "seq_len", "vocab", "vocab_padded", "causal",
        "math_mode")] + [(n, C.c_double) for n in ("lr", "beta1", "beta2", "eps")]


class hm_cnn_layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("type", "cin", "cout", "h", "w", "skip")]


class hm_cnn_model(C.Structure):
    _fields_ = [("n_layer", C.c_int32), ("layers", C.POINTER(hm_cnn_layer)), ("classes", C.c_int32),
                ("classes_padded", C.c_int32)] + [(n, C.c_double) for n in ("lr", "beta1", "beta2", "eps")]


_lib = None


def lib() -> C.CDLL:
    """Load the native library once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise WrapschedError(
            f"{LIB_NAME} is not built (expected at {LIB_PATH}); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    sig = {
        "hm_last_error": (C.c_char_p, []),
        "hm_version": (C.c_char_p, []),
        "hm_plan_build": (C.c_void_p, [P(hm_task), C.c_int32, P(C.c_int32), P(hm_entry),
                                       P(hm_machine), P(hm_profile), P(C.c_int32)]),
        "hm_plan_simulate": (C.c_int, [C.c_void_p, P(C.c_int64)]),
        "hm_plan_item_count": (C.c_int32, [C.c_void_p]),
        "hm_plan_items": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_plan_edge_count": (C.c_int32, [C.c_void_p]),
        "hm_plan_edges": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32), C.c_int32]),
        "hm_plan_free": (None, [C.c_void_p]),
        "hm_pack_layers": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p]),
        "hm_runtime_create": (C.c_void_p, [C.c_int32, P(hm_model), C.c_int64, P(C.c_int32)]),
        "hm_runtime_arena": (C.c_void_p, [C.c_void_p, C.c_int32, P(C.c_int64)]),
        "hm_runtime_layer_offsets": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_int32]),
        "hm_runtime_load_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]),
        "hm_runtime_run_iteration": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                               P(C.c_double)]),
        "hm_runtime_ledger_count": (C.c_int32, [C.c_void_p]),
        "hm_runtime_run_steps": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32,
                                           P(C.c_double), P(C.c_int64)]),
        "hm_runtime_ledger": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_runtime_trace_count": (C.c_int32, [C.c_void_p]),
        "hm_runtime_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_runtime_counters": (C.c_int, [C.c_void_p, P(C.c_int64), C.c_int32]),
        "hm_runtime_create_cnn": (C.c_void_p, [C.c_int32, P(hm_cnn_model), C.c_int64, P(C.c_int32)]),
        "hm_k_relu_bwd": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_void_p]),
        "hm_k_pool2_fwd": (C.c_int, [C.c_void_p] * 2 + [C.c_int32] * 4 + [C.c_void_p]),
        "hm_k_pool2_relu_bwd": (C.c_int, [C.c_void_p] * 3 + [C.c_int32] * 4 + [C.c_void_p]),
        "hm_k_gap_fwd": (C.c_int, [C.c_void_p] * 2 + [C.c_int32] * 3 + [C.c_void_p]),
        "hm_k_gap_bwd": (C.c_int, [C.c_void_p] * 2 + [C.c_int32] * 3 + [C.c_void_p]),
        "hm_k_add_bf16": (C.c_int, [C.c_void_p] * 3 + [C.c_int64, C.c_void_p]),
        "hm_runtime_debug_read": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]),
        "hm_runtime_free": (None, [C.c_void_p]),
        "hm_nccl_unique_id": (C.c_int, [C.c_char_p, C.c_void_p]),
        "hm_runtime_init_comm": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int32, C.c_int32]),
        "hm_runtime_set_graph": (C.c_int, [C.c_void_p, C.c_int32]),
        "hm_runtime_get_step": (C.c_int, [C.c_void_p]),
        "hm_runtime_set_step": (C.c_int, [C.c_void_p, C.c_int32]),
        "hm_runtime_set_w_payload": (C.c_int, [C.c_void_p, C.c_int32]),
        "hm_runtime_share_arenas": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int32, C.c_int64]),
        "hm_runtime_ipc_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_runtime_ipc_import": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_runtime_init_ipc_reduce": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32]),
        "hm_runtime_numa_node": (C.c_int, [C.c_void_p]),
        "hm_runtime_gemm_shapes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
        "hm_k_gemm_replay": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
        "hm_k_gemm_precise": (C.c_int, [C.c_void_p] * 3 + [C.c_int64] * 6 + [C.c_int32] * 3
                              + [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_void_p]),
        "hm_k_attn_fwd_f32": (C.c_int, [C.c_void_p] * 3 + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_k_attn_bwd_f32": (C.c_int, [C.c_void_p] * 6 + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_k_layernorm_fwd_f32": (C.c_int, [C.c_void_p] * 6 + [C.c_int64, C.c_int32, C.c_void_p]),
        "hm_k_cross_entropy_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                                             C.c_void_p, C.c_void_p, C.c_float, C.c_void_p]),
        "hm_runtime_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
        "hm_runtime_kernel_stats": (C.c_int, [C.c_void_p, P(C.c_double), C.c_int32]),
        "hm_runtime_kernel_launches": (C.c_int, [C.c_void_p, P(C.c_double), C.c_int32]),
        "hm_k_adam": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                C.c_double, C.c_double, C.c_double, C.c_int32, C.c_float, C.c_void_p]),
        "hm_k_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                                C.c_int64, C.c_void_p]),
        "hm_k_gemm_tile": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, P(C.c_int32),
                                     P(C.c_int32), P(C.c_int32)]),
        "hm_k_gemm_set_tile": (C.c_int, [C.c_int32, C.c_int32, C.c_int32]),
        "hm_k_conv_fwd": (C.c_int, [C.c_void_p] * 3 + [C.c_int32] * 6 + [C.c_void_p] * 3),
        "hm_k_conv_dgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int32] * 6 + [C.c_void_p] * 2),
        "hm_k_conv_wgrad": (C.c_int, [C.c_void_p] * 3 + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_launch_count": (C.c_int64, []),
        "hm_k_attn_fwd": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_k_attn_fwd_tc": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p] + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_k_attn_bwd": (C.c_int, [C.c_void_p] * 7 + [C.c_int32] * 5 + [C.c_void_p]),
        "hm_k_cast_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
        "hm_k_cast_w_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
        "hm_k_w_split": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
        "hm_k_w_join": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
        "hm_k_embed_fwd": (C.c_int, [C.c_void_p] * 4 + [C.c_int32] * 3 + [C.c_void_p]),
        "hm_k_embed_bwd": (C.c_int, [C.c_void_p] * 4 + [C.c_int32] * 3 + [C.c_void_p]),
        "hm_k_layernorm_fwd": (C.c_int, [C.c_void_p] * 6 + [C.c_int64, C.c_int32, C.c_void_p]),
        "hm_k_layernorm_bwd": (C.c_int, [C.c_void_p] * 10 + [C.c_int64, C.c_int32, C.c_void_p]),
        "hm_k_cross_entropy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32,
                                         C.c_void_p, C.c_void_p, C.c_float, C.c_void_p]),
        "hm_k_bias_grad": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_int64,
                                     C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        try:
            fn = getattr(L, name)
        except AttributeError:
            continue  # reported by tests/test_native_abi.py
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Names the header declares (parsed from include/harmony_b200.h)."""
    import re
    here = os.path.dirname(os.path.abspath(__file__))
    hdr = os.path.join(os.path.dirname(here), "include", "harmony_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", text)))


def last_error() -> str:
    msg = lib().hm_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> int:
    if code < 0:
        raise_for_status(code, last_error())
    return code
