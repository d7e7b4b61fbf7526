"""ctypes loader for librepops.so and the symbol table of include/repops.h.

Argument marshalling only.  If the library is missing the import fails loudly
(there is no CPU fallback and no other backend).
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librepops.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "repops.h")

i64, i32, f32, vp, u8p = C.c_int64, C.c_int, C.c_float, C.c_void_p, C.c_void_p


class TensorDesc(C.Structure):
    """verde_tensor_desc (repops.h)"""
    _fields_ = [("data", C.c_void_p), ("nbytes", C.c_int64), ("dtype", C.c_int32), ("rank", C.c_int32),
                ("dims", C.c_int64 * 8), ("digest", C.c_void_p), ("mode", C.c_int32), ("reserved", C.c_int32),
                ("leaves_out", C.c_void_p), ("base_leaves", C.c_void_p), ("dirty", C.c_void_p)]


class Node(C.Structure):
    """verde_node (repops.h)"""
    _fields_ = [("index", C.c_uint32), ("op", C.c_uint16), ("shard", C.c_uint32),
                ("n_attr", C.c_int32), ("attr_keys", C.c_void_p), ("attr_vals", C.c_void_p),
                ("n_in", C.c_int32), ("in_src_node", C.c_void_p), ("in_src_slot", C.c_void_p),
                ("in_digests", C.c_void_p), ("n_dst", C.c_int32), ("dst_nodes", C.c_void_p),
                ("n_out", C.c_int32), ("out_digests", C.c_void_p)]


SIGNATURES = {
    "repops_abi_version": (i32, []),
    "repops_last_error": (C.c_char_p, []),
    "repops_launch_count": (i64, []),
    "repops_gemm": (i32, [i64, i64, i64, vp, i64, i32, vp, i64, i32, i32, vp, f32, vp, i64, vp]),
    "repops_gemm_strided_batched_causal": (i32, [i64, i64, i64, vp, i64, i32, i64, i64, vp, i64, i32, i64, i64,
                                                 i32, vp, f32, vp, i64, i64, i64, i64, i64, i32, vp, i64, i64, i64,
                                                 vp]),
    "repops_causal_suffix_flags": (i32, [vp, i64, i64, i64, i64, i64, i64, i64, vp, i64, i64, i64, vp]),
    "repops_gemm_strided_batched": (i32, [i64, i64, i64, vp, i64, i32, i64, i64, vp, i64, i32, i64, i64,
                                          i32, vp, f32, vp, i64, i64, i64, i64, i64, vp]),
    "repops_gemm_cfg": (i32, [i64, i64, i64, vp, i64, i32, vp, i64, i32, i32, vp, f32, vp, i64, vp, i32]),
    "repops_sum_rows": (i32, [vp, i64, i64, i64, vp, vp]),
    "repops_sum_cols_seq": (i32, [vp, i64, i64, i64, i64, vp, i64, vp]),
    "repops_tree_sum": (i32, [vp, i32, i64, vp, vp]),
    "repops_softmax": (i32, [vp, i64, i64, i64, i32, vp, i64, vp]),
    "repops_softmax_backward": (i32, [vp, i64, vp, i64, i64, i64, f32, vp, i64, vp]),
    "repops_layernorm": (i32, [vp, vp, vp, i64, i64, f32, vp, vp, vp, vp]),
    "repops_layernorm_backward": (i32, [vp, vp, vp, vp, vp, vp, i64, i64, vp, vp]),
    "repops_layernorm_backward_params": (i32, [vp, vp, vp, vp, i64, i64, i64, vp, vp, i64, vp]),
    "repops_cross_entropy": (i32, [vp, i64, i64, i64, vp, f32, vp, vp, i64, vp]),
    "repops_exp": (i32, [vp, i64, vp, vp]),
    "repops_log": (i32, [vp, i64, vp, vp]),
    "repops_tanh": (i32, [vp, i64, vp, vp]),
    "repops_rsqrt": (i32, [vp, i64, vp, vp]),
    "repops_gelu": (i32, [vp, i64, vp, vp]),
    "repops_relu": (i32, [vp, i64, vp, vp]),
    "repops_adamw_segments": (i32, [vp, vp, vp, vp, i32, vp, vp, i64, f32, f32, f32, f32, f32, vp]),
    "repops_sin": (i32, [vp, i64, vp, vp]),
    "repops_cos": (i32, [vp, i64, vp, vp]),
    "repops_erf": (i32, [vp, i64, vp, vp]),
    "repops_attention_fwd_supported": (i32, [i64, i64]),
    "repops_attention_probs_supported": (i32, [i64, i64]),
    "repops_attention_probs": (i32, [i64, i64, vp, i64, i64, i64, vp, i64, i64, i64, f32, i32, vp, i64, i64, i64,
                                     i64, vp]),
    "repops_attention_dscores": (i32, [i64, i64, vp, i64, i64, i64, vp, i64, i64, i64, vp, i64, i64, f32, vp, i64,
                                       i64, i64, i64, vp]),
    "repops_attention_fwd": (i32, [i64, i64, vp, vp, vp, i64, i64, i64, f32, i32, vp, vp, i64, i64, vp, i64, i64, i64,
                                   i64, i64, vp]),
    "repops_convert": (i32, [vp, i32, i64, i64, i64, vp, i32, i64, vp]),
    "repops_gemm_ex_workspace_bytes": (i64, [i64, i64, i64, i32, i32, i32]),
    "repops_gemm_ex": (i32, [i64, i64, i64, vp, i32, i64, i32, vp, i32, i64, i32, i32, vp, f32, vp, i32, i64, vp, i64,
                             vp]),
    "repops_rand_uniform": (i32, [C.c_uint64, C.c_uint64, i64, vp, vp]),
    "repops_dropout": (i32, [vp, i64, f32, C.c_uint64, C.c_uint64, vp, vp, vp]),
    "repops_dropout_backward": (i32, [vp, i64, f32, C.c_uint64, C.c_uint64, vp, vp]),
    "repops_ipc_alloc": (i32, [i64, vp, vp]),
    "repops_ipc_open": (i32, [vp, vp]),
    "repops_ipc_close": (i32, [vp]),
    "repops_ipc_free": (i32, [vp]),
    "repops_p2p_tree_combine": (i32, [vp, i32, i64, i64, vp, vp, vp]),
    "repops_p2p_signal": (i32, [vp, i32, i32, C.c_uint32, vp]),
    "repops_p2p_wait": (i32, [vp, i32, C.c_uint32, i64, vp, vp]),
    "repops_gelu_erf": (i32, [vp, i64, vp, vp]),
    "repops_gelu_erf_backward": (i32, [vp, vp, i64, vp, vp]),
    "repops_rope_tables": (i32, [vp, i64, i64, vp, vp, vp]),
    "repops_relu_backward": (i32, [vp, vp, i64, vp, vp]),
    "repops_gelu_backward": (i32, [vp, vp, i64, vp, vp]),
    "repops_add": (i32, [vp, vp, i64, vp, vp]),
    "repops_embedding": (i32, [vp, i64, i64, vp, vp, i64, vp, vp]),
    "repops_embedding_backward": (i32, [vp, i64, i64, vp, i64, vp, vp, vp]),
    "repops_adamw": (i32, [vp, vp, vp, vp, i64, i64, f32, f32, f32, f32, f32, i32, vp]),
    "repops_flip_bit": (i32, [vp, i64, i32, vp]),
    "repops_transpose": (i32, [vp, i64, i64, i64, vp, i64, vp]),
    "repops_copy2d_batched": (i32, [vp, i64, i64, i64, i64, vp, i64, i64, i64, vp]),
    "repops_gemm_post": (i32, [i64, i64, i64, vp, i64, i32, vp, i64, i32, i32, vp, f32, vp, i64, i32, vp, i64, vp,
                               i64, vp]),
    "repops_rmsnorm": (i32, [vp, vp, i64, i64, f32, vp, vp, vp]),
    "repops_copy2d": (i32, [vp, i64, i64, i64, vp, i64, vp]),
    "repops_swiglu": (i32, [vp, vp, i64, vp, vp]),
    "repops_rope": (i32, [vp, i64, i64, i64, i64, vp, vp, vp, i64, vp]),
    "repops_gather_rows": (i32, [vp, vp, i64, i64, vp, vp]),
    "repops_fill_uniform": (i32, [vp, i64, C.c_uint64, C.c_double, vp]),
    "verde_commit_workspace_bytes": (i64, [vp, i32]),
    "verde_dirty_chunks": (i32, [vp, i64, i64, i64, i32, vp, vp]),
    "verde_sha256_probe": (i32, [i64, i64, vp, vp]),
    "repops_ffma2_probe": (i32, [i64, i64, vp, vp]),
    "verde_commit_tensors": (i32, [vp, i32, vp, i64, vp]),
    "verde_commit_tensor": (i32, [vp, i64, i32, i32, vp, vp, vp, i64, vp]),
    "verde_commit_plan_create": (i32, [vp, i32, vp, i64, vp]),
    "verde_commit_plan_run": (i32, [vp, vp]),
    "verde_commit_plan_destroy": (None, [vp]),
    "verde_merkle_root": (i32, [vp, i64, vp]),
    "verde_digest_from_subroots": (i32, [vp, i64, i32, i32, vp, i64, vp]),
    "verde_sha256": (i32, [vp, i64, vp]),
    "verde_node_digest": (i32, [vp, vp]),
    "verde_node_digests": (i32, [i64, vp, vp, vp, vp, vp, i64, vp, vp]),
    "verde_first_divergence": (i32, [vp, vp, i64, vp, vp]),
    "verde_first_divergence_hashed": (i32, [vp, vp, i64, vp, vp]),
    "verde_merkle_root_hashed": (i32, [vp, i64, vp]),
    "verde_merkle_audit_path": (i32, [vp, i64, i64, i32, vp, vp]),
    "verde_merkle_verify_path": (i32, [vp, i64, i64, vp, i32, vp, vp]),
    "verde_tensor_digest_from_root": (i32, [vp, i32, i32, vp, i64, vp]),
    "verde_chunk_leaves": (i32, [vp, i64, vp, vp]),
    "verde_root_plan_workspace_bytes": (i64, [i64]),
    "verde_root_plan_create": (i32, [i64, vp, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
    "verde_root_plan_run": (i32, [vp, vp]),
    "verde_root_plan_destroy": (None, [vp]),
}

_lib = None


class RepopsError(RuntimeError):
    pass


def header_symbols() -> list[str]:
    """Every function declared in include/repops.h."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*((?:repops|verde)_[a-z_0-9]+)\s*\(",
                                 txt, flags=re.M)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RepopsError(f"librepops.so not built ({LIB_PATH}); run __graft_entry__.build() "
                              "-- there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _hooks(L)
        if L.repops_abi_version() != 1:
            raise RepopsError("librepops.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        msg = lib().repops_last_error().decode(errors="replace")
        raise RepopsError(f"{what} failed (status {status}): {msg}")


# tuning / test hooks exported by the library but not part of include/repops.h
def _hooks(L):
    L.repops_gemm_force_cfg.restype = i32
    L.repops_gemm_num_cfgs.restype = i32
    L.repops_gemm_num_cfgs.argtypes = []
    L.repops_gemm_force_cfg.argtypes = [i32]
    L.repops_gemm_smem_floor.restype = i32
    L.repops_gemm_smem_floor.argtypes = [i32]
    L.repops_commit_ctas_per_sm.restype = i32
    L.repops_commit_ctas_per_sm.argtypes = [i32]
