"""Thin ctypes binding of libnnt.so (include/nnt.h) — argument marshalling only.

Every function has the C name and argument order of the ABI.  Tensor arguments
may be torch tensors (their data_ptr() is passed), plain integers (raw
pointers) or None (NULL).  ``stream`` defaults to torch's current CUDA stream.
Non-OK statuses raise NNTError carrying nnt_last_error().  There is no
fallback: if libnnt.so is missing this module fails to import.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# NNT_LIB: an alternative build of the same ABI (A/B timing of kernel variants in one run)
LIB_PATH = os.environ.get("NNT_LIB") or os.path.join(_PKG, "libnnt.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built; run `python -m paper_2504_13236_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
NNT_OK = 0
NNT_ERR_NULL, NNT_ERR_SHAPE, NNT_ERR_TILE, NNT_ERR_DTYPE, NNT_ERR_ALIGN = 1, 2, 3, 4, 5
NNT_ERR_UNSUPPORTED, NNT_ERR_WORKSPACE, NNT_ERR_CUDA, NNT_ERR_ARG = 6, 7, 8, 9
STATUS_NAMES = {0: "NNT_OK", 1: "NNT_ERR_NULL", 2: "NNT_ERR_SHAPE", 3: "NNT_ERR_TILE", 4: "NNT_ERR_DTYPE",
                5: "NNT_ERR_ALIGN", 6: "NNT_ERR_UNSUPPORTED", 7: "NNT_ERR_WORKSPACE", 8: "NNT_ERR_CUDA",
                9: "NNT_ERR_ARG"}
NNT_F32, NNT_BF16 = 0, 1
NNT_NOTRANS, NNT_TRANS = 0, 1
NNT_CAUSAL_NONE, NNT_CAUSAL_OUT_LOWER, NNT_CAUSAL_A_LOWER, NNT_CAUSAL_A_UPPER = 0, 1, 2, 3
NNT_ACT_NONE, NNT_ACT_GELU, NNT_ACT_GELU_BWD, NNT_ACT_SOFTMAX_BWD, NNT_ACT_ROWSTATS, NNT_ACT_SOFTMAX = 0, 1, 2, 3, 4, 5
NNT_CAUSAL_ALIGN = 128
KERNEL_CLASSES = ("gemm_tc", "gemm_tc_attn", "gemm_simt", "maxsumexp", "softmax", "softmax_bwd", "ln_fwd", "ln_bwd", "gelu",
                  "bias_grad", "adam", "misc")
OP_NAMES = ("ln1", "qkv", "scores", "maxsumexp", "softmax", "pv", "out", "ln2", "fc", "proj",
            "proj_db", "proj_dw", "proj_dx", "fc_db", "fc_dw", "fc_dx", "ln2_bwd", "out_db", "out_dw", "out_dx",
            "att_dp", "att_dv", "softmax_bwd", "att_dq", "att_dk", "qkv_db", "qkv_dw", "qkv_dx", "ln1_bwd")

# The exported symbols include/nnt.h declares (checked by tests/test_abi.py).
EXPORTS = ("nnt_abi_version", "nnt_last_error", "nnt_device_check", "nnt_tile_grid", "nnt_tile_extent",
           "nnt_partition", "nnt_tile_gemm", "nnt_tile_gemm_workspace_bytes", "nnt_maxsumexp",
           "nnt_maxsumexp_merge", "nnt_attn_rowdot", "nnt_softmax", "nnt_softmax_bwd",
           "nnt_layernorm_fwd", "nnt_layernorm_bwd_scratch_bytes", "nnt_layernorm_bwd", "nnt_gelu_fwd",
           "nnt_gelu_bwd", "nnt_bias_grad_scratch_bytes", "nnt_bias_grad", "nnt_adam_step", "nnt_adam_tick", "nnt_sgd_step",
           "nnt_convert",
           "nnt_scale", "nnt_dot_scratch_bytes", "nnt_dot", "nnt_block_workspace_size", "nnt_block_fwd", "nnt_block_bwd", "nnt_block_bwd_streams",
           "nnt_block_tp_workspace_size", "nnt_block_tp_fwd", "nnt_block_tp_bwd",
           "nnt_op_name", "nnt_block_dag_describe", "nnt_timing_enable", "nnt_timing_read", "nnt_timing_trace",
           "nnt_launch_count", "nnt_embedding_fwd", "nnt_embedding_bwd_scratch_bytes", "nnt_embedding_bwd",
           "nnt_cross_entropy", "nnt_attention_fused_supported", "nnt_attention_fwd_pv", "nnt_attention_bwd_kv",
           "nnt_attention_stats", "nnt_attention_stats_enabled",
           "nnt_stf_build", "nnt_attention_trace", "nnt_tp_signal", "nnt_tp_reduce_gather", "nnt_tp_wait")


class NNTError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# ---------------------------------------------------------------- structs
NNT_TP_MAX = 8


class nnt_tp_comm(C.Structure):
    _fields_ = [("R", C.c_int), ("rank", C.c_int), ("rows", C.c_int64), ("cols", C.c_int64),
                ("recv", C.c_void_p * NNT_TP_MAX), ("flags", C.c_void_p * NNT_TP_MAX)]


class nnt_epilogue(C.Structure):
    _fields_ = [("bias", C.c_void_p), ("residual", C.c_void_p), ("ld_residual", C.c_int64), ("act", C.c_int),
                ("aux", C.c_void_p), ("ld_aux", C.c_int64), ("causal", C.c_int), ("workspace", C.c_void_p),
                ("workspace_bytes", C.c_size_t), ("row_stats", C.c_void_p), ("ld_row_stats", C.c_int64),
                ("rowvec", C.c_void_p), ("rowscale", C.c_float), ("a_rowsum", C.c_void_p),
                ("scatter", C.POINTER(nnt_tp_comm))]


class nnt_adam_hparams(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("lr", "beta1", "beta2", "eps", "weight_decay", "bias_corr1",
                                          "bias_corr2", "grad_scale")] + [("bias_corr_dev", C.c_void_p),
                                                                          ("one_minus_beta1", C.c_float),
                                                                          ("one_minus_beta2", C.c_float)]


def adam_hparams(lr, beta1, beta2, eps, weight_decay=0.0, t=None, grad_scale=1.0):
    """nnt_adam_hparams with the caller-side fp64 terms (R12, R23): bias corrections 1 - beta^t
    (1.0 when t is None: the device-side corrections of a captured graph are used) and 1 - beta."""
    bc1, bc2 = (1.0, 1.0) if t is None else (1.0 - beta1 ** t, 1.0 - beta2 ** t)
    hp = nnt_adam_hparams(lr, beta1, beta2, eps, weight_decay, bc1, bc2, grad_scale)
    hp.one_minus_beta1 = 1.0 - beta1
    hp.one_minus_beta2 = 1.0 - beta2
    return hp


class nnt_block_cfg(C.Structure):
    _fields_ = [("E", C.c_int64), ("H", C.c_int64), ("S", C.c_int64), ("B", C.c_int64), ("tile_e", C.c_int64),
                ("tile_f", C.c_int64), ("tile_s", C.c_int64), ("tile_t", C.c_int64), ("dtype", C.c_int),
                ("ln_eps", C.c_float), ("causal", C.c_int)]


class nnt_block_params(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("ln1_g", "ln1_b", "b_qkv", "b_o", "ln2_g", "ln2_b", "b_fc", "b_pr",
                                           "w_qkv", "w_o", "w_fc", "w_pr")]


class nnt_block_grads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_o", "b_o", "ln2_g", "ln2_b",
                                           "w_fc", "b_fc", "w_pr", "b_pr")]


class nnt_block_bwd_links(C.Structure):
    _fields_ = [("dy_bf16", C.c_void_p), ("dy_colsum_done", C.c_int), ("dx_colsum", C.c_void_p),
                ("dx_bf16", C.c_void_p), ("side_done", C.c_void_p), ("wait_before_dx", C.c_void_p)]


class nnt_block_tp(C.Structure):
    _fields_ = [("heads", C.c_int64), ("ffn", C.c_int64), ("add_bias", C.c_int), ("comm", C.POINTER(nnt_tp_comm))]


class nnt_task(C.Structure):
    _fields_ = [("op", C.c_int32), ("level", C.c_int32), ("tile", C.c_int64 * 3), ("n_deps", C.c_int32),
                ("group", C.c_int32)]


class nnt_launch_group(C.Structure):
    _fields_ = [("op", C.c_int32), ("level", C.c_int32), ("n_tasks", C.c_int64), ("side_stream_ok", C.c_int32)]


# ---------------------------------------------------------------- signatures
_i64, _i32, _vp, _f32, _sz = C.c_int64, C.c_int, C.c_void_p, C.c_float, C.c_size_t
_P64 = C.POINTER(C.c_int64)
_sig = {
    "nnt_abi_version": (C.c_int, []),
    "nnt_last_error": (C.c_char_p, []),
    "nnt_device_check": (_i32, [_i32]),
    "nnt_tile_grid": (_i32, [_i32, _P64, _P64, _P64]),
    "nnt_tile_extent": (_i32, [_i64, _i64, _i64, _P64, _P64]),
    "nnt_partition": (_i32, [_i64, _i32, _i32, _P64, _P64]),
    "nnt_tile_gemm": (_i32, [_i32, _i32, _i64, _i64, _i64, _P64, _f32, _vp, _i32, _i64, _P64, _vp, _i32, _i64, _P64,
                             _f32, _vp, _i32, _i64, _P64, _P64, C.POINTER(nnt_epilogue), _vp]),
    "nnt_tile_gemm_workspace_bytes": (_sz, [_i64, _i64, _i64, _i32, _i32, _i32, _i64]),
    "nnt_maxsumexp": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _i64, _vp, _i32, _vp]),
    "nnt_maxsumexp_merge": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _i64, _vp, _vp]),
    "nnt_attn_rowdot": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp]),
    "nnt_attention_fused_supported": (_i32, [_i64, _i64]),
    "nnt_stf_build": (_i32, [_i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64]),
    "nnt_attention_trace": (_i32, [_i32, _vp, _i64]),
    "nnt_attention_fwd_pv": (_i32, [_vp, _i64, _i64, _i64, _i64, C.c_float, _i32, _vp, _vp, _vp, _vp]),
    "nnt_attention_stats": (_i32, [_vp, _i64, _i64, _i64, _i64, C.c_float, _i32, _vp, _vp]),
    "nnt_attention_stats_enabled": (_i32, []),
    "nnt_attention_bwd_kv": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, C.c_float, _i32, _vp, _vp, _vp]),
    "nnt_softmax": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _i64, _vp, _vp, _i32, _i64, _vp]),
    "nnt_softmax_bwd": (_i32, [_vp, _i32, _i64, _vp, _i64, _i64, _i64, _i32, _i64, _f32, _vp, _i32, _i64, _vp]),
    "nnt_layernorm_fwd": (_i32, [_vp, _i64, _i64, _i64, _i64, _vp, _vp, _f32, _vp, _i32, _i64, _vp, _vp, _vp]),
    "nnt_layernorm_bwd_scratch_bytes": (_sz, [_i64, _i64]),
    "nnt_layernorm_bwd": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp,
                                 _vp, _i32, _vp, _sz, _vp]),
    "nnt_gelu_fwd": (_i32, [_vp, _vp, _i32, _i64, _vp]),
    "nnt_gelu_bwd": (_i32, [_vp, _vp, _vp, _i32, _i64, _vp]),
    "nnt_bias_grad_scratch_bytes": (_sz, [_i64, _i64]),
    "nnt_bias_grad": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _i32, _vp, _vp, _sz, _vp]),
    "nnt_adam_step": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, C.POINTER(nnt_adam_hparams), _vp]),
    "nnt_convert": (_i32, [_vp, _i32, _vp, _i32, _i64, _vp]),
    "nnt_sgd_step": (_i32, [_i64, _vp, _vp, _vp, _vp, _f32, _f32, _f32, _vp]),
    "nnt_adam_tick": (_i32, [C.c_double, C.c_double, _vp, _vp, _vp]),
    "nnt_scale": (_i32, [_vp, _f32, _vp, _i64, _vp]),
    "nnt_dot_scratch_bytes": (_sz, [_i64]),
    "nnt_dot": (_i32, [_vp, _vp, _i64, _f32, _vp, _vp, _sz, _vp]),
    "nnt_embedding_fwd": (_i32, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "nnt_embedding_bwd_scratch_bytes": (_sz, [_i64, _i64]),
    "nnt_embedding_bwd": (_i32, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i32, _i32, _vp, _sz, _vp]),
    "nnt_cross_entropy": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _f32, _vp, _vp, _vp, _i64, _vp]),
    "nnt_block_workspace_size": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(_sz), C.POINTER(_sz)]),
    "nnt_block_fwd": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_params), _vp, _vp, _vp, _vp, _vp]),
    "nnt_block_bwd": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_params), _vp, _vp, _vp, _vp, _vp,
                             C.POINTER(nnt_block_grads), _i32, C.POINTER(_vp), _vp]),
    "nnt_block_bwd_streams": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_params), _vp, _vp, _vp, _vp,
                                     _vp, C.POINTER(nnt_block_grads), _i32, C.POINTER(_vp), _vp, _vp,
                                     C.POINTER(nnt_block_bwd_links)]),
    "nnt_block_tp_workspace_size": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_tp), C.POINTER(_sz),
                                           C.POINTER(_sz)]),
    "nnt_block_tp_fwd": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_tp), C.POINTER(nnt_block_params), _i32,
                                _vp, _vp, _vp, _vp, _vp, _vp]),
    "nnt_block_tp_bwd": (_i32, [C.POINTER(nnt_block_cfg), C.POINTER(nnt_block_tp), C.POINTER(nnt_block_params), _i32,
                                _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(nnt_block_grads), _i32, _vp]),
    "nnt_tp_signal": (_i32, [C.POINTER(nnt_tp_comm), C.c_uint32, _i32, _vp]),
    "nnt_tp_reduce_gather": (_i32, [C.POINTER(nnt_tp_comm), C.POINTER(_vp), C.c_uint32, _vp]),
    "nnt_tp_wait": (_i32, [C.POINTER(nnt_tp_comm), C.c_uint32, _vp]),
    "nnt_op_name": (C.c_char_p, [_i32]),
    "nnt_block_dag_describe": (_i32, [C.POINTER(nnt_block_cfg), _i32, C.POINTER(nnt_task), _i64, _P64,
                                      C.POINTER(nnt_launch_group), _i64, _P64]),
    "nnt_timing_enable": (_i32, [_i32]),
    "nnt_timing_read": (_i32, [C.POINTER(C.c_double), _P64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "nnt_timing_trace": (_i32, [C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i64, _P64]),
    "nnt_launch_count": (_i64, []),
}
for _name, (_res, _args) in _sig.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


# ---------------------------------------------------------------- marshalling helpers
def ptr(x):
    """torch tensor / int / None -> void* value."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _arr64(vals):
    if vals is None:
        return None
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])


def check(status):
    if status != NNT_OK:
        raise NNTError(status, lib.nnt_last_error().decode())
    return status


def dtype_code(t):
    import torch
    return {torch.float32: NNT_F32, torch.bfloat16: NNT_BF16}[t.dtype]


# ---------------------------------------------------------------- ABI functions (same names)
def nnt_abi_version():
    return lib.nnt_abi_version()


def nnt_last_error():
    return lib.nnt_last_error().decode()


def nnt_device_check(device=0):
    return check(lib.nnt_device_check(device))


def nnt_tile_grid(shape, tile):
    g = (C.c_int64 * len(shape))()
    check(lib.nnt_tile_grid(len(shape), _arr64(shape), _arr64(tile), g))
    return list(g)


def nnt_tile_extent(dim, tile, idx):
    o, e = C.c_int64(), C.c_int64()
    check(lib.nnt_tile_extent(dim, tile, idx, C.byref(o), C.byref(e)))
    return o.value, e.value


def nnt_partition(n_units, n_ranks, rank):
    b, e = C.c_int64(), C.c_int64()
    check(lib.nnt_partition(n_units, n_ranks, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def make_epilogue(bias=None, residual=None, ld_residual=0, act=NNT_ACT_NONE, aux=None, ld_aux=0,
                  causal=NNT_CAUSAL_NONE, workspace=None, workspace_bytes=0, row_stats=None, ld_row_stats=0,
                  rowvec=None, rowscale=1.0, a_rowsum=None, scatter=None):
    """The caller keeps every tensor passed here alive until the launch has run (scatter: an
    nnt_tp_comm, kept alive too)."""
    if workspace is not None and not workspace_bytes and hasattr(workspace, "numel"):
        workspace_bytes = workspace.numel() * workspace.element_size()
    return nnt_epilogue(ptr(bias), ptr(residual), ld_residual, act, ptr(aux), ld_aux, causal, ptr(workspace),
                        workspace_bytes, ptr(row_stats), ld_row_stats, ptr(rowvec), rowscale, ptr(a_rowsum),
                        C.pointer(scatter) if scatter is not None else None)


def make_tp_comm(R, rank, rows, cols, recv, flags):
    """nnt_tp_comm for rank `rank` of R: recv[o] / flags[o] are device tensors or raw device addresses
    (rank o's buffers as mapped into this process).  Keep the buffers alive while it is used."""
    c = nnt_tp_comm()
    c.R, c.rank, c.rows, c.cols = R, rank, rows, cols
    for o in range(R):
        c.recv[o] = recv[o] if isinstance(recv[o], int) else ptr(recv[o])
        c.flags[o] = flags[o] if isinstance(flags[o], int) else ptr(flags[o])
    return c


def nnt_tp_signal(comm, epoch, which, stream=None):
    return check(lib.nnt_tp_signal(C.byref(comm), epoch, which, _stream(stream)))


def nnt_tp_reduce_gather(comm, out, epoch, stream=None):
    arr = (_vp * len(out))(*[o if isinstance(o, int) else ptr(o) for o in out])
    return check(lib.nnt_tp_reduce_gather(C.byref(comm), arr, epoch, _stream(stream)))


def nnt_tp_wait(comm, epoch, stream=None):
    return check(lib.nnt_tp_wait(C.byref(comm), epoch, _stream(stream)))


def nnt_tile_gemm_workspace_bytes(M, N, K, c_dtype, act=NNT_ACT_NONE, causal=NNT_CAUSAL_NONE, batch_items=1):
    return lib.nnt_tile_gemm_workspace_bytes(M, N, K, c_dtype, act, causal, batch_items)


def nnt_tile_gemm(trans_a, trans_b, M, N, K, batch, alpha, A, a_dtype, lda, stride_a, B, b_dtype, ldb, stride_b,
                  beta, Cm, c_dtype, ldc, stride_c, tile=None, epi=None, stream=None):
    return check(lib.nnt_tile_gemm(trans_a, trans_b, M, N, K, _arr64(batch), alpha, ptr(A), a_dtype, lda,
                                   _arr64(stride_a), ptr(B), b_dtype, ldb, _arr64(stride_b), beta, ptr(Cm),
                                   c_dtype, ldc, _arr64(stride_c), _arr64(tile),
                                   C.byref(epi) if epi is not None else None, _stream(stream)))


def nnt_maxsumexp(x, rows, cols, ldx, tile_k, causal, seq_q, stats, accumulate=0, stream=None):
    return check(lib.nnt_maxsumexp(ptr(x), rows, cols, ldx, tile_k, causal, seq_q, ptr(stats), accumulate,
                                   _stream(stream)))


def nnt_maxsumexp_merge(part, rows, nparts, ld_parts, part_cols, causal, seq_q, stats, stream=None):
    return check(lib.nnt_maxsumexp_merge(ptr(part), rows, nparts, ld_parts, part_cols, causal, seq_q, ptr(stats),
                                         _stream(stream)))


def nnt_attn_rowdot(dO, O, dtype, B, S, H, h, D, stream=None):
    return check(lib.nnt_attn_rowdot(ptr(dO), ptr(O), dtype, B, S, H, h, ptr(D), _stream(stream)))


def nnt_stf_build(n_handles, tasks):
    """tasks: list of [(handle, mode), ...] in submission order (modes 0 R, 1 W, 2 RW, 3 Reduce).
    Returns (levels, deps) with deps[t] the sorted predecessor list of task t."""
    import numpy as np
    n = len(tasks)
    n_acc = np.array([len(t) for t in tasks], np.int32)
    hs = np.array([h for t in tasks for h, _ in t], np.int64)
    ms = np.array([m for t in tasks for _, m in t], np.int32)
    level = np.zeros(max(n, 1), np.int32)
    offs = np.zeros(n + 1, np.int64)
    cap = max(1, n * n)
    ids = np.zeros(cap, np.int32)
    p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    check(lib.nnt_stf_build(n_handles, n, p(n_acc), p(hs), p(ms), level.ctypes.data, offs.ctypes.data,
                            ids.ctypes.data, cap))
    return level[:n].tolist(), [ids[offs[t]:offs[t + 1]].tolist() for t in range(n)]


def nnt_attention_trace(enable, out=None):
    """out: a numpy uint64 array (filled with the last trace) or None."""
    return check(lib.nnt_attention_trace(enable, out.ctypes.data if out is not None else None,
                                         out.size if out is not None else 0))


def nnt_attention_fused_supported(S, h):
    return bool(lib.nnt_attention_fused_supported(S, h))


def nnt_attention_stats(qkv, B, S, H, h, scale, causal, stats, stream=None):
    return check(lib.nnt_attention_stats(ptr(qkv), B, S, H, h, scale, causal, ptr(stats), _stream(stream)))


def nnt_attention_stats_enabled():
    return lib.nnt_attention_stats_enabled()


def nnt_attention_fwd_pv(qkv, B, S, H, h, scale, causal, stats, P, O, stream=None):
    return check(lib.nnt_attention_fwd_pv(ptr(qkv), B, S, H, h, scale, causal, ptr(stats), ptr(P), ptr(O),
                                          _stream(stream)))


def nnt_attention_bwd_kv(qkv, dO, P, D, B, S, H, h, scale, causal, dA, dqkv, stream=None):
    return check(lib.nnt_attention_bwd_kv(ptr(qkv), ptr(dO), ptr(P), ptr(D), B, S, H, h, scale, causal, ptr(dA),
                                          ptr(dqkv), _stream(stream)))


def nnt_softmax(x, rows, cols, ldx, tile_k, causal, seq_q, stats, y, y_dtype, ldy, stream=None):
    return check(lib.nnt_softmax(ptr(x), rows, cols, ldx, tile_k, causal, seq_q, ptr(stats), ptr(y), y_dtype, ldy,
                                 _stream(stream)))


def nnt_softmax_bwd(p, p_dtype, ldp, dp, lddp, rows, cols, causal, seq_q, scale, da, da_dtype, ldda, stream=None):
    return check(lib.nnt_softmax_bwd(ptr(p), p_dtype, ldp, ptr(dp), lddp, rows, cols, causal, seq_q, scale, ptr(da),
                                     da_dtype, ldda, _stream(stream)))


def nnt_layernorm_fwd(x, T, E, ldx, tile_e, gamma, beta, eps, y, y_dtype, ldy, mean, rstd, stream=None):
    return check(lib.nnt_layernorm_fwd(ptr(x), T, E, ldx, tile_e, ptr(gamma), ptr(beta), eps, ptr(y), y_dtype, ldy,
                                       ptr(mean), ptr(rstd), _stream(stream)))


def nnt_layernorm_bwd_scratch_bytes(T, E):
    return lib.nnt_layernorm_bwd_scratch_bytes(T, E)


def nnt_layernorm_bwd(dy, lddy, x, ldx, mean, rstd, gamma, T, E, dres, dx, lddx, dx_bf16, dgamma, dbeta,
                      dx_colsum, accumulate_params, scratch, scratch_bytes, stream=None):
    return check(lib.nnt_layernorm_bwd(ptr(dy), lddy, ptr(x), ldx, ptr(mean), ptr(rstd), ptr(gamma), T, E,
                                       ptr(dres), ptr(dx), lddx, ptr(dx_bf16), ptr(dgamma), ptr(dbeta),
                                       ptr(dx_colsum), accumulate_params, ptr(scratch), scratch_bytes,
                                       _stream(stream)))


def nnt_gelu_fwd(x, y, dtype, n, stream=None):
    return check(lib.nnt_gelu_fwd(ptr(x), ptr(y), dtype, n, _stream(stream)))


def nnt_gelu_bwd(x, dy, dx, dtype, n, stream=None):
    return check(lib.nnt_gelu_bwd(ptr(x), ptr(dy), ptr(dx), dtype, n, _stream(stream)))


def nnt_bias_grad_scratch_bytes(T, N):
    return lib.nnt_bias_grad_scratch_bytes(T, N)


def nnt_bias_grad(dy, dy_dtype, T, N, lddy, db, accumulate, dy_bf16_out, scratch, scratch_bytes, stream=None):
    return check(lib.nnt_bias_grad(ptr(dy), dy_dtype, T, N, lddy, ptr(db), accumulate, ptr(dy_bf16_out),
                                   ptr(scratch), scratch_bytes, _stream(stream)))


def nnt_adam_step(n, w, g, m, v, w_bf16, hp, stream=None):
    return check(lib.nnt_adam_step(n, ptr(w), ptr(g), ptr(m), ptr(v), ptr(w_bf16), C.byref(hp), _stream(stream)))


def nnt_sgd_step(n, w, g, buf, w_bf16, lr, momentum, weight_decay, stream=None):
    return check(lib.nnt_sgd_step(n, ptr(w), ptr(g), ptr(buf), ptr(w_bf16), lr, momentum, weight_decay,
                                  _stream(stream)))


def nnt_adam_tick(beta1, beta2, t_dev, bias_corr_dev, stream=None):
    return check(lib.nnt_adam_tick(beta1, beta2, ptr(t_dev), ptr(bias_corr_dev), _stream(stream)))


def nnt_convert(x, x_dtype, y, y_dtype, n, stream=None):
    return check(lib.nnt_convert(ptr(x), x_dtype, ptr(y), y_dtype, n, _stream(stream)))


def nnt_scale(x, alpha, y, n, stream=None):
    return check(lib.nnt_scale(ptr(x), alpha, ptr(y), n, _stream(stream)))


def nnt_dot_scratch_bytes(n):
    return lib.nnt_dot_scratch_bytes(n)


def nnt_dot(y, r, n, scale, out, scratch, scratch_bytes, stream=None):
    return check(lib.nnt_dot(ptr(y), ptr(r), n, scale, ptr(out), ptr(scratch), scratch_bytes, _stream(stream)))


def nnt_embedding_fwd(ids, T, S, wte, V, wpe, E, x, stream=None):
    return check(lib.nnt_embedding_fwd(ptr(ids), T, S, ptr(wte), V, ptr(wpe), E, ptr(x), _stream(stream)))


def nnt_embedding_bwd_scratch_bytes(T, V):
    return lib.nnt_embedding_bwd_scratch_bytes(T, V)


def nnt_embedding_bwd(ids, T, S, dx, E, dwte, V, dwpe, accumulate_wte, accumulate_wpe, scratch, scratch_bytes,
                      stream=None):
    return check(lib.nnt_embedding_bwd(ptr(ids), T, S, ptr(dx), E, ptr(dwte), V, ptr(dwpe), accumulate_wte,
                                       accumulate_wpe, ptr(scratch), scratch_bytes, _stream(stream)))


def nnt_cross_entropy(logits, dtype, rows, V, ld, labels, scale, loss_rows, stats, dlogits, ld_d, stream=None):
    return check(lib.nnt_cross_entropy(ptr(logits), dtype, rows, V, ld, ptr(labels), scale, ptr(loss_rows), ptr(stats),
                                       ptr(dlogits), ld_d, _stream(stream)))


def nnt_block_workspace_size(cfg):
    a, b = C.c_size_t(), C.c_size_t()
    check(lib.nnt_block_workspace_size(C.byref(cfg), C.byref(a), C.byref(b)))
    return a.value, b.value


def nnt_block_tp_workspace_size(cfg, tp):
    a, b = C.c_size_t(), C.c_size_t()
    check(lib.nnt_block_tp_workspace_size(C.byref(cfg), C.byref(tp), C.byref(a), C.byref(b)))
    return a.value, b.value


def nnt_block_tp_fwd(cfg, tp, params, stage, x, x1, y, saved, scratch, stream=None):
    return check(lib.nnt_block_tp_fwd(C.byref(cfg), C.byref(tp), C.byref(params), stage, ptr(x), ptr(x1), ptr(y),
                                      ptr(saved), ptr(scratch), _stream(stream)))


def nnt_block_tp_bwd(cfg, tp, params, stage, x, x1, saved, scratch, dy, dh, dx, grads, accumulate_grads,
                     stream=None):
    return check(lib.nnt_block_tp_bwd(C.byref(cfg), C.byref(tp), C.byref(params), stage, ptr(x), ptr(x1), ptr(saved),
                                      ptr(scratch), ptr(dy), ptr(dh), ptr(dx), C.byref(grads), accumulate_grads,
                                      _stream(stream)))


def nnt_block_fwd(cfg, params, x, y, saved, scratch, stream=None):
    return check(lib.nnt_block_fwd(C.byref(cfg), C.byref(params), ptr(x), ptr(y), ptr(saved), ptr(scratch),
                                   _stream(stream)))


def nnt_block_bwd_streams(cfg, params, x, saved, scratch, dy, dx, grads, accumulate_grads, grad_ready=None,
                          stream=None, side_stream=None, links=None):
    ev = _events(grad_ready)
    return check(lib.nnt_block_bwd_streams(C.byref(cfg), C.byref(params), ptr(x), ptr(saved), ptr(scratch), ptr(dy),
                                           ptr(dx), C.byref(grads), accumulate_grads, ev, _stream(stream),
                                           None if side_stream is None else _stream(side_stream),
                                           C.byref(links) if links is not None else None))


def _events(grad_ready):
    if grad_ready is None:
        return None
    handles = [e.cuda_event if hasattr(e, "cuda_event") else e for e in grad_ready]
    # torch creates an Event's CUDA handle lazily at its first record(): a 0 handle here would
    # silently disable the event (the library skips NULL events) and race the comm stream
    if not all(handles):
        raise ValueError("nnt_block_bwd: grad_ready events must be created (record() once) before use")
    return (C.c_void_p * 4)(*handles)


def nnt_block_bwd(cfg, params, x, saved, scratch, dy, dx, grads, accumulate_grads, grad_ready=None, stream=None):
    return check(lib.nnt_block_bwd(C.byref(cfg), C.byref(params), ptr(x), ptr(saved), ptr(scratch), ptr(dy), ptr(dx),
                                   C.byref(grads), accumulate_grads, _events(grad_ready), _stream(stream)))


def nnt_op_name(op):
    return lib.nnt_op_name(op).decode()


def nnt_block_dag_describe(cfg, pass_):
    nt, ng = C.c_int64(), C.c_int64()
    check(lib.nnt_block_dag_describe(C.byref(cfg), pass_, None, 0, C.byref(nt), None, 0, C.byref(ng)))
    tasks = (nnt_task * nt.value)()
    groups = (nnt_launch_group * ng.value)()
    check(lib.nnt_block_dag_describe(C.byref(cfg), pass_, tasks, nt.value, C.byref(nt), groups, ng.value,
                                     C.byref(ng)))
    return list(tasks), list(groups)


def nnt_timing_enable(enable=True):
    return check(lib.nnt_timing_enable(1 if enable else 0))


def nnt_timing_read():
    n = len(KERNEL_CLASSES)
    ms, cnt, by, fl = (C.c_double * n)(), (C.c_int64 * n)(), (C.c_double * n)(), (C.c_double * n)()
    check(lib.nnt_timing_read(ms, cnt, by, fl))
    return {KERNEL_CLASSES[i]: dict(ms=ms[i], launches=cnt[i], bytes=by[i], flops=fl[i]) for i in range(n)}


def nnt_timing_trace():
    """[(kernel class name, kernels launched)] for every recorded launch scope, in issue order."""
    n = C.c_int64()
    check(lib.nnt_timing_trace(None, None, 0, C.byref(n)))
    kc, kn = (C.c_int32 * max(n.value, 1))(), (C.c_int32 * max(n.value, 1))()
    check(lib.nnt_timing_trace(kc, kn, n.value, C.byref(n)))
    return [(KERNEL_CLASSES[kc[i]], kn[i]) for i in range(n.value)]


def nnt_launch_count():
    return lib.nnt_launch_count()
