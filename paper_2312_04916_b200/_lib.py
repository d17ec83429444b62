"""ctypes binding of libee.so (the C-ABI declared in include/ee.h).

The product path has exactly one backend: the sm_100a CUDA library built
in-tree.  There is no CPU fallback — if the library is missing or no CUDA
device is present, every compute entry point raises.  Return codes map onto
the reference exception classes (`eepipe/errors.py:4-25`).
"""

from __future__ import annotations

import ctypes
import os

from .errors import ConfigError, NonFiniteError, ShapeError, TokenError

HERE = os.path.dirname(os.path.abspath(__file__))
# EE_LIB_PATH (profiling A/B only): load another in-tree build of the same ABI
LIB_PATH = os.environ.get("EE_LIB_PATH") or os.path.join(HERE, "libee.so")

EE_OK, EE_ESHAPE, EE_ETOKEN, EE_ENONFINITE, EE_ECONFIG, EE_ECUDA = range(6)
EE_F32, EE_BF16, EE_BF16_TILED = 0, 1, 2
EE_EPI_STORE, EE_EPI_RESIDUAL, EE_EPI_GELU = 0, 1, 2
EE_OP_ATTENTION, EE_OP_EXIT_HEAD, EE_OP_DECODER, EE_OP_EXIT_HEAD_TRAIN = 1, 2, 3, 4
EE_OP_RMSNORM_BWD = 5
EE_OP_PREFILL = 6
EE_OPT_SGD, EE_OPT_ADAM, EE_OPT_ACCUM = 0, 1, 2

_ERRORS = {EE_ESHAPE: ShapeError, EE_ETOKEN: TokenError, EE_ENONFINITE: NonFiniteError,
           EE_ECONFIG: ConfigError, EE_ECUDA: RuntimeError}

c_void_p, c_int64, c_int32, c_int, c_float, c_size_t = (
    ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int, ctypes.c_float, ctypes.c_size_t)


class EeLayer(ctypes.Structure):
    _fields_ = [("attn_norm", c_void_p), ("wqkv", c_void_p), ("wo", c_void_p),
                ("mlp_norm", c_void_p), ("w1", c_void_p), ("w2", c_void_p),
                ("kcache", c_void_p), ("vcache", c_void_p)]


class EeDecoder(ctypes.Structure):
    _fields_ = [("h", c_int64), ("nh", c_int64), ("s_max", c_int64), ("max_rows", c_int64),
                ("dtype", c_int), ("eps", c_float), ("x", c_void_p), ("xb", c_void_p),
                ("ssq", c_void_p), ("xn", c_void_p), ("q", c_void_p), ("attn", c_void_p),
                ("ws", c_void_p), ("ws_bytes", c_size_t), ("pf_ws", c_void_p),
                ("pf_ws_bytes", c_size_t)]


class EeHead(ctypes.Structure):
    _fields_ = [("tap", c_int32), ("is_final", c_int32), ("kind", c_int32), ("norm", c_void_p),
                ("pre_norm", c_void_p), ("w1t", c_void_p), ("w2t", c_void_p), ("W", c_void_p),
                ("V", c_int64)]


class EeEngine(ctypes.Structure):
    _fields_ = [("dec", c_void_p), ("layers", c_void_p), ("n_layers", c_int32),
                ("heads", c_void_p), ("n_heads", c_int32), ("dcode", c_int), ("wcode", c_int),
                ("eps", c_float), ("tok_emb", c_void_p), ("pos_emb", c_void_p),
                ("ctrl", c_void_p), ("ctrl_host", c_void_p), ("ctrl_cap", c_int64),
                ("head_ws", c_void_p), ("head_ws_bytes", c_size_t), ("head_x", c_void_p),
                ("head_xn", c_void_p), ("head_mid", c_void_p), ("res", c_void_p),
                ("res_host", c_void_p), ("res_stride", c_int32), ("max_slots", c_int32),
                ("off_tok", c_int32), ("off_conf", c_int32), ("off_fire", c_int32),
                ("off_bad", c_int32), ("stream", c_void_p), ("pf_ws", c_void_p),
                ("pf_ws_bytes", c_size_t)]


class EeGenerateArgs(ctypes.Structure):
    _fields_ = [("engine", c_void_p), ("prompt", c_void_p), ("prompt_len", c_int32),
                ("max_new", c_int32), ("max_deferred", c_int32), ("s_max", c_int32),
                ("head_max_rows", c_int32), ("threshold", c_float), ("n_heads", c_int32),
                ("tokens", c_void_p), ("exit_layers", c_void_p), ("pass_depths", c_void_p),
                ("latency_s", c_void_p), ("conf", c_void_p), ("kv_mask", c_void_p),
                ("n_generated", c_int32), ("flushed", c_int32), ("total_s", ctypes.c_double),
                ("launches", c_int64), ("h2d_bytes", c_int64), ("d2h_bytes", c_int64)]


# name -> (restype, argtypes); every symbol declared in include/ee.h
SIGNATURES = {
    "ee_last_error": (ctypes.c_char_p, []),
    "ee_abi_version": (c_int, []),
    "ee_device_sms": (c_int, []),
    "ee_workspace_bytes": (c_size_t, [c_int, c_int64, c_int64, c_int64, c_int64, c_int64]),
    "ee_tiled_weight_bytes": (c_size_t, [c_int64, c_int64]),
    "ee_pack_tiled": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "ee_row_stats": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "ee_embed": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int, c_void_p,
                         c_void_p]),
    "ee_embed_stats": (c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int,
                               c_void_p, c_void_p, c_void_p, c_void_p]),
    "ee_copy_h2d": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
    "ee_generate_kv_recompute": (c_int, [c_void_p]),
    "ee_rmsnorm_rows": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_float,
                                c_void_p, c_int, c_void_p]),
    "ee_gemv": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int, c_int, c_void_p,
                        c_int64, c_void_p]),
    "ee_qkv_kvwrite": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p]),
    "ee_decode_attention": (c_int, [c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                    c_int64, c_int64, c_int, c_void_p, c_void_p, c_size_t,
                                    c_void_p]),
    "ee_exit_head_infer": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p,
                                   c_float, c_void_p, c_int64, c_int, c_float, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ee_decode_layer": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int32,
                                c_void_p]),
    "ee_decode_layers": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p,
                                 c_int32, c_void_p]),
    "ee_exit_head_train": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                   c_float, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                   c_void_p]),
    "ee_wgrad_accum": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                               c_void_p]),
    "ee_rmsnorm_fwd": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_float, c_void_p, c_void_p,
                               c_void_p]),
    "ee_rmsnorm_bwd": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int64,
                               c_void_p, c_void_p, c_int, c_void_p, c_size_t, c_void_p]),
    "ee_mlp_up_gelu": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                               c_void_p]),
    "ee_mlp_gelu_bwd": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                c_void_p]),
    "ee_linear_fwd": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                              c_void_p]),
    "ee_linear_dgrad": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                c_void_p]),
    "ee_linear_fwd_stacked": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                      c_void_p, c_void_p]),
    "ee_linear_dgrad_stacked": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                        c_void_p, c_void_p, c_void_p]),
    "ee_wgrad_accum_stacked": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int64,
                                       c_void_p, c_void_p]),
    "ee_attn_train_fwd": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64,
                                  c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p]),
    "ee_attn_train_bwd": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                  c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                  c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                  c_void_p]),
    "ee_exit_head_train_fwd": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                       c_float, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ee_exit_head_train_bwd": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ee_optimizer_step": (c_int, [c_void_p, c_int32, c_int64, c_int, c_int, c_float, c_float,
                                  c_float, c_float, c_float, c_float, c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the library.  Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"libee.so not found at {path}; build it with "
            "`python -m paper_2312_04916_b200.build_lib` (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    if rc != EE_OK:
        msg = _lib.ee_last_error().decode(errors="replace") if _lib is not None else ""
        raise _ERRORS.get(rc, RuntimeError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args):
    lib = load()
    check(getattr(lib, name)(*args), name)


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2312_04916_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    load()


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def dtype_code(torch_dtype):
    import torch
    if torch_dtype == torch.float32:
        return EE_F32
    if torch_dtype == torch.bfloat16:
        return EE_BF16
    raise ConfigError(f"unsupported compute dtype {torch_dtype}")
