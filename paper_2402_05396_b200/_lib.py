"""ctypes binding of libtaser_b200.so (the C-ABI in include/taser_b200.h).

This is the only place Python touches native code.  There is no fallback:
the library is mapped on first use (``lib``, ``load()``) and a missing
library raises ImportError there; every entry point checks that its tensors
live on a CUDA device.  Loading lazily keeps CPU-only processes that only
read spec tables (bench.py's reference arm) from mapping the product .so.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_double, c_int, c_int32, c_int64, c_uint64, c_ulonglong, c_void_p

import numpy as np

LIB_NAME = "libtaser_b200.so"
ABI_VERSION = 4  # include/taser_b200.h TG_ABI_VERSION: the struct layouts below
# TG_LIB_PATH: a diagnosis build of the same sources (csrc/Makefile EXTRA=...)
LIB_PATH = os.environ.get("TG_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

TG_OK, TG_EVALUE, TG_EINDEX, TG_EDATA, TG_ECONFIG, TG_ECUDA, TG_EFLOAT = 0, -1, -2, -3, -4, -5, -6
TG_RECENT, TG_UNIFORM = 0, 1


class DataError(ValueError):
    """Malformed input data (mirrors graph.py:20 DataError)."""


class ConfigError(ValueError):
    """Invalid sampler configuration (mirrors sampler.py:25 ConfigError)."""


class tg_rowmap(Structure):
    _fields_ = [("split", c_int64), ("base0", c_int64), ("base1", c_int64)]


class tg_graph(Structure):
    _fields_ = [("offsets", c_void_p), ("nbr", c_void_p), ("adj_ts", c_void_p), ("adj_eid", c_void_p),
                ("num_nodes", c_int64), ("num_adj", c_int64), ("coarse_off", c_void_p), ("coarse_ts", c_void_p),
                ("coarse_shift", c_int32), ("reserved", c_int32)]


class tg_feat_store(Structure):
    _fields_ = [("table", c_void_p), ("hot", c_void_p), ("peers", c_void_p), ("shard_rows", c_int64),
                ("n_peers", c_int32), ("d", c_int32), ("ld", c_int64), ("hot_ld", c_int64),
                ("num_rows", c_int64)]


class tg_gather_seg(Structure):
    _fields_ = [("ids", c_void_p), ("mask", c_void_p), ("n", c_int64), ("out", c_void_p)]


class tg_cache_dev(Structure):
    _fields_ = [("slot_of", c_void_p), ("counters", c_void_p), ("stats", c_void_p), ("num_edges", c_int64)]


class tg_find_args(Structure):
    _fields_ = [("qv", c_void_p), ("qt", c_void_p), ("B", c_int64), ("m", c_int32), ("policy", c_int32),
                ("seed", c_uint64), ("rows", tg_rowmap),
                ("idx", c_void_p), ("cnt", c_void_p), ("ids", c_void_p), ("eids", c_void_p),
                ("dts", c_void_p), ("tss", c_void_p), ("mask", c_void_p),
                ("next_v", c_void_p), ("next_t", c_void_p), ("feat_out", c_void_p), ("feat_ld", c_int64),
                ("valid_count", c_void_p), ("window", c_void_p), ("seed_ptr", c_void_p)]


class tg_pcg64(Structure):
    _fields_ = [("state_hi", c_uint64), ("state_lo", c_uint64), ("inc_hi", c_uint64), ("inc_lo", c_uint64),
                ("jmul_hi", c_uint64), ("jmul_lo", c_uint64), ("jadd_hi", c_uint64), ("jadd_lo", c_uint64)]


class tg_score_model(Structure):
    _fields_ = [("dtype", c_int32), ("decoder", c_int32), ("m", c_int32), ("F", c_int32), ("d_v", c_int32),
                ("d_e", c_int32), ("d_enc", c_int32), ("d_tv", c_int32), ("gemm_path", c_int32),
                ("slope", c_double)] + [
        (name, c_void_p) for name in ("W_node", "W_edge", "ln1_g", "ln1_b", "Wc1", "bc1", "Wc2", "bc2", "ln2_g",
                                      "ln2_b", "Wt1", "bt1", "Wt2", "bt2", "w_linear", "W_gat", "a_gat", "W_gatv2",
                                      "a_gatv2", "W_trans_target", "W_trans_nbr", "omega", "fe_table")]


GRAD_FIELDS = ("W_node", "W_edge", "ln1_g", "ln1_b", "Wc1", "bc1", "Wc2", "bc2", "ln2_g", "ln2_b", "Wt1", "bt1",
               "Wt2", "bt2", "w_linear", "W_gat", "a_gat", "W_gatv2", "a_gatv2", "W_trans_target", "W_trans_nbr")


class tg_score_grads(Structure):
    _fields_ = [(name, c_void_p) for name in GRAD_FIELDS]


class tg_gmixer_model(Structure):
    _fields_ = [("dtype", c_int32), ("n", c_int32), ("d_v", c_int32), ("d_e", c_int32), ("d_time", c_int32),
                ("gemm_path", c_int32)] + [
        (name, c_void_p) for name in ("time_w", "time_b", "ln1_g", "ln1_b", "Wc1", "bc1", "Wc2", "bc2", "ln2_g",
                                      "ln2_b", "Wt1", "bt1", "Wt2", "bt2")]


class tg_tgat_layer(Structure):
    _fields_ = [("dtype", c_int32), ("gemm_path", c_int32), ("d_in", c_int32), ("d_e", c_int32),
                ("d_time", c_int32), ("d_out", c_int32), ("s", c_int32)] + [
        (name, c_void_p) for name in ("time_w", "time_b", "W_q", "b_s", "W_k", "b_k", "W_v", "b_v")]


# name -> (restype, argtypes); must cover every symbol in include/taser_b200.h
_SIGNATURES = {
    "tg_abi_version": (c_int, []),
    "tg_last_error": (ctypes.c_char_p, []),
    "tg_launch_count": (c_ulonglong, []),
    "tg_device_sms": (c_int, [POINTER(c_int)]),
    "tg_graph_launch": (c_int, [c_void_p, c_void_p]),
    "tg_graph_upload": (c_int, [c_void_p, c_void_p]),
    "tg_tcsr_check": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, POINTER(c_int64), c_void_p]),
    "tg_tcsr_build": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_tcsr_coarse": (c_int, [POINTER(tg_graph), c_int32, c_void_p, c_void_p, c_void_p]),
    "tg_gather_rows_f32": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_void_p]),
    "tg_find": (c_int, [POINTER(tg_graph), POINTER(tg_find_args), POINTER(tg_feat_store), POINTER(tg_cache_dev),
                        c_void_p]),
    "tg_find_batch": (c_int, [POINTER(tg_graph), POINTER(tg_find_args), c_int32, POINTER(tg_cache_dev), c_void_p]),
    "tg_lookup_gather": (c_int, [c_void_p, c_void_p, c_int64, POINTER(tg_feat_store), POINTER(tg_cache_dev),
                                 c_int32, c_void_p, c_int64, c_void_p]),
    "tg_gather_rows": (c_int, [c_void_p, c_void_p, c_int64, POINTER(tg_feat_store), c_void_p, c_int32, c_void_p,
                               c_int64, c_void_p]),
    "tg_gather_rows_multi": (c_int, [POINTER(tg_gather_seg), c_int32, POINTER(tg_feat_store), c_void_p, c_int32,
                                     c_int64, c_void_p]),
    "tg_cache_lookup": (c_int, [c_void_p, c_int64, POINTER(tg_cache_dev), c_void_p, POINTER(tg_feat_store),
                                c_void_p, c_int64, c_void_p]),
    "tg_check_range": (c_int, [c_void_p, c_int64, c_int64, c_void_p]),
    "tg_cache_replace": (c_int, [POINTER(tg_cache_dev), c_int64, c_int64, POINTER(tg_feat_store), c_void_p, c_int64,
                                 POINTER(c_int64), c_void_p]),
    "tg_topk_mask": (c_int, [c_void_p, c_int64, c_int64, c_void_p, POINTER(c_int64), c_void_p]),
    "tg_sample_wor": (c_int, [c_void_p, c_void_p, c_int32, c_int64, c_int32, c_int32, POINTER(tg_pcg64), tg_rowmap,
                              c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_select_expand": (c_int, [c_void_p] * 7 + [c_int64, c_int32, c_int32] + [c_void_p] * 6),
    "tg_score_workspace": (c_int, [POINTER(tg_score_model), c_int64, POINTER(ctypes.c_size_t)]),
    "tg_score": (c_int, [POINTER(tg_score_model), c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                         c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, ctypes.c_size_t, c_void_p]),
    "tg_tc_gemm_workspace": (c_int, [c_int64, c_int, c_int, POINTER(ctypes.c_size_t)]),
    "tg_tc_gemm": (c_int, [c_void_p, c_int64, c_int64, c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p, c_int64,
                           c_void_p, c_void_p]),
    "tg_graphmixer_workspace": (c_int, [POINTER(tg_gmixer_model), c_int64, POINTER(ctypes.c_size_t)]),
    "tg_score_backward_workspace": (c_int, [POINTER(tg_score_model), c_int64, POINTER(ctypes.c_size_t)]),
    "tg_score_backward": (c_int, [POINTER(tg_score_model), c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                  c_int64, c_void_p, c_int64, c_int64, c_void_p, POINTER(tg_score_grads), c_void_p,
                                  ctypes.c_size_t, c_void_p]),
    "tg_score_stage_workspace": (c_int, [POINTER(tg_score_model), c_int64, POINTER(ctypes.c_size_t)]),
    "tg_encode_neighborhood": (c_int, [POINTER(tg_score_model), c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                       c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p, ctypes.c_size_t,
                                       c_void_p]),
    "tg_encode_target": (c_int, [POINTER(tg_score_model), c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p,
                                 ctypes.c_size_t, c_void_p]),
    "tg_mixer_transform": (c_int, [POINTER(tg_score_model), c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                   c_void_p, ctypes.c_size_t, c_void_p]),
    "tg_decode_policy": (c_int, [POINTER(tg_score_model), c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64,
                                 c_void_p, c_int64, c_void_p, c_void_p, c_void_p, ctypes.c_size_t, c_void_p]),
    "tg_graphmixer_forward": (c_int, [POINTER(tg_gmixer_model), c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                      c_void_p, c_int64, c_void_p, c_int64, c_void_p, ctypes.c_size_t, c_void_p]),
    "tg_tgat_workspace": (c_int, [POINTER(tg_tgat_layer), c_int64, POINTER(ctypes.c_size_t)]),
    "tg_tgat_forward": (c_int, [POINTER(tg_tgat_layer), c_void_p, c_int64, c_int32, c_void_p, c_int64, c_int32,
                                c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_void_p,
                                c_void_p, ctypes.c_size_t, c_void_p]),
    "tg_ingest_lines": (c_int, [c_void_p, c_int64, c_void_p, POINTER(c_int64), c_void_p]),
    "tg_ingest_classify": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                   POINTER(c_int64), c_void_p]),
    "tg_ingest_parse": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int32,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                                POINTER(c_int64), c_void_p]),
    "tg_select_batch": (c_int, [c_void_p, c_int64, c_int64, POINTER(tg_pcg64), c_int64, c_void_p, POINTER(c_int64),
                                c_void_p]),
    "tg_update_scores": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_double, c_void_p]),
    "tg_scatter_scores": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "tg_tgat_sample_coeffs": (c_int, [c_int32, c_int64, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_graphmixer_sample_coeffs": (c_int, [c_int32, c_int64, c_int32, c_int32, c_int32, c_int32, c_void_p, c_int64,
                                            c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_void_p, c_void_p]),
    "tg_mixer_sample_coeffs": (c_int, [c_int32, c_int64, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_int64,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_logq_surrogate_grad": (c_int, [c_int32, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_adam_step": (c_int, [c_int32, c_void_p, c_int32, c_double, c_double, c_double, c_double, c_double,
                             c_double, c_void_p]),
    "tg_ipc_handle_size": (c_int, []),
    "tg_ipc_export": (c_int, [c_void_p, c_void_p, POINTER(c_int64)]),
    "tg_ipc_open": (c_int, [c_void_p, POINTER(c_void_p)]),
    "tg_ipc_close": (c_int, [c_void_p]),
    "tg_peer_access": (c_int, [c_int, POINTER(c_int)]),
    "tg_synth_events": (c_int, [c_int64, c_int64, c_int64, c_int64, c_uint64, c_void_p, c_void_p, c_int32, c_double,
                                c_void_p, c_void_p, c_void_p, c_void_p]),
    "tg_synth_features": (c_int, [c_int64, c_int64, c_int32, c_uint64, c_void_p, c_int64, c_void_p]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2402_05396_b200/csrc`).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tg_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI {lib.tg_abi_version()}, this package binds ABI {ABI_VERSION}: rebuild it")
    return lib


def load():
    """The ctypes handle of libtaser_b200.so, mapped on first call."""
    global _handle
    if _handle is None:
        _handle = _load()
    return _handle


_handle = None


def __getattr__(name):
    # module attribute ``_lib.lib`` (PEP 562): map the library on first access
    if name == "lib":
        return load()
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")

_EXC = {TG_EVALUE: ValueError, TG_EINDEX: IndexError, TG_EDATA: DataError, TG_ECONFIG: ConfigError,
        TG_ECUDA: RuntimeError, TG_EFLOAT: FloatingPointError}


def check(rc):
    """Raise the reference's exception type for a non-zero status."""
    if rc != TG_OK:
        msg = load().tg_last_error().decode("utf-8", "replace")
        raise _EXC.get(rc, RuntimeError)(msg)


def launch_count():
    return int(load().tg_launch_count())


# ---------------------------------------------------------------------------
# tensor plumbing (torch is the device-memory/stream provider)
# ---------------------------------------------------------------------------

def torch():
    import torch as _t
    return _t


def require_cuda(what="this operation"):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(f"{what} needs a CUDA device (B200); there is no CPU path")


def stream_ptr(stream=None):
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(x):
    """Device address of a tensor (None -> NULL)."""
    if x is None:
        return None
    if not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return ctypes.c_void_p(x.data_ptr())


def to_device(x, dtype, device=None, rows_ok=False):
    """numpy / list / tensor -> contiguous CUDA tensor of `dtype`.
    rows_ok: a 2-d CUDA tensor whose rows are contiguous (a row-pitched
    feature table view) is passed through without a copy."""
    t = torch()
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    if isinstance(x, t.Tensor):
        if (rows_ok and x.is_cuda and x.dtype == dtype and x.dim() == 2 and x.stride(1) == 1
                and (device is None or x.device == t.device(dev))):
            return x
        return x.to(device=dev, dtype=dtype).contiguous()
    arr = np.asarray(x)
    return t.as_tensor(np.ascontiguousarray(arr)).to(device=dev, dtype=dtype).contiguous()


class tg_adam_tensor(ctypes.Structure):
    _fields_ = [("p", c_void_p), ("g", c_void_p), ("m", c_void_p), ("v", c_void_p), ("n", c_int64),
                ("g_dtype", c_int32)]


def rowmap(split=None, base0=0, base1=0):
    if split is None:
        split = 1 << 62
    return tg_rowmap(int(split), int(base0), int(base1))


def u128_split(x):
    x &= (1 << 128) - 1
    return (x >> 64) & 0xFFFFFFFFFFFFFFFF, x & 0xFFFFFFFFFFFFFFFF
