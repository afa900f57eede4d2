"""ctypes binding of the C-ABI in include/sparselex_b200.h (libsparselex_b200.so).

Loading fails loudly when the shared library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPARSELEX_LIB") or os.path.join(_HERE, "libsparselex_b200.so")  # env: tuning variants
SYNTH_PATH = os.path.join(_HERE, "libsl_synth.so")

SL_OK, SL_EINVAL, SL_ECUDA, SL_ENCCL, SL_ENOMEM, SL_ECORRUPT, SL_EUNSUPPORTED, SL_EIO = range(8)
SL_MEM_HOST, SL_MEM_DEVICE = 0, 1

# name, restype, argtypes — every symbol declared in include/sparselex_b200.h
_vp, _u8p, _u32, _u64, _i32 = C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32


class Params(C.Structure):
    _fields_ = [("variant", C.c_int32), ("k1", C.c_double), ("b", C.c_double), ("delta", C.c_double)]


class BuildDesc(C.Structure):
    _fields_ = [
        ("doc_offsets", C.c_void_p),
        ("token_ids", C.c_void_p),
        ("num_docs", C.c_uint32),
        ("vocab_size", C.c_uint32),
        ("doc_base", C.c_uint32),
        ("mem", C.c_int32),
        ("params", Params),
        ("device", C.c_int32),
        ("keep_tf", C.c_int32),
        ("dense_min_density", C.c_float),
        ("comm", C.c_void_p),
        ("global_df", C.c_void_p),
        ("global_num_docs", C.c_uint32),
        ("global_total_len", C.c_uint64),
    ]


class IndexInfo(C.Structure):
    _fields_ = [
        ("num_docs_local", C.c_uint32),
        ("num_docs_global", C.c_uint32),
        ("vocab_size", C.c_uint32),
        ("doc_base", C.c_uint32),
        ("nnz_local", C.c_uint64),
        ("total_len_global", C.c_uint64),
        ("avg_len", C.c_double),
        ("dense_rows", C.c_uint32),
        ("skip_rows", C.c_uint32),
        ("tile_docs", C.c_uint32),
        ("num_tiles", C.c_uint32),
        ("device_bytes", C.c_uint64),
        ("build_ms", C.c_float),
    ]


class RetrieveStats(C.Structure):
    _fields_ = [
        ("total_ms", C.c_float),
        ("score_kernel_ms", C.c_float),
        ("merge_ms", C.c_float),
        ("posting_bytes", C.c_uint64),
        ("scorevec_bytes", C.c_uint64),
        ("unique_posting_bytes", C.c_uint64),
        ("kernels_launched", C.c_uint32),
    ]


class TokenizerConfig(C.Structure):
    _fields_ = [("lowercase", C.c_int32), ("stemmer", C.c_int32), ("stopwords", C.c_char_p),
                ("stopwords_bytes", C.c_uint64)]


SIGNATURES = {
    "sl_abi_version": (_i32, []),
    "sl_last_error": (C.c_char_p, []),
    "sl_status_string": (C.c_char_p, [_i32]),
    "sl_params_validate": (_i32, [C.POINTER(Params)]),
    "sl_default_delta": (C.c_double, [_i32]),
    "sl_variant_from_string": (_i32, [C.c_char_p, C.POINTER(_i32)]),
    "sl_variant_to_string": (C.c_char_p, [_i32]),
    "sl_is_sparse_variant": (_i32, [_i32]),
    "sl_idf": (_i32, [_i32, _u32, _u32, C.POINTER(C.c_double)]),
    "sl_tf_component": (_i32, [C.c_double, C.c_double, _u32, C.c_double, C.POINTER(Params), C.POINTER(C.c_double)]),
    "sl_score": (_i32, [C.c_double, _u32, C.c_double, _u32, C.c_double, C.POINTER(Params), C.POINTER(C.c_double)]),
    "sl_nonoccurrence_score": (_i32, [_u32, _u32, C.POINTER(Params), C.POINTER(C.c_double)]),
    "sl_index_build": (_i32, [C.POINTER(BuildDesc), C.POINTER(C.c_void_p)]),
    "sl_index_destroy": (None, [_vp]),
    "sl_index_get_info": (_i32, [_vp, C.POINTER(IndexInfo)]),
    "sl_index_export": (_i32, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sl_index_save": (_i32, [_vp, C.c_char_p]),
    "sl_index_load": (_i32, [C.c_char_p, _i32, C.c_float, C.POINTER(C.c_void_p)]),
    "sl_retrieve_batch": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _i32, _vp, _vp]),
    "sl_retrieve_batch_timed": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _vp, _vp, C.POINTER(RetrieveStats)]),
    "sl_score_query": (_i32, [_vp, _vp, _u32, _i32, _vp]),
    "sl_top_k": (_i32, [_vp, _u32, _u32, _i32, _i32, _i32, _vp, _vp]),
    "sl_comm_unique_id": (_i32, [_u8p]),
    "sl_comm_init": (_i32, [_u8p, _i32, _i32, _i32, C.POINTER(C.c_void_p)]),
    "sl_comm_destroy": (None, [_vp]),
    "sl_retrieve_local": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _vp, _vp]),
    "sl_merge_candidates": (_i32, [_vp, _u32, _u32, _u32, _vp, _i32, _i32, _vp, _vp]),
    "sl_vocab_create": (_i32, [_i32, C.POINTER(C.c_void_p)]),
    "sl_vocab_destroy": (_i32, [_vp]),
    "sl_vocab_size": (_i32, [_vp, C.POINTER(_u32)]),
    "sl_vocab_export": (_i32, [_vp, _vp, _vp, C.POINTER(_u64)]),
    "sl_vocab_import": (_i32, [_vp, _vp, _vp, _u32]),
    "sl_tokenize": (_i32, [_vp, C.POINTER(TokenizerConfig), _i32, _vp, _vp, _u32, _i32, C.POINTER(C.c_void_p)]),
    "sl_tokenize_stream": (_i32, [_vp, C.POINTER(TokenizerConfig), _i32, _vp, _vp, _u32, _u64, _vp, _vp, _u64,
                                  C.POINTER(_u64)]),
    "sl_token_batch_info": (_i32, [_vp, C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_vp), C.POINTER(_vp)]),
    "sl_token_batch_copy": (_i32, [_vp, _vp, _vp]),
    "sl_token_batch_destroy": (_i32, [_vp]),
    "sl_stem_batch": (_i32, [_vp, _vp, _u32, _i32, _vp, _vp]),
    "sl_text_index_build": (_i32, [_vp, _vp, _vp, _vp, _u32, C.POINTER(Params), C.POINTER(TokenizerConfig), _i32,
                                   C.c_float, C.POINTER(C.c_void_p)]),
    "sl_text_index_destroy": (None, [_vp]),
    "sl_text_index_save": (_i32, [_vp, C.c_char_p]),
    "sl_text_index_load": (_i32, [C.c_char_p, _i32, C.c_float, C.POINTER(C.c_void_p)]),
    "sl_text_index_index": (_vp, [_vp]),
    "sl_text_index_vocab": (_vp, [_vp]),
    "sl_text_index_config": (_i32, [_vp, C.POINTER(TokenizerConfig)]),
    "sl_text_index_num_docs": (_i32, [_vp, C.POINTER(_u32)]),
    "sl_text_index_external_id": (_i32, [_vp, _u32, C.POINTER(C.c_void_p), C.POINTER(_u64)]),
    "sl_text_index_retrieve": (_i32, [_vp, _vp, _vp, _u32, _u32, _i32, _vp, _vp]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libsparselex_b200.so (raises if absent — the product has no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C paper_2407_03618_b200/csrc` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        # PyTorch carries the process's libnccl.so.2 / libcudart; load it first so the
        # library's lazily-resolved NCCL binds to the same copy torch.distributed uses.
        import torch  # noqa: F401
        L = C.CDLL(LIB_PATH)
        ab_build = bool(os.environ.get("SPARSELEX_LIB"))  # A/B tuning builds may predate some entry points
        for name, (res, args) in SIGNATURES.items():
            if ab_build and not hasattr(L, name):
                continue
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SparselexError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class SparselexInvalid(SparselexError, ValueError):
    """SL_EINVAL: the reference throws std::invalid_argument here."""


class SparselexIOError(SparselexError, OSError):
    """SL_EIO: file I/O failure (SPEC save_index / load_index)."""


def check(status: int) -> None:
    if status == SL_OK:
        return
    msg = (lib().sl_last_error() or b"").decode(errors="replace")
    if status == SL_EINVAL:
        raise SparselexInvalid(status, msg)
    if status == SL_EIO:
        raise SparselexIOError(status, msg)
    raise SparselexError(status, msg)


_synth = None


def synth_lib() -> C.CDLL:
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise RuntimeError(f"{SYNTH_PATH} is missing: build with `make -C paper_2407_03618_b200/csrc`")
        L = C.CDLL(SYNTH_PATH)
        L.sl_synth_tokens_device.restype = _i32
        L.sl_synth_tokens_device.argtypes = [_vp, _u32, _u32, _u64, _u64, _i32, _vp]
        _synth = L
    return _synth
