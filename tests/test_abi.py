"""The C-ABI library loads and exports every symbol include/*.h declares (no GPU calls)."""
import ctypes
import os
import re

from paper_2407_03618_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "sparselex_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sl_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_binding_table():
    assert declared_functions() == sorted(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(L, f)]
    assert not missing, missing


def test_abi_version_and_status_strings():
    L = _lib.lib()
    assert L.sl_abi_version() == 1
    assert L.sl_status_string(0) == b"ok"
    assert L.sl_status_string(1) == b"invalid argument"


def test_params_validate_is_host_only():
    from paper_2407_03618_b200 import BM25Params, Variant
    BM25Params().validate()
    import pytest
    for bad, msg in [(BM25Params(Variant.lucene, 0.0), "k1 must be > 0"),
                     (BM25Params(Variant.lucene, 1.5, 1.5), "b must be in"),
                     (BM25Params(Variant.bm25l, 1.5, 0.75, -1.0), "delta must be >= 0"),
                     (BM25Params(Variant.tfldp, 1.5, 0.75, 0.2), "tfldp requires")]:
        with pytest.raises(ValueError, match=msg):
            bad.validate()
    assert BM25Params.for_variant(Variant.bm25plus).delta == 1.0
    assert BM25Params.for_variant(Variant.bm25l).delta == 0.5
    assert BM25Params.for_variant(Variant.lucene).delta == 0.0


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        return
    import numpy as np
    import pytest
    from paper_2407_03618_b200 import build_index
    with pytest.raises(RuntimeError, match="no CUDA device"):
        build_index(np.array([0, 2], np.uint64), np.array([0, 1], np.uint32), 2)
