"""The bm25.hpp half of the drop-in boundary: reference code that includes
<sparselex/bm25.hpp> links against libsparselex_b200.so unchanged and gets the reference's results.

tests/cpp/bm25_caller.cpp (a reference-side caller of every bm25.hpp function) is compiled with
the REFERENCE's own header twice: linked with the reference's proj/src/scoring.cpp, and linked with
libsparselex_b200.so instead. On 6,000 random argument tuples (valid and invalid) every result
must be bit-identical and every std::invalid_argument message identical. The same caller is also
built against this repo's include/sparselex/bm25.hpp, and the C-ABI twins (sl_idf, ...) are checked
against the reference. Host-only: no GPU.
"""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from paper_2407_03618_b200._lib import Params, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2407_03618_b200")
REF = "/root/reference/proj"
CALLER = os.path.join(ROOT, "tests", "cpp", "bm25_caller.cpp")
HAVE_REF = os.path.exists(os.path.join(REF, "src", "scoring.cpp"))


def _build(tmp_path, name, include, link_ours):
    out = str(tmp_path / f"lib{name}.so")
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-I", include, CALLER]
    if link_ours:
        cmd += ["-L", PKG, "-lsparselex_b200", f"-Wl,-rpath,{PKG}", "-Wl,--no-undefined"]
    else:
        cmd += [os.path.join(REF, "src", "scoring.cpp")]
    subprocess.run(cmd + ["-o", out], check=True)
    L = C.CDLL(out)
    d, u, i, p = C.c_double, C.c_uint32, C.c_int, C.c_void_p
    sig = {"caller_msg": (C.c_char_p, []), "caller_from_string": (i, [C.c_char_p, C.POINTER(i)]),
           "caller_to_string": (i, [i, C.c_char_p, i]), "caller_is_sparse": (i, [i]),
           "caller_default_delta": (d, [i]), "caller_for_variant": (i, [i, d, d, p]),
           "caller_validate": (i, [i, d, d, d]), "caller_idf": (i, [i, u, u, C.POINTER(d)]),
           "caller_tf_component": (i, [d, d, d, i, d, d, d, C.POINTER(d)]),
           "caller_score": (i, [d, u, d, u, d, i, d, d, d, C.POINTER(d)]),
           "caller_nonoccurrence": (i, [u, u, i, d, d, d, C.POINTER(d)])}
    for n, (r, a) in sig.items():
        getattr(L, n).restype = r
        getattr(L, n).argtypes = a
    return L


def _call(L, fn, *args):
    out = C.c_double()
    rc = getattr(L, fn)(*args, C.byref(out))
    return (rc, out.value if rc == 0 else L.caller_msg().decode())


def _tuples(n=6000, seed=7):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        v = int(rng.integers(0, 6))
        N = int(rng.integers(1, 10**7))
        df = int(rng.integers(0, N + 2))  # includes df = 0 and df > N (invalid)
        tf = float(rng.integers(-1, 60)) if rng.random() < 0.9 else float(rng.uniform(0, 5))
        dl = float(rng.integers(0, 3000))
        avg = float(rng.uniform(1, 500)) if rng.random() < 0.97 else 0.0
        k1 = float(rng.uniform(0.0, 2.5))
        b = float(rng.uniform(-0.1, 1.1))
        delta = float(rng.choice([0.0, 0.1, 0.3, 0.5, 1.0, float(rng.uniform(0, 2))]))
        yield v, N, df, tf, dl, avg, k1, b, delta


def _compare(A, B):
    for name in ("robertson", "atire", "lucene", "bm25l", "bm25plus", "tfldp", "BM25", "", "okapi"):
        ra, rb = C.c_int(-1), C.c_int(-1)
        ea = A.caller_from_string(name.encode(), C.byref(ra))
        ma = A.caller_msg().decode() if ea else ra.value
        eb = B.caller_from_string(name.encode(), C.byref(rb))
        mb = B.caller_msg().decode() if eb else rb.value
        assert (ea, ma) == (eb, mb), name
    for v in range(-1, 7):
        ba, bb = C.create_string_buffer(32), C.create_string_buffer(32)
        ea, eb = A.caller_to_string(v, ba, 32), B.caller_to_string(v, bb, 32)
        assert (ea, ba.value if ea == 0 else A.caller_msg()) == (eb, bb.value if eb == 0 else B.caller_msg()), v
        if 0 <= v < 6:
            assert A.caller_is_sparse(v) == B.caller_is_sparse(v)
            assert A.caller_default_delta(v) == B.caller_default_delta(v)
            oa, ob = (C.c_double * 4)(), (C.c_double * 4)()
            assert A.caller_for_variant(v, 1.2, 0.4, oa) == B.caller_for_variant(v, 1.2, 0.4, ob) == 0
            assert list(oa) == list(ob)
    for v, N, df, tf, dl, avg, k1, b, delta in _tuples():
        va, vb = A.caller_validate(v, k1, b, delta), B.caller_validate(v, k1, b, delta)
        assert va == vb and (va == 0 or A.caller_msg() == B.caller_msg())
        assert _call(A, "caller_idf", v, df, N) == _call(B, "caller_idf", v, df, N)
        args = (tf, dl, avg, v, k1, b, delta)
        assert _call(A, "caller_tf_component", *args) == _call(B, "caller_tf_component", *args), args
        args = (tf, df, dl, N, avg, v, k1, b, delta)
        assert _call(A, "caller_score", *args) == _call(B, "caller_score", *args), args
        args = (df, N, v, k1, b, delta)
        assert _call(A, "caller_nonoccurrence", *args) == _call(B, "caller_nonoccurrence", *args), args


@pytest.mark.skipif(not HAVE_REF, reason="reference tree absent (the comparison needs its scoring.cpp)")
def test_reference_caller_links_unchanged(tmp_path):
    ref = _build(tmp_path, "caller_ref", os.path.join(REF, "include"), link_ours=False)
    ours = _build(tmp_path, "caller_ours", os.path.join(REF, "include"), link_ours=True)
    _compare(ref, ours)


@pytest.mark.skipif(not HAVE_REF, reason="reference tree absent (the comparison needs its scoring.cpp)")
def test_our_header_matches_reference(tmp_path):
    ref = _build(tmp_path, "caller_ref2", os.path.join(REF, "include"), link_ours=False)
    ours = _build(tmp_path, "caller_ours2", os.path.join(ROOT, "include"), link_ours=True)
    _compare(ref, ours)


def test_our_header_links(tmp_path):
    ours = _build(tmp_path, "caller_ours3", os.path.join(ROOT, "include"), link_ours=True)
    assert _call(ours, "caller_idf", 2, 1, 3)[0] == 0
    assert _call(ours, "caller_idf", 2, 0, 3) == (1, "idf: df must satisfy 1 <= df <= num_docs")


def test_c_abi_scoring_twins():
    import oracle
    L = lib()
    out = C.c_double()
    iv = C.c_int32()
    assert L.sl_variant_from_string(b"bm25plus", C.byref(iv)) == 0 and iv.value == 4
    assert L.sl_variant_from_string(b"okapi", C.byref(iv)) == 1
    assert L.sl_last_error() == b"unknown BM25 variant: okapi"
    assert L.sl_variant_to_string(3) == b"bm25l" and L.sl_variant_to_string(9) is None
    assert [L.sl_is_sparse_variant(v) for v in range(6)] == [1, 1, 1, 0, 0, 0]
    R = oracle.ref() if oracle.ref_available() else None
    for v, N, df, tf, dl, avg, k1, b, delta in _tuples(1500, seed=8):
        p = Params(v, k1, b, delta)
        rc = L.sl_idf(v, df, N, C.byref(out))
        want = oracle.idf(v, df, N) if R is None else R.ref_idf(v, df, N)
        assert (rc == 0 and out.value == want) or (rc == 1 and np.isnan(want)), (v, df, N)
        rc = L.sl_score(tf, df, dl, N, avg, C.byref(p), C.byref(out))
        want = R.ref_score(tf, df, dl, N, avg, v, k1, b, delta) if R else None
        if R is not None:
            assert (rc == 0 and out.value == want) or (rc == 1 and np.isnan(want)), (v, tf, df, dl, N, avg)
        rc = L.sl_nonoccurrence_score(df, N, C.byref(p), C.byref(out))
        if R is not None:
            want = R.ref_nonoccurrence(df, N, v, k1, b, delta)
            assert (rc == 0 and out.value == want) or (rc == 1 and np.isnan(want))
