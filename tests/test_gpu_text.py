"""Device text pipeline (sl_tokenize / sl_stem_batch) against the
reference's golden fixtures and the CPU oracle (oracle/text_oracle.cpp, itself pinned to the
reference compiled in place). Token ids, per-document token offsets and the vocabulary (its
strings in id order) must be identical."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.text import TextOracle, bundled_stopwords
from paper_2407_03618_b200 import BM25Params, Variant
from paper_2407_03618_b200 import text as T
from paper_2407_03618_b200._lib import SparselexError
from tests.helpers import assert_topk_match, query_scale
from tests.text_words import make_corpus, make_words

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "text_golden.json")
CONFIGS = [(True, False, False), (True, True, False), (True, False, True), (True, True, True), (False, False, True)]


def cfg_of(lc, stop, stem):
    return T.TokenizerConfig(bool(lc), frozenset(bundled_stopwords()) if stop else frozenset(),
                             T.StemmerKind.snowball_english if stem else T.StemmerKind.none)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN, encoding="utf-8") as f:
        return json.load(f)


@pytest.fixture(scope="module")
def port():
    return TextOracle("port")


def gpu_tokenize(text, off, lc, stop, stem, vocab=None):
    v = vocab if vocab is not None else T.Vocabulary()
    b = T.tokenize_build((text, off), cfg_of(lc, stop, stem), v)
    toff, ids = b.to_numpy()
    b.close()
    return toff, ids, v.tokens(), v


def test_ac4_golden(cuda_ok, golden):
    texts = [bytes.fromhex(r["text_hex"]) for r in golden["ac4"]]
    for ci, (lc, stop, stem) in enumerate(golden["configs"]):
        v = T.Vocabulary()
        lists = T.tokenize_build(texts, cfg_of(lc, stop, stem), v).lists()
        toks = v.tokens()
        for row, ids in zip(golden["ac4"], lists):
            assert [toks[i] for i in ids] == row["tokens"][ci], (bytes.fromhex(row["text_hex"]), lc, stop, stem)


def test_stems_golden(cuda_ok, golden):
    words = [w for w, _ in golden["stems"]]
    assert T.stem_batch(words) == [s for _, s in golden["stems"]]


def test_stems_vs_oracle(cuda_ok, port):
    words = make_words(100000, seed=33, unicode_frac=0.1)
    words = words + [w.upper() for w in words[:5000]] + ["'" + w for w in words[:5000]] + [w + "'s" for w in words[:5000]]
    got = T.stem_batch(words)
    want = [port.stem(w).decode("utf-8") for w in words]
    bad = [(w, g, x) for w, g, x in zip(words, got, want) if g != x]
    assert not bad, bad[:10]
    # malformed input comes back unchanged (stemmer.cpp:393)
    raw = [b"ab\xffcd", b"\xc3", b"runn\xe2\x82ing"]
    assert T.stem_batch(raw) == [port.stem(r) for r in raw]


@pytest.mark.parametrize("lc,stop,stem", CONFIGS)
def test_corpus_vs_oracle(cuda_ok, port, lc, stop, stem):
    words = make_words(6000, seed=12, unicode_frac=0.08)
    text, off = make_corpus(4000, words, seed=8, malformed_frac=0.02, case_frac=0.3)
    a = gpu_tokenize(text, off, lc, stop, stem)
    b = port.tokenize_corpus(text, off, lc, stop, stem)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])
    assert a[2] == b[2]


def test_incremental_and_query(cuda_ok, port):
    """Two build calls share one vocabulary (ids continue in first-encounter order); query
    mode drops out-of-vocabulary tokens."""
    words = make_words(3000, seed=41)
    t1, o1 = make_corpus(700, words[:2000], seed=1)
    t2, o2 = make_corpus(500, words, seed=2)
    v = T.Vocabulary()
    g1 = gpu_tokenize(t1, o1, 1, 1, 1, v)
    g2 = gpu_tokenize(t2, o2, 1, 1, 1, v)
    ov = port.vocab_new()
    want1 = [port.tokenize(ov, t1[o1[d]:o1[d + 1]], True, 1, 1, 1) for d in range(len(o1) - 1)]
    want2 = [port.tokenize(ov, t2[o2[d]:o2[d + 1]], True, 1, 1, 1) for d in range(len(o2) - 1)]
    assert [g1[1][g1[0][d]:g1[0][d + 1]].tolist() for d in range(len(o1) - 1)] == want1
    assert [g2[1][g2[0][d]:g2[0][d + 1]].tolist() for d in range(len(o2) - 1)] == want2
    assert v.tokens() == port.vocab_tokens(ov)
    # query mode against the frozen vocabulary
    words_q = words + make_words(500, seed=99)  # some unseen words
    tq, oq = make_corpus(300, words_q, seed=5, mean_words=6)
    qb = T.tokenize_query((tq, oq), cfg_of(1, 1, 1), v)
    lists = qb.lists()
    assert len(v.tokens()) == len(port.vocab_tokens(ov))  # frozen
    for d in range(len(oq) - 1):
        assert lists[d] == port.tokenize(ov, tq[oq[d]:oq[d + 1]], False, 1, 1, 1)
    port.vocab_free(ov)


def test_edges(cuda_ok, port):
    long_word = "Internationalizations" * 5  # > 64 bytes: the global-scratch path
    docs = [b"", b"a", b"  ..  ", b"ab", long_word.encode(), ("Ü" * 40 + "ing").encode(), b"caf\xc3",
            b"\xa9abc d\xc3\xa9f", b"the and of", b"x" * 200, "Ǆ" * 70, b"\xf0\x9f", b"\x98\x80 ok"]
    docs = [d.encode() if isinstance(d, str) else d for d in docs]
    off = np.zeros(len(docs) + 1, np.uint64)
    off[1:] = np.cumsum([len(d) for d in docs])
    text = b"".join(docs)
    for lc, stop, stem in CONFIGS:
        a = gpu_tokenize(text, off, lc, stop, stem)
        b = port.tokenize_corpus(text, off, lc, stop, stem)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], (lc, stop, stem)
    # no documents / no tokens at all
    v = T.Vocabulary()
    b = T.tokenize_build([], cfg_of(1, 0, 0), v)
    assert b.num_docs == 0 and b.num_tokens == 0
    b = T.tokenize_build(["", "!", "a b"], cfg_of(1, 0, 0), v)
    assert b.lists() == [[], [], []] and v.size() == 0


def test_split_and_spec_examples(cuda_ok):
    assert T.split_text("Hello, World! a_b x") == ["hello", "world", "a_b"]
    assert T.split_text("Hello World", lowercase=False) == ["Hello", "World"]
    # SPEC.md:65-67
    cfg = T.TokenizerConfig(True, frozenset({"the", "is"}), T.StemmerKind.snowball_english)
    v = T.Vocabulary()
    ids = T.tokenize_build(["the cat is running"], cfg, v).lists()[0]
    assert [v.token(i) for i in ids] == ["cat", "run"]
    ids = T.tokenize_build(["cat cat"], T.TokenizerConfig(), v).lists()[0]
    assert ids[0] == ids[1]
    assert T.tokenize_query(["zebra"], T.TokenizerConfig(), v).lists() == [[]]
    assert T.StemmerKind.from_string("snowball-english") == T.StemmerKind.snowball_english
    with pytest.raises(ValueError, match="unknown stemmer"):
        T.StemmerKind.from_string("porter")


def test_text_index_retrieval_vs_oracle(cuda_ok, port, tmp_path):
    """SPEC build_index(corpus texts) + retrieve(text): GPU tokenization + index + top-k
    against the oracle tokenizer feeding the oracle index."""
    words = make_words(5000, seed=77)
    text, off = make_corpus(3000, words, seed=6, mean_words=40)
    corpus = [(f"d{d}", text[off[d]:off[d + 1]].decode("utf-8")) for d in range(len(off) - 1)]
    cfg = T.TokenizerConfig.english()
    p = BM25Params.for_variant(Variant.bm25plus)
    ti = T.build_text_index(corpus, p, cfg)
    toff, tids, toks = port.tokenize_corpus(text, off, 1, 1, 1)
    assert ti.vocab.tokens() == toks
    oi = oracle.OracleIndex(toff, tids, len(toks), int(p.variant), p.k1, p.b, p.delta)
    exp = oi.export()
    g = ti.index.export()
    for key in ("indptr", "docids", "df", "doclens"):
        assert np.array_equal(g[key], exp[key]), key
    qtext, qoff = make_corpus(200, words + ["unseenword"], seed=9, mean_words=5)
    queries = [qtext[qoff[q]:qoff[q + 1]].decode("utf-8") for q in range(len(qoff) - 1)]
    res = T.retrieve_text_batch(ti, queries, 10)
    ov = port.vocab_new()
    port.tokenize_corpus(text, off, 1, 1, 1, vocab=ov)
    qlists = [port.tokenize(ov, q, False, 1, 1, 1) for q in queries]
    port.vocab_free(ov)
    qo = np.zeros(len(qlists) + 1, np.uint64)
    qo[1:] = np.cumsum([len(q) for q in qlists])
    qt = np.array([t for q in qlists for t in q] or [0], np.uint32)
    rid, rsc = oi.retrieve_batch(qo, qt, 10)
    gid = np.stack([r.doc_indices for r in res])
    gsc = np.stack([r.scores for r in res])
    assert_topk_match(gid, gsc, rid, rsc, 10, len(corpus), lambda b: oi.score_query(qlists[b]),
                      lambda b: query_scale(exp, qlists[b]), "text")
    # save / load roundtrip answers identically
    ti.save(str(tmp_path / "ix"))
    with open(tmp_path / "ix" / "vocab.json", encoding="utf-8") as f:
        assert json.load(f) == {t: i for i, t in enumerate(toks)}
    tl = T.load_text_index(str(tmp_path / "ix"))
    assert tl.doc_ids == [c[0] for c in corpus] and tl.vocab.tokens() == toks
    res2 = T.retrieve_text_batch(tl, queries, 10)
    for a, b in zip(res, res2):
        assert np.array_equal(a.doc_indices, b.doc_indices) and np.array_equal(a.scores, b.scores)
        assert a.external_ids == b.external_ids == [corpus[int(d)][0] for d in a.doc_indices]
    with open(tmp_path / "ix" / "meta.json", encoding="utf-8") as f:
        meta = json.load(f)
    assert meta["tokenizer"] == {"lowercase": True, "stopwords_hash": T.stopwords_hash(cfg.stopwords),
                                 "stemmer": "snowball-english"}
    assert tl.config.stopwords == cfg.stopwords and tl.config.stemmer == cfg.stemmer


def test_text_index_external_ids_json_roundtrip(cuda_ok, tmp_path):
    """External ids with quotes, backslashes, control characters and non-ASCII survive save/load
    (docs.json is parsed as JSON, not by counting quote characters); int ids become strings."""
    corpus = [('a "quoted" id', "cat sat"), ("back\\slash\ttab", "dog ran"), ("ünï/€", "cat cat cat"), (7, "dog dog")]
    ti = T.build_text_index(corpus, BM25Params(), T.TokenizerConfig())
    assert ti.doc_ids == [str(c[0]) for c in corpus]
    ti.save(str(tmp_path / "ix"))
    with open(tmp_path / "ix" / "docs.json", encoding="utf-8") as f:
        assert json.load(f) == [str(c[0]) for c in corpus]
    tl = T.load_text_index(str(tmp_path / "ix"))
    assert tl.doc_ids == ti.doc_ids
    r = T.retrieve_text(tl, "cat", 2)
    assert r.external_ids == ["ünï/€", 'a "quoted" id']
    # a stopword list that no longer matches meta.json's hash is refused
    meta = json.load(open(tmp_path / "ix" / "meta.json", encoding="utf-8"))
    meta["stopwords"] = ["the"]
    json.dump(meta, open(tmp_path / "ix" / "meta.json", "w", encoding="utf-8"))
    with pytest.raises(RuntimeError, match="stopwords_hash"):
        T.load_text_index(str(tmp_path / "ix"))


def test_text_index_errors(cuda_ok):
    with pytest.raises(ValueError, match="empty corpus"):
        T.build_text_index([])
    with pytest.raises(ValueError, match="duplicate external ids"):
        T.build_text_index([("a", "x y"), ("a", "z w")])
    with pytest.raises(ValueError, match="degenerate corpus"):
        T.build_text_index([("a", "the"), ("b", "! ?")])
    import ctypes as C
    from paper_2407_03618_b200 import _lib
    v = T.Vocabulary()
    bad = _lib.TokenizerConfig(1, 7, None, 0)
    h = C.c_void_p()
    off = np.array([0, 2], np.uint64)
    with pytest.raises(SparselexError, match="unknown stemmer"):
        _lib.check(_lib.lib().sl_tokenize(v.handle, C.byref(bad), 1, b"ab", off.ctypes.data, 1, 0, C.byref(h)))
    off = np.array([1, 2], np.uint64)
    with pytest.raises(ValueError, match="doc_offsets"):
        T.tokenize_build((b"ab", off), T.TokenizerConfig(), v)


def test_device_input_unaligned(cuda_ok, port):
    """Device-resident text (zero-copy): 16-byte aligned input takes the 16-byte SWAR classifier,
    4-byte aligned the 4-byte one, odd addresses the byte-wise classifier; all identical."""
    import torch
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE
    words = make_words(2000, seed=61, unicode_frac=0.1)
    text, off = make_corpus(500, words, seed=3, malformed_frac=0.02)
    want = port.tokenize_corpus(text, off, 1, 1, 1)
    for shift in (0, 1, 3, 4, 8):
        buf = torch.zeros(len(text) + 16, dtype=torch.uint8, device="cuda")
        buf[shift:shift + len(text)] = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
        doff = torch.from_numpy(off.view(np.int64)).cuda()
        v = T.Vocabulary()
        b = T._tokenize_raw(buf.data_ptr() + shift, doff.data_ptr(), len(off) - 1, cfg_of(1, 1, 1), v, True,
                            SL_MEM_DEVICE)
        got_off, got_ids = b.to_numpy()
        assert np.array_equal(got_off, want[0]) and np.array_equal(got_ids, want[1]) and v.tokens() == want[2], shift


def test_many_distinct_strings_table_growth(cuda_ok):
    """More distinct raw strings than the raw table's first size (grows and retries); ids in
    first-encounter order against a plain dict reference (lowercase ASCII, no stop/stem)."""
    rng = np.random.default_rng(17)
    n = 1_500_000
    letters = np.frombuffer(b"abcdefghijklmnopqrstuvwxyz", np.uint8)
    lens = rng.integers(3, 9, n)
    chars = letters[rng.integers(0, 26, int(lens.sum()))]
    words, p = [], 0
    for L in lens:
        words.append(chars[p:p + L].tobytes())
        p += L
    words += words[: n // 3]  # repeats
    text = b" ".join(words)
    ref_ids, seen = [], {}
    for w in words:
        ref_ids.append(seen.setdefault(w, len(seen)))
    v = T.Vocabulary()
    off = np.array([0, len(text)], np.uint64)
    b = T.tokenize_build((text, off), T.TokenizerConfig(), v)
    _, ids = b.to_numpy()
    assert len(seen) > 1_000_000 and v.size() == len(seen)
    assert np.array_equal(ids, np.array(ref_ids, np.uint32))


def test_all_ascii_bytes_classifier(cuda_ok, port):
    """Every ASCII byte value (controls, punctuation, digits, both cases, '_', DEL) in random
    documents: the SWAR fast path of the 16-byte classifier against the oracle port."""
    import torch
    from paper_2407_03618_b200._lib import SL_MEM_DEVICE
    rng = np.random.default_rng(29)
    alphabet = np.arange(1, 128, dtype=np.uint8)
    weights = np.where((alphabet >= ord("a")) & (alphabet <= ord("z")), 8.0, 1.0)
    weights /= weights.sum()
    lens = rng.integers(0, 400, 600)
    off = np.zeros(len(lens) + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    text = rng.choice(alphabet, int(off[-1]), p=weights).astype(np.uint8).tobytes()
    for cfg in ((1, 1, 1), (0, 0, 0)):
        want = port.tokenize_corpus(text, off, *cfg)
        buf = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
        assert buf.data_ptr() % 16 == 0
        doff = torch.from_numpy(off.view(np.int64)).cuda()
        v = T.Vocabulary()
        b = T._tokenize_raw(buf.data_ptr(), doff.data_ptr(), len(off) - 1, cfg_of(*cfg), v, True, SL_MEM_DEVICE)
        got_off, got_ids = b.to_numpy()
        assert np.array_equal(got_off, want[0]) and np.array_equal(got_ids, want[1]) and v.tokens() == want[2], cfg


@pytest.mark.parametrize("chunk", [1 << 10, 1 << 14, 64 << 20])
def test_stream_tokenize_matches_single_call(cuda_ok, port, chunk):
    """sl_tokenize_stream (document-aligned chunks, overlapped copies) gives exactly the
    single-call result: ids, token offsets and vocabulary order, build and query; chunks smaller
    than some documents, empty documents, a document longer than a chunk."""
    words = make_words(3000, seed=71, unicode_frac=0.05)
    text, off = make_corpus(1500, words, seed=9, malformed_frac=0.01, case_frac=0.2)
    # an empty document and one long document
    text = text + " ".join(words[:900]).encode("utf-8")
    off = np.concatenate([off, [off[-1], len(text)]]).astype(np.uint64)
    cfg = cfg_of(1, 1, 1)
    want = port.tokenize_corpus(text, off, 1, 1, 1)
    v = T.Vocabulary()
    got_off, got_ids = T.tokenize_build_stream(text, off, cfg, v, chunk_bytes=chunk)
    assert np.array_equal(got_off, want[0]) and np.array_equal(got_ids, want[1]) and v.tokens() == want[2]
    # query mode against the single call on the frozen vocabulary
    b = T.tokenize_query((text, off), cfg, v)
    qo, qi = b.to_numpy()
    so, si = T.tokenize_query_stream(text, off, cfg, v, chunk_bytes=chunk)
    assert np.array_equal(so, qo) and np.array_equal(si, qi)
    # capacity too small fails loudly
    with pytest.raises(ValueError, match="ids_capacity"):
        T.tokenize_query_stream(text, off, cfg, v, chunk_bytes=chunk, out_ids=np.empty(3, np.uint32))


@pytest.mark.parametrize("lc,stop,stem", [(True, True, True), (False, False, False)])
def test_identity_is_bytes_under_forced_collisions(cuda_ok, port, monkeypatch, lc, stop, stem):
    """Vocabulary identity is byte equality (vocabulary.hpp:26-33), not a hash: with
    SL_TEXT_WEAK_HASH=1 every raw string of one length collides in the raw-string table, every
    new normalised string of one length collides in the dedup table and all vocabulary first
    hashes fall into 4 values. Byte verification reseeds the tables / keeps probing, and the
    ids, offsets and vocabulary stay identical to the oracle (incremental builds and query mode
    included)."""
    monkeypatch.setenv("SL_TEXT_WEAK_HASH", "1")
    words = make_words(3000, seed=12, unicode_frac=0.08)
    t1, o1 = make_corpus(1500, words[:2000], seed=8, malformed_frac=0.02, case_frac=0.3)
    t2, o2 = make_corpus(800, words, seed=9, case_frac=0.3)
    v = T.Vocabulary()
    g1 = gpu_tokenize(t1, o1, lc, stop, stem, v)
    g2 = gpu_tokenize(t2, o2, lc, stop, stem, v)
    ov = port.vocab_new()
    w1 = port.tokenize_corpus(t1, o1, lc, stop, stem, vocab=ov)
    w2 = port.tokenize_corpus(t2, o2, lc, stop, stem, vocab=ov)
    for g, w in ((g1, w1), (g2, w2)):
        assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1])
    assert v.tokens() == port.vocab_tokens(ov)
    tq, oq = make_corpus(200, words + make_words(300, seed=98), seed=5, mean_words=6)
    lists = T.tokenize_query((tq, oq), cfg_of(lc, stop, stem), v).lists()
    for d in range(len(oq) - 1):
        assert lists[d] == port.tokenize(ov, tq[oq[d]:oq[d + 1]], False, lc, stop, stem)
    port.vocab_free(ov)
