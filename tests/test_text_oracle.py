"""CPU: the text-pipeline oracle (oracle/text_oracle.cpp) against the reference's golden
fixtures and, where oracle/_ref was built, against the reference itself."""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.text import TextOracle, ref_available
from tests.text_words import make_corpus, make_words

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "text_golden.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN, encoding="utf-8") as f:
        return json.load(f)


@pytest.fixture(scope="module")
def port():
    return TextOracle("port")


def test_ac4_fixture(golden, port):
    """SPEC AC4: >= 30 strings x the Table 2 configurations (+ lowercase off)."""
    assert len(golden["ac4"]) >= 30
    for row in golden["ac4"]:
        text = bytes.fromhex(row["text_hex"])
        for (lc, stop, stem), want in zip(golden["configs"], row["tokens"]):
            v = port.vocab_new()
            ids = port.tokenize(v, text, True, lc, stop, stem)
            toks = port.vocab_tokens(v)
            port.vocab_free(v)
            assert [toks[i] for i in ids] == want, (text, lc, stop, stem)


def test_stems_golden(golden, port):
    for w, s in golden["stems"]:
        assert port.stem(w).decode("utf-8") == s, w


def test_unicode_tables_digest(golden, port):
    wc, lo = hashlib.sha256(), hashlib.sha256()
    for cp in range(0x110000):
        if 0xD800 <= cp <= 0xDFFF:
            continue
        if port.L.orc_is_word(cp):
            wc.update(cp.to_bytes(4, "little"))
            lo.update(cp.to_bytes(4, "little") + port.L.orc_to_lower(cp).to_bytes(4, "little"))
    assert wc.hexdigest() == golden["word_class_sha256"]
    assert lo.hexdigest() == golden["lower_sha256"]


def test_spec_examples(port):
    # SPEC.md:65-67 ("the cat is running", stopwords {the, is}, snowball) -> ["cat", "run"]
    v = port.vocab_new()
    ids = port.tokenize(v, "the cat is running", True, True, True, True)
    assert [port.vocab_tokens(v)[i] for i in ids] == ["cat", "run"]
    ids = port.tokenize(v, "cat cat", True, True, False, False)
    assert ids[0] == ids[1]
    assert port.tokenize(v, "zebra", False) == []
    port.vocab_free(v)


def test_first_encounter_ids(port):
    text, off = make_corpus(50, make_words(300, seed=5), seed=2)
    toff, ids, toks = port.tokenize_corpus(text, off, True, False, False)
    seen = -1
    for i in ids:  # every new id is exactly the next one
        if i > seen:
            assert i == seen + 1
            seen = i
    assert len(toks) == seen + 1


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (reference tree absent)")
def test_port_matches_reference_corpus(port):
    ref = TextOracle("ref")
    words = make_words(4000, seed=9, unicode_frac=0.1)
    text, off = make_corpus(1500, words, seed=4, malformed_frac=0.02, case_frac=0.3)
    for lc, stop, stem in [(1, 0, 0), (1, 1, 0), (1, 0, 1), (1, 1, 1), (0, 0, 1)]:
        a = port.tokenize_corpus(text, off, lc, stop, stem)
        b = ref.tokenize_corpus(text, off, lc, stop, stem)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], (lc, stop, stem)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (reference tree absent)")
def test_port_matches_reference_stems(port):
    ref = TextOracle("ref")
    for w in make_words(60000, seed=21, unicode_frac=0.1):
        for x in (w, w.lower(), "'" + w, w + "'s"):
            assert port.stem(x) == ref.stem(x), x
