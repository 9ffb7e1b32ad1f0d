"""Host formats around the path (lexicon.py) vs the reference's own outputs
(tests/golden/lexicon.json, made by tests/golden/make_golden_lexicon.py):
vocabulary construction (vocab.py:107-139), ARPA write/read
(ngram.py:212-306), perplexity (ngram.py:188-203), leaf_path
(huffman.py:107-111).  All comparisons are exact."""
import json
import math
from pathlib import Path

import pytest

from paper_2007_11794_b200 import build_huffman
from paper_2007_11794_b200.lexicon import (EmptyCorpusError, Vocabulary, build_vocabulary, leaf_path,
                                           load_arpa, perplexity, read_sentences, save_arpa)
from paper_2007_11794_b200.model import NgramModel

G = json.loads((Path(__file__).parent / "golden" / "lexicon.json").read_text())


def dec(pairs):
    return {tuple(k): (-math.inf if v == "-inf" else v) for k, v in pairs}


@pytest.mark.parametrize("mc", ["1", "2"])
def test_build_vocabulary_matches_reference(mc):
    vb = build_vocabulary(G["corpus"], min_count=int(mc))
    assert vb.words == G["vocab"][mc]["words"]
    assert vb.counts == G["vocab"][mc]["counts"]


def test_vocabulary_errors_and_roundtrip(tmp_path):
    with pytest.raises(EmptyCorpusError):
        build_vocabulary(["", "   "])
    with pytest.raises(ValueError):
        build_vocabulary(["a b"], min_count=0)
    with pytest.raises(ValueError):
        Vocabulary(words=["<unk>", "a", "a"], counts=[1, 1, 1])
    vb = build_vocabulary(G["corpus"], min_count=2)
    vb.save(tmp_path / "v.txt")
    back = Vocabulary.load(tmp_path / "v.txt")
    assert back.words == vb.words and back.counts == vb.counts
    (tmp_path / "bad.txt").write_text("<unk>\t1\nbroken line\n")
    with pytest.raises(ValueError, match="malformed"):
        Vocabulary.load(tmp_path / "bad.txt")
    assert vb.tokenize("w1 never-seen") == [vb.ids["w1"], vb.unk_id]


def test_leaf_path_matches_reference():
    vb = build_vocabulary(G["corpus"], min_count=2)
    tree = build_huffman(vb)
    for w, path in G["leaf_paths"].items():
        assert leaf_path(tree, int(w)) == [tuple(p) for p in path]
    with pytest.raises(ValueError):
        leaf_path(tree, vb.size)


@pytest.mark.parametrize("order", ["2", "3"])
def test_arpa_read_write_matches_reference(order, tmp_path):
    vb = build_vocabulary(G["corpus"], min_count=2)
    ref = G["models"][order]
    p = tmp_path / "ref.arpa"
    p.write_text(ref["arpa"], encoding="utf-8")
    m = load_arpa(p, vb)
    assert m.order == int(order)
    assert m.probs == dec(ref["probs"])                 # bit-exact floats
    assert m.backoffs == dec(ref["backoffs"])
    q = tmp_path / "ours.arpa"
    save_arpa(m, vb, q)                                 # what the reference wrote, byte for byte
    assert q.read_text(encoding="utf-8") == ref["arpa"]
    sents = read_sentences(G["held"], vb)
    assert sents == G["held_ids"]
    assert perplexity(m, sents) == ref["perplexity"]


def test_arpa_hand_written_whitespace_placeholders(tmp_path):
    vb = build_vocabulary(G["corpus"], min_count=2)
    p = tmp_path / "hand.arpa"
    p.write_text(G["hand"]["arpa"], encoding="utf-8")
    m = load_arpa(p, vb)
    assert m.order == G["hand"]["order"]
    assert m.probs == dec(G["hand"]["probs"])
    assert m.backoffs == dec(G["hand"]["backoffs"])


def test_arpa_errors(tmp_path):
    vb = build_vocabulary(G["corpus"], min_count=2)
    cases = {"nodata.arpa": "ngram 1=1\n", "nocounts.arpa": "\\data\\\n\n\\1-grams:\n-1 w1\n",
             "stray.arpa": "\\data\\\nngram 1=1\n-1 w1\n", "words.arpa": "\\data\\\nngram 2=1\n\\2-grams:\n-1\tw1\n"}
    for name, text in cases.items():
        (tmp_path / name).write_text(text)
        with pytest.raises(ValueError):
            load_arpa(tmp_path / name, vb)
    with pytest.raises(ValueError):
        perplexity(NgramModel(order=2, vocab_size=3, bos_id=1, eos_id=2), [])
