"""Golden fixture for the host-side formats around the path (lexicon.py),
produced by the REFERENCE (otflm) in the build container:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_lexicon.py

Writes tests/golden/lexicon.json: a synthetic corpus (synth.zipfian_corpus,
synth.py:20-32, plus rare words so min_count folding happens), the reference
build_vocabulary result (vocab.py:107-139) at min_count 1 and 2, KN models of
order 2 and 3 (train_ngram, ngram.py:66) written by save_arpa (ngram.py:212-239)
-- the file text itself -- and the tables load_arpa (ngram.py:242-306) reads
back, perplexity (ngram.py:188-203) on held-out sentences, leaf_path
(huffman.py:107-111) for a few words, and load_arpa of a hand-written
whitespace-separated ARPA with placeholders and -99 entries.
"""
import json, math, os, sys, tempfile
sys.path.insert(0, "/root/reference/pkg/src")
from otflm import synth, vocab as V, ngram as N, huffman as Hf  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "lexicon.json")


def enc(d):
    """dict of tuple -> float as sorted [[ids...], value] with -inf spelled out."""
    return [[list(k), ("-inf" if v == -math.inf else v)] for k, v in sorted(d.items())]


def main():
    corpus = synth.zipfian_corpus(240, 60, seed=11) + ["rare1 w1 w2", "w3 rare2 rare3 w4", ""]
    held = synth.zipfian_corpus(40, 60, seed=12) + ["w1 unseen w2"]
    out = {"corpus": corpus, "held": held, "vocab": {}, "models": {}}
    for mc in (1, 2):
        vb = V.build_vocabulary(corpus, min_count=mc)
        out["vocab"][str(mc)] = {"words": vb.words, "counts": vb.counts}
    vb = V.build_vocabulary(corpus, min_count=2)
    tree = Hf.build_huffman(vb)
    out["leaf_paths"] = {str(w): [list(p) for p in Hf.leaf_path(tree, w)] for w in (0, 1, 2, 5, vb.size - 1)}
    sents = V.read_sentences(held, vb)
    out["held_ids"] = sents
    with tempfile.TemporaryDirectory() as td:
        for order in (2, 3):
            m = N.train_ngram(corpus, vb, order)
            p = os.path.join(td, f"m{order}.arpa")
            N.save_arpa(m, vb, p)
            text = open(p, encoding="utf-8").read()
            back = N.load_arpa(p, vb)
            out["models"][str(order)] = {
                "arpa": text, "probs": enc(back.probs), "backoffs": enc(back.backoffs),
                "perplexity": N.perplexity(back, sents),
                "roundtrip_exact": back.probs == m.probs and back.backoffs == m.backoffs}
        hand = ("junk before\n\\data\\\nngram 1=4\nngram 2=2\n\n\\1-grams:\n-1.5 <unk>\n-99 <s> -0.25\n"
                "-0.5 </s>\n-0.75 w1 -0.125\n\n\\2-grams:\n-0.3 <s> w1\n-99 w1 </s>\n\\end\\\n")
        p = os.path.join(td, "hand.arpa")
        open(p, "w", encoding="utf-8").write(hand)
        h = N.load_arpa(p, vb)
        out["hand"] = {"arpa": hand, "order": h.order, "probs": enc(h.probs), "backoffs": enc(h.backoffs)}
    json.dump(out, open(OUT, "w"), indent=0)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
