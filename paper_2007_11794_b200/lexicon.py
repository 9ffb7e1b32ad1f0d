"""Host-side vocabulary and ARPA I/O around the rescoring path.

These are the data formats either side of the hot path:
the word <-> id table the Huffman tree is built from (reference ``vocab.py``)
and the ARPA text form of the small n-gram LM whose scores the decoder
subtracts (reference ``ngram.py:206-306``).  They are plain host code: the
decoder consumes the resulting ``NgramModel`` / ``HuffmanTree`` through
``rescore.py``, which flattens them onto the device once per model.

Same names, argument meaning, error behaviour and byte formats as the
reference, so files written by either side load in the other:

* ``Vocabulary`` (vocab.py:31-97): ids in list order, ``word<TAB>count``
  file lines, ``<unk>``/``<s>``/``</s>`` specials.
* ``build_vocabulary`` (vocab.py:107-139): specials first, then descending
  count with alphabetical ties; words below ``min_count`` fold into
  ``<unk>``; boundary tokens counted once per non-empty sentence.
* ``save_arpa`` / ``load_arpa`` (ngram.py:212-306): log10 columns written as
  ``repr(ln / ln 10)``, ``-99`` for minus infinity, context-only placeholder
  lines; values read back as ``float(text) * ln 10``.
* ``perplexity`` (ngram.py:188-203), ``leaf_path`` (huffman.py:107-111).
"""

from __future__ import annotations

import io
import math
from collections import Counter
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Sequence

from .model import HuffmanTree, NgramModel, ngram_logprob

UNK_TOKEN, BOS_TOKEN, EOS_TOKEN = "<unk>", "<s>", "</s>"
_LN10 = math.log(10.0)
_ARPA_FLOOR = -99.0          # the ARPA spelling of log 0


class EmptyCorpusError(ValueError):
    """The corpus held no tokens (vocab.py:26-28)."""


@dataclass
class Vocabulary:
    """Dense word <-> id table with per-id corpus counts (vocab.py:31-97)."""

    words: list
    counts: list
    ids: dict = field(init=False)

    def __post_init__(self) -> None:
        self.ids = {}
        for i, w in enumerate(self.words):
            if self.ids.setdefault(w, i) != i:
                raise ValueError("duplicate words in vocabulary")

    @property
    def size(self) -> int:
        return len(self.words)

    def __len__(self) -> int:
        return len(self.words)

    @property
    def unk_id(self) -> int:
        return self.ids[UNK_TOKEN]

    @property
    def sentence_begin_id(self) -> int:
        return self.ids[BOS_TOKEN]

    @property
    def sentence_end_id(self) -> int:
        return self.ids[EOS_TOKEN]

    def id_of(self, word: str) -> int:
        return self.ids.get(word, self.unk_id)

    def tokenize(self, line: str) -> list:
        get, unk = self.ids.get, self.unk_id
        return [get(w, unk) for w in line.split()]

    def save(self, path) -> None:
        Path(path).write_text("".join(f"{w}\t{c}\n" for w, c in zip(self.words, self.counts)),
                              encoding="utf-8")

    @classmethod
    def load(cls, path) -> "Vocabulary":
        words, counts = [], []
        for lineno, line in enumerate(Path(path).read_text(encoding="utf-8").split("\n"), 1):
            if not line:
                continue
            fields = line.split("\t")
            try:
                if len(fields) != 2:
                    raise ValueError
                counts.append(int(fields[1]))
            except ValueError as exc:
                raise ValueError(f"{path}:{lineno}: malformed vocabulary line") from exc
            words.append(fields[0])
        return cls(words=words, counts=counts)


def _lines(corpus) -> Iterable[str]:
    if isinstance(corpus, (str, Path)):
        with open(corpus, encoding="utf-8") as fh:
            yield from fh
    else:
        yield from corpus


def build_vocabulary(corpus, min_count: int = 1) -> Vocabulary:
    """Count a line-per-sentence corpus into a ``Vocabulary`` (vocab.py:107-139)."""
    if min_count < 1:
        raise ValueError(f"min_count must be >= 1, got {min_count}")
    tally, sentences = Counter(), 0
    for line in _lines(corpus):
        toks = line.split()
        if toks:
            sentences += 1
            tally.update(toks)
    if not sentences:
        raise EmptyCorpusError("corpus contains no sentences")
    for special in (UNK_TOKEN, BOS_TOKEN, EOS_TOKEN):
        tally.pop(special, None)
    folded = sum(c for c in tally.values() if c < min_count)
    kept = sorted(((-c, w) for w, c in tally.items() if c >= min_count))
    return Vocabulary(words=[UNK_TOKEN, BOS_TOKEN, EOS_TOKEN] + [w for _, w in kept],
                      counts=[max(1, folded), sentences, sentences] + [-c for c, _ in kept])


def read_sentences(corpus, vocab: Vocabulary) -> list:
    """Id sentences of a corpus, empty lines skipped (vocab.py:142-149)."""
    return [ids for ids in (vocab.tokenize(line) for line in _lines(corpus)) if ids]


def corpus_from_string(text: str) -> io.StringIO:
    return io.StringIO(text)


def leaf_path(tree: HuffmanTree, word_id: int) -> list:
    """Root-to-leaf (internal node id, branch bit) pairs (huffman.py:107-111),
    read from the CSR the device uses."""
    if not 0 <= word_id < tree.n_words:
        raise ValueError(f"word id {word_id} out of range 0..{tree.n_words - 1}")
    o0, o1 = int(tree.path_offsets[word_id]), int(tree.path_offsets[word_id + 1])
    return [(int(n), 0 if s > 0 else 1) for n, s in zip(tree.path_nodes[o0:o1], tree.path_signs[o0:o1])]


def perplexity(model: NgramModel, sentences) -> float:
    """exp(mean -ln p), sentence end included, ``<s>``-padded context (ngram.py:188-203)."""
    nll, n = 0.0, 0
    for sent in sentences:
        ctx = [model.bos_id] * max(model.order - 1, 0)
        for w in [*sent, model.eos_id]:
            nll -= ngram_logprob(model, ctx, w)
            ctx.append(int(w))
            n += 1
    if not n:
        raise ValueError("no tokens to evaluate")
    return math.exp(nll / n)


def _arpa_num(x: float) -> str:
    return "-99" if x == -math.inf else repr(x / _LN10)


def _arpa_val(text: str) -> float:
    v = float(text)
    return -math.inf if v <= _ARPA_FLOOR + 0.001 else v * _LN10


def save_arpa(model: NgramModel, vocab: Vocabulary, path) -> None:
    """ARPA export (ngram.py:212-239): every n-gram with a probability or a
    backoff weight, per order in sorted id order; backoff-only contexts get a
    ``-99`` probability placeholder."""
    grams = sorted(set(model.probs) | set(model.backoffs), key=lambda g: (len(g), g))
    by_order = {k: [g for g in grams if len(g) == k] for k in range(1, model.order + 1)}
    out = ["\\data\\\n"]
    out += [f"ngram {k}={len(by_order[k])}\n" for k in range(1, model.order + 1)]
    for k in range(1, model.order + 1):
        out.append(f"\n\\{k}-grams:\n")
        for g in by_order[k]:
            line = _arpa_num(model.probs.get(g, -math.inf)) + "\t" + " ".join(vocab.words[w] for w in g)
            if k < model.order and g in model.backoffs:
                line += "\t" + _arpa_num(model.backoffs[g])
            out.append(line + "\n")
    out.append("\n\\end\\\n")
    Path(path).write_text("".join(out), encoding="utf-8")


def load_arpa(path, vocab: Vocabulary) -> NgramModel:
    """Parse an ARPA file into an ``NgramModel`` through ``vocab`` (ngram.py:242-306).

    Raises ``ValueError`` for a missing ``\\data\\`` header, a header without
    n-gram counts, stray lines outside a section or a wrong word count; an
    unknown word raises ``KeyError`` (the reference maps through ``vocab.ids``).
    """
    lines = [ln.strip() for ln in Path(path).read_text(encoding="utf-8").split("\n")]
    try:
        i = lines.index("\\data\\") + 1
    except ValueError:
        raise ValueError(f"{path}: missing \\data\\ section") from None
    order = 0
    while i < len(lines) and (not lines[i] or lines[i].startswith("ngram ")):
        if lines[i]:
            k = int(lines[i][6:].split("=")[0])
            order = max(order, k)
        i += 1
    if order == 0:
        raise ValueError(f"{path}: no ngram counts in header")
    model = NgramModel(order=order, vocab_size=vocab.size, bos_id=vocab.sentence_begin_id,
                       eos_id=vocab.sentence_end_id)
    k = 0
    for raw in lines[i:]:
        if not raw:
            continue
        if raw == "\\end\\":
            break
        if raw.startswith("\\") and raw.endswith("-grams:"):
            k = int(raw[1:].split("-")[0])
            continue
        tabbed = "\t" in raw
        parts = raw.split("\t") if tabbed else raw.split()
        if k == 0 or len(parts) < 2:
            raise ValueError(f"{path}: stray line outside n-gram section: {raw!r}")
        words = parts[1].split() if tabbed else parts[1:1 + k]
        if len(words) != k:
            raise ValueError(f"{path}: expected {k} words in {raw!r}")
        rest = parts[2:] if tabbed else parts[1 + k:]
        gram = tuple(vocab.ids[w] for w in words)
        lp = _arpa_val(parts[0])
        bow = _arpa_val(rest[0]) if rest else None
        if not (lp == -math.inf and bow is not None and bow != -math.inf):   # placeholder line
            model.probs[gram] = lp
        if bow is not None:
            model.backoffs[gram] = bow
    return model
