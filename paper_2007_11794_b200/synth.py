"""Seeded synthetic inputs for the BASELINE.json configs.

Everything is deterministic for fixed seeds and built with numpy only (the
GPU box has no reference package).  The recurrent model follows the
reference's own benchmark fixture (``benchmarks/kernel_speed.py:29-38`` on
``RnnlmModel.new`` = ``rnnlm.py:104-124``), so the same weights come out
bit-for-bit (checked against ``tests/golden/decode_a.npz``).

Configs
-------
a  V=1,000   H=64   MaxEnt 2^20  1 utterance  x 300 frames, breadth 3, beam 8
b  V=20,000  H=256  MaxEnt 2^21  64 utterances x 300 frames, breadth 3, beam 8
c  V=65,536  H=512  MaxEnt 2^22  beam sweep {1..64} on 8 utterances
d  V=65,536  H=512  1,048,576 isolated (history, word) queries
e  V=65,536  H=512  4,096 utterances x 300 frames (sharded over GPUs)
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lattice import Lattice, _BigramIndex, generate_lattice
from .model import HuffmanTree, NgramModel, RnnlmModel, build_huffman_from_counts

CONFIGS = {
    "a": dict(V=1000, H=64, bits=20, n_utt=1, T=300, breadth=3, beam=8),
    "b": dict(V=20000, H=256, bits=21, n_utt=64, T=300, breadth=3, beam=8),
    # SURVEY.md §8d config (b) "fat variant": breadth 16, beam 64
    "b_fat": dict(V=20000, H=256, bits=21, n_utt=64, T=300, breadth=16, beam=64),
    "c": dict(V=65536, H=512, bits=22, n_utt=8, T=300, breadth=3, beam=8),
    "d": dict(V=65536, H=512, bits=22, n_queries=1 << 20, n_ctx=1 << 18),
    "e": dict(V=65536, H=512, bits=22, n_utt=4096, T=300, breadth=3, beam=8),
}


def zipf_counts(V: int) -> np.ndarray:
    r = np.arange(1, V + 1, dtype=np.float64)
    return np.maximum(1, np.floor(1e7 / r ** 1.05)).astype(np.int64)


def synth_model(V: int, H: int, bits: int) -> RnnlmModel:
    """RnnlmModel.new(V, H, 3, bits, seed=2) + RandomState(3) output layer."""
    m = RnnlmModel.new(V, hidden_size=H, maxent_order=3, maxent_table_bits=bits, seed=2)
    rng = np.random.RandomState(3)
    m.node_vectors[:] = rng.uniform(-0.3, 0.3, m.node_vectors.shape).astype(np.float32)
    m.maxent_table[:] = rng.uniform(-0.1, 0.1, m.maxent_size).astype(np.float32)
    return m


def synth_bigram(V: int, seed: int = 1, per_ctx: int = 8, bos: int = 1, eos: int = 2) -> NgramModel:
    """Back-off bigram with a Zipf unigram and ``per_ctx`` explicit
    successors per context word (values drawn, not trained: a stand-in for
    the KN bigram of the reference recipe, with the same table shapes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    r = np.arange(1, V + 1, dtype=np.float64)
    p = 1.0 / r ** 1.05
    p /= p.sum()
    uni = np.log(p)
    probs = {(w,): float(uni[w]) for w in range(V)}
    ctx = np.arange(V)
    succ = rng.choice(V, size=(V, per_ctx), p=p)
    vals = np.log(rng.uniform(0.02, 0.6, size=(V, per_ctx)))
    keys = ctx[:, None] * V + succ
    flat_k, first = np.unique(keys.ravel(), return_index=True)
    flat_v = vals.ravel()[first]
    for k, v in zip(flat_k.tolist(), flat_v.tolist()):
        probs[(k // V, k % V)] = v
    bo = np.log(rng.uniform(0.05, 0.9, size=V))
    backoffs = {(w,): float(bo[w]) for w in range(V)}
    return NgramModel(order=2, vocab_size=V, bos_id=bos, eos_id=eos, probs=probs,
                      backoffs=backoffs)


def reference_sentences(V: int, n: int, T: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    r = np.arange(1, V - 2, dtype=np.float64)
    p = 1.0 / r ** 1.05
    p /= p.sum()
    return rng.choice(V - 3, size=(n, T), p=p) + 3


@dataclass
class Setup:
    name: str
    model: RnnlmModel
    tree: HuffmanTree
    small_lm: NgramModel
    lattices: list
    beam: int
    breadth: int


def build_setup(name: str, n_utt: int | None = None, T: int | None = None,
                seed: int = 7) -> Setup:
    cfg = dict(CONFIGS[name])
    if n_utt is not None:
        cfg["n_utt"] = n_utt
    if T is not None:
        cfg["T"] = T
    V, H, bits = cfg["V"], cfg["H"], cfg["bits"]
    model = synth_model(V, H, bits)
    tree = build_huffman_from_counts(zipf_counts(V))
    lm = synth_bigram(V)
    index = _BigramIndex(lm)
    refs = reference_sentences(V, cfg["n_utt"], cfg["T"], seed)
    lats = [generate_lattice(refs[i], V, lm, cfg["breadth"], noise_seed=seed * 100003 + i,
                             index=index) for i in range(cfg["n_utt"])]
    return Setup(name, model, tree, lm, lats, cfg["beam"], cfg["breadth"])


def more_lattices(setup: Setup, n_utt: int, T: int, seed: int) -> list:
    """Another batch of lattices over the same model / small LM."""
    V = setup.model.vocab_size
    index = _BigramIndex(setup.small_lm)
    refs = reference_sentences(V, n_utt, T, seed)
    return [generate_lattice(refs[i], V, setup.small_lm, setup.breadth, noise_seed=seed * 100003 + i,
                             index=index) for i in range(n_utt)]


def lattices_for_ids(setup: Setup, ids, T: int, seed_base: int = 1000) -> list:
    """One lattice per utterance id, a function of the id alone (so any
    sharding of the ids over ranks sees the same utterances)."""
    V = setup.model.vocab_size
    index = _BigramIndex(setup.small_lm)
    out = []
    for u in ids:
        ref = reference_sentences(V, 1, T, seed_base + int(u))[0]
        out.append(generate_lattice(ref, V, setup.small_lm, setup.breadth,
                                    noise_seed=(seed_base + int(u)) * 100003, index=index))
    return out


def query_set(model: RnnlmModel, n_queries: int, n_ctx: int, seed_w: int = 4, seed_c: int = 5):
    """Config (d): words ~ Zipf(1.05) over V, distinct contexts with
    h ~ U(0.001, 0.999) and 3-word histories ~ U[0, V)."""
    V, H, order = model.vocab_size, model.hidden_size, model.maxent_order
    rw = np.random.Generator(np.random.PCG64(seed_w))
    r = np.arange(1, V + 1, dtype=np.float64)
    p = 1.0 / r ** 1.05
    p /= p.sum()
    words = rw.choice(V, size=n_queries, p=p).astype(np.int32)
    rc = np.random.Generator(np.random.PCG64(seed_c))
    hidden = rc.uniform(0.001, 0.999, size=(n_ctx, H)).astype(np.float32)
    hist = rc.integers(0, V, size=(n_ctx, order)).astype(np.int32)
    hlen = np.full(n_ctx, order, dtype=np.int32)
    ctx_of_query = rw.integers(0, n_ctx, size=n_queries).astype(np.int32)
    return words, hidden, hist, hlen, ctx_of_query
