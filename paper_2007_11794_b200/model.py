"""Host-side model containers mirroring the reference's L1 types.

These are plain numpy holders handed to the device once (``DeviceModel``);
nothing here computes on the hot path.  Field names and validation follow
the reference so its own objects can be passed interchangeably:

* ``RnnlmModel`` / ``RnnlmContext``  -- reference ``rnnlm.py:51-132``
* ``HuffmanTree`` / ``build_huffman_from_counts`` -- ``huffman.py:20-104``
* ``NgramModel`` / ``ngram_logprob`` -- ``ngram.py:34-46``, ``:161-179``
"""

from __future__ import annotations

import heapq
import math
import struct
from dataclasses import dataclass, field
from pathlib import Path
from typing import Sequence

import numpy as np

# RNLM file (docs/protocol.md:55-69): 4-byte magic, a little-endian header
# (version, H, V, MaxEnt order, MaxEnt size, hash seed), then the four f32
# weight blocks in field order.
MODEL_MAGIC = b"RNLM"
MODEL_VERSION = 1
_HEADER = np.dtype([("magic", "S4"), ("version", "<u4"), ("H", "<u4"), ("V", "<u4"),
                    ("order", "<u4"), ("M", "<u8"), ("seed", "<u8")])
_WEIGHTS = ("input_weights", "recurrent_weights", "node_vectors", "maxent_table")


@dataclass(eq=False)
class RnnlmContext:
    """Immutable scoring context (reference rnnlm.py:51-66): the f32 hidden
    state and the word history (most recent last)."""

    hidden: np.ndarray
    history: tuple

    def __post_init__(self) -> None:
        h = np.array(self.hidden, dtype=np.float32, copy=True)
        h.setflags(write=False)
        self.hidden = h
        self.history = tuple(map(int, self.history))


def _weight_shapes(H: int, V: int, M: int) -> dict:
    return {"input_weights": (V, H), "recurrent_weights": (H, H),
            "node_vectors": (V - 1, H), "maxent_table": (M,)}


@dataclass(eq=False)
class RnnlmModel:
    """The HS + MaxEnt RNNLM's weights (the reference's rnnlm.py:69-124
    field schema, so reference and repo objects are interchangeable).  Host
    holder only: DeviceModel uploads it once; the validation raises
    ValueError like the reference does."""

    hidden_size: int
    vocab_size: int
    maxent_order: int
    maxent_size: int
    hash_seed: int
    input_weights: np.ndarray
    recurrent_weights: np.ndarray
    node_vectors: np.ndarray
    maxent_table: np.ndarray

    def __post_init__(self) -> None:
        M = int(self.maxent_size)
        problems = [msg for bad, msg in (
            (M < 1 or (M & (M - 1)) != 0, f"maxent_size must be a positive power of two (got {M})"),
            (self.maxent_order < 1, f"maxent_order must be positive (got {self.maxent_order})"),
            (self.vocab_size < 2, f"vocab_size must be at least 2 (got {self.vocab_size})"),
        ) if bad]
        if problems:
            raise ValueError("; ".join(problems))
        for name, shape in _weight_shapes(self.hidden_size, self.vocab_size, M).items():
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.float32)
            if arr.shape != shape:
                raise ValueError(f"{name}: shape {arr.shape} does not match {shape}")
            if not np.isfinite(arr).all():
                raise ValueError(f"{name}: non-finite weight")
            setattr(self, name, arr)

    @classmethod
    def new(cls, vocab_size: int, hidden_size: int = 100, maxent_order: int = 3,
            maxent_table_bits: int = 20, seed: int = 1,
            hash_seed: int = 0x5DEECE66D) -> "RnnlmModel":
        """Fresh model with the reference's initial distribution
        (rnnlm.py:104-124): U then W ~ U(-0.1, 0.1) from one PCG64 stream,
        zero output layer -- the same draws, so the same weights."""
        rng = np.random.Generator(np.random.PCG64(seed))
        V, H, M = vocab_size, hidden_size, 1 << maxent_table_bits
        draws = [rng.uniform(-0.1, 0.1, shape).astype(np.float32) for shape in ((V, H), (H, H))]
        return cls(hidden_size=H, vocab_size=V, maxent_order=maxent_order, maxent_size=M,
                   hash_seed=hash_seed, input_weights=draws[0], recurrent_weights=draws[1],
                   node_vectors=np.zeros((V - 1, H), np.float32), maxent_table=np.zeros(M, np.float32))

    @property
    def hash_mask(self) -> np.uint64:
        return np.uint64(self.maxent_size - 1)

    def zero_context(self) -> RnnlmContext:
        return RnnlmContext(np.zeros(self.hidden_size, np.float32), ())

    def save(self, path) -> None:
        """RNLM file: structured header + the weight blocks, written in place."""
        hdr = np.array([(MODEL_MAGIC, MODEL_VERSION, self.hidden_size, self.vocab_size,
                         self.maxent_order, self.maxent_size, self.hash_seed)], dtype=_HEADER)
        with open(path, "wb") as fh:
            hdr.tofile(fh)
            for name in _WEIGHTS:
                getattr(self, name).astype("<f4", copy=False).tofile(fh)

    @classmethod
    def load(cls, path) -> "RnnlmModel":
        """RNLM file through one memory map: the header is parsed as a
        structured record and the weight blocks are views at their offsets
        (copied once, when the model validates them)."""
        raw = np.memmap(path, dtype=np.uint8, mode="r")
        if raw.size < _HEADER.itemsize:
            raise ValueError(f"{path}: shorter than the RNLM header")
        hdr = raw[:_HEADER.itemsize].view(_HEADER)[0]
        if bytes(hdr["magic"]) != MODEL_MAGIC:
            raise ValueError(f"{path}: not an RNLM file (magic {bytes(hdr['magic'])!r})")
        if int(hdr["version"]) != MODEL_VERSION:
            raise ValueError(f"{path}: RNLM version {int(hdr['version'])} is not supported")
        H, V, M = int(hdr["H"]), int(hdr["V"]), int(hdr["M"])
        shapes = _weight_shapes(H, V, M)
        sizes = [int(np.prod(shapes[n])) * 4 for n in _WEIGHTS]
        if raw.size < _HEADER.itemsize + sum(sizes):
            raise ValueError(f"{path}: weight blocks truncated")
        offs = _HEADER.itemsize + np.concatenate([[0], np.cumsum(sizes)[:-1]])
        blocks = {n: raw[o:o + sz].view("<f4").reshape(shapes[n])
                  for n, o, sz in zip(_WEIGHTS, offs, sizes)}
        return cls(hidden_size=H, vocab_size=V, maxent_order=int(hdr["order"]), maxent_size=M,
                   hash_seed=int(hdr["seed"]), **blocks)


# --------------------------------------------------------------------------
# Huffman tree (reference huffman.py)
# --------------------------------------------------------------------------

@dataclass
class HuffmanTree:
    """Flat CSR of root-to-leaf paths (reference huffman.py:20-51).

    ``path_nodes`` int32 internal-node ids (root = n_words - 2),
    ``path_signs`` float32 (+1 for branch bit 0, -1 for bit 1),
    ``path_offsets`` int64 [n_words + 1].
    """

    n_words: int
    children: np.ndarray  # [n_words - 1, 2] child refs (< n_words = leaf)
    path_nodes: np.ndarray = field(repr=False, default=None)
    path_signs: np.ndarray = field(repr=False, default=None)
    path_offsets: np.ndarray = field(repr=False, default=None)

    @property
    def n_internal(self) -> int:
        return self.n_words - 1

    @property
    def root(self) -> int:
        return self.n_words - 2

    @property
    def leaf_paths(self):
        out = []
        for w in range(self.n_words):
            o0, o1 = self.path_offsets[w], self.path_offsets[w + 1]
            out.append([(int(n), 0 if s > 0 else 1)
                        for n, s in zip(self.path_nodes[o0:o1], self.path_signs[o0:o1])])
        return out

    def code_length(self, word_id: int) -> int:
        return int(self.path_offsets[word_id + 1] - self.path_offsets[word_id])

    def weighted_length(self, counts) -> int:
        return int(sum(int(c) * self.code_length(w) for w, c in enumerate(counts)))


def build_huffman_from_counts(counts) -> HuffmanTree:
    """Deterministic greedy merge (reference huffman.py:74-104).

    Heap entries (weight, tiebreak, ref) with tiebreak = word id for leaves
    and n + j for the j-th merge; branch bit 0 is the first node popped.
    Paths are read off parent pointers instead of the reference's DFS, which
    yields the same root-to-leaf sequences.
    """
    counts = [int(c) for c in counts]
    n = len(counts)
    if n < 2:
        raise ValueError(f"need at least 2 words to build a tree, got {n}")
    heap = [(c, w, w) for w, c in enumerate(counts)]
    heapq.heapify(heap)
    children = np.zeros((n - 1, 2), dtype=np.int64)
    parent = np.full(2 * n - 1, -1, dtype=np.int64)
    bit = np.zeros(2 * n - 1, dtype=np.int8)
    for j in range(n - 1):
        w0, _, left = heapq.heappop(heap)
        w1, _, right = heapq.heappop(heap)
        children[j] = (left, right)
        parent[left], bit[left] = n + j, 0
        parent[right], bit[right] = n + j, 1
        heapq.heappush(heap, (w0 + w1, n + j, n + j))
    # depth of every leaf by walking parents (vectorised over leaves)
    depth = np.zeros(n, dtype=np.int64)
    cur = np.arange(n, dtype=np.int64)
    active = parent[cur] >= 0
    while active.any():
        depth[active] += 1
        cur = np.where(active, parent[cur], cur)
        active = parent[cur] >= 0
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(depth, out=offsets[1:])
    nodes = np.zeros(int(offsets[-1]), dtype=np.int32)
    signs = np.zeros(int(offsets[-1]), dtype=np.float32)
    # fill from the leaf end backwards: position offsets[w] + depth - 1 - k
    cur = np.arange(n, dtype=np.int64)
    k = np.zeros(n, dtype=np.int64)
    active = parent[cur] >= 0
    while active.any():
        idx = np.nonzero(active)[0]
        par = parent[cur[idx]]
        pos = offsets[idx] + depth[idx] - 1 - k[idx]
        nodes[pos] = (par - n).astype(np.int32)
        signs[pos] = np.where(bit[cur[idx]] == 0, 1.0, -1.0).astype(np.float32)
        cur[idx] = par
        k[idx] += 1
        active = parent[cur] >= 0
    return HuffmanTree(n_words=n, children=children, path_nodes=nodes, path_signs=signs,
                       path_offsets=offsets)


def build_huffman(vocab) -> HuffmanTree:
    return build_huffman_from_counts(vocab.counts)


# --------------------------------------------------------------------------
# Back-off n-gram LM (reference ngram.py)
# --------------------------------------------------------------------------

@dataclass
class NgramModel:
    """ARPA-style tables keyed by word tuples (reference ngram.py:34-46)."""

    order: int
    vocab_size: int
    bos_id: int
    eos_id: int
    probs: dict = field(default_factory=dict)
    backoffs: dict = field(default_factory=dict)

    def logprob(self, context: Sequence[int], w: int) -> float:
        return ngram_logprob(self, context, w)


def ngram_logprob(model, context: Sequence[int], w: int) -> float:
    """ln P(w | context) of a back-off LM (the reference's ngram.py:161-179
    semantics): the longest stored n-gram ending in w over the last
    order - 1 context words, plus the back-off weights (0 when absent) of the
    longer contexts that did not match, added from the shortest one outward
    -- the reference's float64 evaluation order.  Host helper (lattice arc
    scores, tests); the decoder's lookups run on the device (decode.cuh)."""
    w = int(w)
    if w < 0 or w >= model.vocab_size:
        raise ValueError(f"word id {w} outside the vocabulary [0, {model.vocab_size})")
    keep = max(int(model.order) - 1, 0)
    hist = tuple(int(x) for x in context)[-keep:] if keep else ()
    # depth d = number of leading history words dropped before the match
    matched = next((d for d in range(len(hist) + 1) if hist[d:] + (w,) in model.probs), None)
    if matched is None:
        raise KeyError(f"word {w} missing from unigram table")
    lp = model.probs[hist[matched:] + (w,)]
    for d in range(matched - 1, -1, -1):
        lp = model.backoffs.get(hist[d:], 0.0) + lp
    return lp


def ngram_from_arrays(order, V, bos, eos, pk, pl, pv, bk, bl, bv) -> NgramModel:
    """Rebuild dict tables from flat (keys, lens, vals) arrays."""
    probs = {tuple(int(x) for x in pk[i, :pl[i]]): float(pv[i]) for i in range(len(pl))}
    bows = {tuple(int(x) for x in bk[i, :bl[i]]): float(bv[i]) for i in range(len(bl))}
    return NgramModel(order=int(order), vocab_size=int(V), bos_id=int(bos), eos_id=int(eos),
                      probs=probs, backoffs=bows)


def ngram_flat(model):
    """Flatten probs/backoffs to padded int32 keys + lens + float64 values."""
    order = int(model.order)
    width = max(order, 1)

    def flat(d):
        n = len(d)
        keys = np.zeros((max(n, 1), width), dtype=np.int32)
        lens = np.zeros(max(n, 1), dtype=np.int32)
        vals = np.zeros(max(n, 1), dtype=np.float64)
        if n:
            ks = list(d.keys())
            lens[:n] = [len(k) for k in ks]
            for L in set(lens[:n].tolist()):
                sel = np.nonzero(lens[:n] == L)[0]
                if L:
                    keys[sel, :L] = np.array([ks[i] for i in sel], dtype=np.int32).reshape(-1, L)
            vals[:n] = np.fromiter(d.values(), dtype=np.float64, count=n)
        return n, keys, lens, vals

    return order, flat(model.probs), flat(model.backoffs)


def log_half_path_unigram(tree: HuffmanTree, vocab_size: int, bos: int, eos: int) -> NgramModel:
    """Unigram whose values equal a zero-weight model's scores (the reference
    degenerate test, tests/test_decoder.py:61-89)."""
    lh = math.log(0.5)
    uni = NgramModel(order=1, vocab_size=vocab_size, bos_id=bos, eos_id=eos)
    for w in range(vocab_size):
        total = 0.0
        for _ in range(tree.code_length(w)):
            total += lh
        uni.probs[(w,)] = total
    return uni
