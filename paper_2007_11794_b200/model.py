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

MODEL_MAGIC = b"RNLM"
MODEL_VERSION = 1


@dataclass(eq=False)
class RnnlmContext:
    """Immutable scoring context (reference rnnlm.py:51-66)."""

    hidden: np.ndarray
    history: tuple

    def __post_init__(self) -> None:
        self.hidden = np.ascontiguousarray(self.hidden, dtype=np.float32)
        self.hidden.flags.writeable = False
        self.history = tuple(int(w) for w in self.history)


@dataclass(eq=False)
class RnnlmModel:
    """Weights of the HS + MaxEnt RNNLM (reference rnnlm.py:69-124)."""

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
        if self.maxent_size & (self.maxent_size - 1) or self.maxent_size < 1:
            raise ValueError(f"maxent_size must be a power of two, got {self.maxent_size}")
        if self.maxent_order < 1:
            raise ValueError("maxent_order must be >= 1")
        if self.vocab_size < 2:
            raise ValueError("vocab_size must be >= 2")
        shapes = {
            "input_weights": (self.vocab_size, self.hidden_size),
            "recurrent_weights": (self.hidden_size, self.hidden_size),
            "node_vectors": (self.vocab_size - 1, self.hidden_size),
            "maxent_table": (self.maxent_size,),
        }
        for name, shape in shapes.items():
            arr = np.ascontiguousarray(getattr(self, name), dtype=np.float32)
            if arr.shape != shape:
                raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
            if not np.all(np.isfinite(arr)):
                raise ValueError(f"{name} contains non-finite values")
            setattr(self, name, arr)

    @classmethod
    def new(cls, vocab_size: int, hidden_size: int = 100, maxent_order: int = 3,
            maxent_table_bits: int = 20, seed: int = 1,
            hash_seed: int = 0x5DEECE66D) -> "RnnlmModel":
        """Same initial distribution as reference rnnlm.py:104-124 (PCG64)."""
        rng = np.random.Generator(np.random.PCG64(seed))
        H = hidden_size
        M = 1 << maxent_table_bits
        return cls(
            hidden_size=H, vocab_size=vocab_size, maxent_order=maxent_order,
            maxent_size=M, hash_seed=hash_seed,
            input_weights=rng.uniform(-0.1, 0.1, (vocab_size, H)).astype(np.float32),
            recurrent_weights=rng.uniform(-0.1, 0.1, (H, H)).astype(np.float32),
            node_vectors=np.zeros((vocab_size - 1, H), dtype=np.float32),
            maxent_table=np.zeros(M, dtype=np.float32),
        )

    @property
    def hash_mask(self) -> np.uint64:
        return np.uint64(self.maxent_size - 1)

    def zero_context(self) -> RnnlmContext:
        return RnnlmContext(np.zeros(self.hidden_size, dtype=np.float32), ())

    # RNLM file (docs/protocol.md:55-69; reference rnnlm.py:136-170)
    def save(self, path) -> None:
        header = MODEL_MAGIC + struct.pack("<IIIIQQ", MODEL_VERSION, self.hidden_size,
                                           self.vocab_size, self.maxent_order,
                                           self.maxent_size, self.hash_seed)
        with open(path, "wb") as fh:
            fh.write(header)
            for arr in (self.input_weights, self.recurrent_weights, self.node_vectors,
                        self.maxent_table):
                fh.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())

    @classmethod
    def load(cls, path) -> "RnnlmModel":
        with open(path, "rb") as fh:
            magic = fh.read(4)
            if magic != MODEL_MAGIC:
                raise ValueError(f"{path}: bad magic {magic!r}, expected {MODEL_MAGIC!r}")
            version, H, n, order, M, hash_seed = struct.unpack("<IIIIQQ", fh.read(32))
            if version != MODEL_VERSION:
                raise ValueError(f"{path}: unsupported model version {version}")

            def block(count, shape):
                raw = fh.read(4 * count)
                if len(raw) != 4 * count:
                    raise ValueError(f"{path}: truncated weight block")
                return np.frombuffer(raw, dtype="<f4").reshape(shape).astype(np.float32)

            return cls(hidden_size=H, vocab_size=n, maxent_order=order, maxent_size=M,
                       hash_seed=hash_seed, input_weights=block(n * H, (n, H)),
                       recurrent_weights=block(H * H, (H, H)),
                       node_vectors=block((n - 1) * H, (n - 1, H)),
                       maxent_table=block(M, (M,)))


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
    """Longest stored suffix match + backoffs (reference ngram.py:161-179).

    Host-side helper used when generating lattice arc scores; the decoder's
    per-request lookup runs on the device.
    """
    w = int(w)
    if not 0 <= w < model.vocab_size:
        raise ValueError(f"word id {w} out of range 0..{model.vocab_size - 1}")
    ctx = tuple(int(x) for x in context)
    ctx = ctx[-(model.order - 1):] if model.order > 1 else ()
    suffixes = [ctx[i:] for i in range(len(ctx) + 1)]
    for depth, c in enumerate(suffixes):
        lp = model.probs.get(c + (w,))
        if lp is not None:
            for shorter in reversed(suffixes[:depth]):
                lp = model.backoffs.get(shorter, 0.0) + lp
            return lp
    raise KeyError(f"word {w} missing from unigram table")


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
