"""Word lattices (input graph of the hot path) -- host side.

Mirrors the reference's ``Arc``/``Lattice`` (``lattice.py:37-127``) but keeps
arcs as flat arrays, which is what the device consumes: arcs are uploaded as
CSR records once per utterance batch and never walked on the host.  The
``arcs`` / ``out_arcs`` / ``topo_order`` / ``times`` views exist so the
object is a drop-in for reference code and tests.

``generate_lattice`` builds the same *kind* of synthetic sausage lattice as
the reference generator (``lattice.py:130-183``: reference word plus
``breadth - 1`` confusable alternatives per position, nodes expanded on the
small-LM context so arc LM scores are exact for every path) with a
vectorised sampler; it is an input builder, not part of the parity surface.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Sequence

import numpy as np

from .model import ngram_logprob


class LatticeFormatError(ValueError):
    """Malformed lattice text; message carries the line number."""


@dataclass(frozen=True)
class Arc:
    id: int
    src: int
    dst: int
    word: int
    acoustic: float
    smalllm: float


class Lattice:
    """Acyclic word graph with arcs stored as arrays in arc-id order.

    Node ids are arbitrary non-negative ints; ``n_nodes`` counts distinct
    ids.  Device compilation remaps them monotonically onto 0..n-1, which
    preserves the reference's Kahn smallest-id-first topological order and
    the sorted-finals tie-break.
    """

    def __init__(self, start: int, finals, arcs=None, *, src=None, dst=None, word=None,
                 acoustic=None, smalllm=None):
        self.start = int(start)
        self.finals = set(int(f) for f in finals)
        if arcs is not None:
            arcs = sorted(arcs, key=lambda a: a.id)
            src = [a.src for a in arcs]
            dst = [a.dst for a in arcs]
            word = [a.word for a in arcs]
            acoustic = [a.acoustic for a in arcs]
            smalllm = [a.smalllm for a in arcs]
        self.arc_src = np.ascontiguousarray(src, dtype=np.int64)
        self.arc_dst = np.ascontiguousarray(dst, dtype=np.int64)
        self.arc_word = np.ascontiguousarray(word, dtype=np.int32)
        self.arc_acoustic = np.ascontiguousarray(acoustic, dtype=np.float64)
        self.arc_smalllm = np.ascontiguousarray(smalllm, dtype=np.float64)
        nodes = np.unique(np.concatenate([self.arc_src, self.arc_dst,
                                          np.array([self.start] + sorted(self.finals),
                                                   dtype=np.int64)]))
        self.node_ids = nodes
        self.n_nodes = int(len(nodes))
        self._arcs = None
        self._topo = None

    @property
    def n_arcs(self) -> int:
        return int(len(self.arc_src))

    # --- reference-compatible views (lattice.py:47-86) -------------------
    @property
    def arcs(self) -> list:
        if self._arcs is None:
            self._arcs = [Arc(i, int(s), int(d), int(w), float(a), float(l)) for i, (s, d, w, a, l)
                          in enumerate(zip(self.arc_src, self.arc_dst, self.arc_word,
                                           self.arc_acoustic, self.arc_smalllm))]
        return self._arcs

    @property
    def out_arcs(self) -> dict:
        out = {int(n): [] for n in self.node_ids}
        for a in self.arcs:
            out[a.src].append(a)
        return out

    def _kahn(self):
        if self._topo is None:
            import heapq
            indeg = {int(n): 0 for n in self.node_ids}
            out = self.out_arcs
            for d in self.arc_dst:
                indeg[int(d)] += 1
            ready = [n for n, d in indeg.items() if d == 0]
            heapq.heapify(ready)
            times = {n: 0 for n in ready}
            order = []
            while ready:
                n = heapq.heappop(ready)
                order.append(n)
                for a in out[n]:
                    t = times[n] + 1
                    if times.get(a.dst, -1) < t:
                        times[a.dst] = t
                    indeg[a.dst] -= 1
                    if indeg[a.dst] == 0:
                        heapq.heappush(ready, a.dst)
            if len(order) != self.n_nodes:
                raise LatticeFormatError("lattice contains a cycle")
            self._topo = (order, times)
        return self._topo

    @property
    def topo_order(self) -> list:
        return self._kahn()[0]

    @property
    def times(self) -> dict:
        return self._kahn()[1]

    # --- text format (lattice.py:88-127, docs/protocol.md:84-94) ---------
    def save(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(f"start {self.start}\n")
            for s, d, w, a, l in zip(self.arc_src, self.arc_dst, self.arc_word,
                                     self.arc_acoustic, self.arc_smalllm):
                fh.write(f"{int(s)} {int(d)} {int(w)} {float(a)!r} {float(l)!r}\n")
            fh.write("final " + " ".join(str(n) for n in sorted(self.finals)) + "\n")

    @classmethod
    def load(cls, path) -> "Lattice":
        start = None
        finals: set = set()
        cols = ([], [], [], [], [])
        with open(path, encoding="utf-8") as fh:
            for lineno, line in enumerate(fh, 1):
                parts = line.split()
                if not parts or parts[0].startswith("#"):
                    continue
                try:
                    if parts[0] == "start":
                        start = int(parts[1])
                    elif parts[0] == "final":
                        finals.update(int(p) for p in parts[1:])
                    else:
                        if len(parts) != 5:
                            raise ValueError("expected 5 fields")
                        vals = (int(parts[0]), int(parts[1]), int(parts[2]),
                                float(parts[3]), float(parts[4]))
                        for c, v in zip(cols, vals):
                            c.append(v)
                except (ValueError, IndexError) as exc:
                    raise LatticeFormatError(f"{path}:{lineno}: {exc}") from exc
        if start is None:
            raise LatticeFormatError(f"{path}: missing start line")
        if not finals:
            raise LatticeFormatError(f"{path}: missing final line")
        lat = cls(start, finals, src=cols[0], dst=cols[1], word=cols[2], acoustic=cols[3],
                  smalllm=cols[4])
        try:
            lat._kahn()
        except LatticeFormatError as exc:
            raise LatticeFormatError(f"{path}: {exc}") from exc
        return lat

    @classmethod
    def from_reference(cls, lat) -> "Lattice":
        """Wrap a reference ``otflm.lattice.Lattice`` (or any object with
        ``start``, ``finals``, ``arcs``)."""
        return cls(lat.start, lat.finals, arcs=list(lat.arcs))


def as_lattice(lat) -> Lattice:
    return lat if isinstance(lat, Lattice) else Lattice.from_reference(lat)


# --------------------------------------------------------------------------
# synthetic generator
# --------------------------------------------------------------------------

class _BigramIndex:
    """Vectorised ngram_logprob for order <= 2 models (host input builder)."""

    def __init__(self, lm):
        self.lm = lm
        V = lm.vocab_size
        self.V = V
        uni = np.full(V, np.nan)
        for (k, v) in lm.probs.items():
            if len(k) == 1:
                uni[k[0]] = v
        self.uni = uni
        bo = np.zeros(V)
        for (k, v) in lm.backoffs.items():
            if len(k) == 1:
                bo[k[0]] = v
        self.bo = bo
        keys, vals = [], []
        for (k, v) in lm.probs.items():
            if len(k) == 2:
                keys.append(k[0] * V + k[1])
                vals.append(v)
        order = np.argsort(np.array(keys, dtype=np.int64)) if keys else np.zeros(0, np.int64)
        self.bkeys = np.array(keys, dtype=np.int64)[order] if keys else np.zeros(0, np.int64)
        self.bvals = np.array(vals, dtype=np.float64)[order] if keys else np.zeros(0)

    def __call__(self, h: np.ndarray, w: np.ndarray) -> np.ndarray:
        if self.lm.order == 1:
            out = self.uni[w]
        else:
            q = h.astype(np.int64) * self.V + w.astype(np.int64)
            pos = np.searchsorted(self.bkeys, q)
            pos = np.minimum(pos, max(len(self.bkeys) - 1, 0))
            found = (len(self.bkeys) > 0) & (self.bkeys[pos] == q) if len(self.bkeys) else \
                np.zeros(len(q), bool)
            out = np.where(found, self.bvals[pos] if len(self.bkeys) else 0.0,
                           self.bo[h] + self.uni[w])
        if np.isnan(out).any():
            raise KeyError("word missing from unigram table")
        return out


def generate_lattice(reference: Sequence[int], vocab_size: int, small_lm, confusion_breadth: int,
                     noise_seed: int, specials: Sequence[int] = (0, 1, 2),
                     bos: int = 1, index: _BigramIndex | None = None) -> Lattice:
    """Sausage lattice around *reference* (structure of reference
    lattice.py:130-183).  Alternatives are distinct non-special words other
    than the reference word; acoustic penalties -|N(1, 0.5)|, reference arcs 0.
    Nodes are keyed on (position, last small_lm.order-1 words), ids assigned
    in first-seen order, arcs frontier-major / candidate-minor."""
    reference = [int(w) for w in reference]
    if not reference:
        raise ValueError("reference must be non-empty")
    if confusion_breadth < 1:
        raise ValueError("confusion_breadth must be >= 1")
    rng = np.random.Generator(np.random.PCG64(noise_seed))
    T = len(reference)
    special = np.zeros(vocab_size, bool)
    special[list(specials)] = True
    n_pool = vocab_size - int(special.sum())
    b = confusion_breadth
    cand = np.zeros((T, b), dtype=np.int64)
    cac = np.zeros((T, b), dtype=np.float64)
    cand[:, 0] = reference
    pool = np.nonzero(~special)[0]
    n_alt = min(b - 1, n_pool - 1)
    for t in range(T):
        # the reference's draw (lattice.py:147-156): rng.choice over the pool
        # without the reference word, then one N(1, 0.5) per chosen word --
        # the same generator calls on index arithmetic instead of an O(V)
        # list per position, so the lattices are byte-identical to the
        # reference's generate_lattice for the same seed
        p_ref = int(np.searchsorted(pool, reference[t]))
        in_pool = p_ref < len(pool) and int(pool[p_ref]) == reference[t]
        n_alts = len(pool) - (1 if in_pool else 0)
        k_alt = min(b - 1, n_alts)
        if k_alt:
            i = rng.choice(n_alts, size=k_alt, replace=False)
            if in_pool:
                i = i + (i >= p_ref)
            cand[t, 1:1 + k_alt] = pool[i]
            cac[t, 1:1 + k_alt] = -np.abs(rng.normal(1.0, 0.5, size=k_alt))
    bb = 1 + n_alt
    cand, cac = cand[:, :bb], cac[:, :bb]
    k = max(small_lm.order - 1, 0)
    if k <= 1:
        idx = index or _BigramIndex(small_lm)
        src, dst, word, ac, hist_w = [], [], [], [], []
        frontier = [bos]  # last word of each frontier node (k==1) / dummy (k==0)
        node_base = 0
        next_base = 1
        for t in range(T):
            nf = len(frontier)
            srcs = np.repeat(node_base + np.arange(nf), bb)
            if k == 1:
                dsts = next_base + np.tile(np.arange(bb), nf)
                new_frontier = list(cand[t])
            else:
                dsts = np.full(nf * bb, next_base)
                new_frontier = [0]
            src.append(srcs)
            dst.append(dsts)
            word.append(np.tile(cand[t], nf))
            ac.append(np.tile(cac[t], nf))
            hist_w.append(np.repeat(np.array(frontier), bb))
            node_base = next_base
            next_base += len(new_frontier)
            frontier = new_frontier
        src = np.concatenate(src)
        dst = np.concatenate(dst)
        word = np.concatenate(word)
        ac = np.concatenate(ac)
        hw = np.concatenate(hist_w)
        slm = idx(hw, word) if k == 1 else idx(np.zeros_like(word), word)
        finals = list(range(node_base, next_base))
        return Lattice(0, finals, src=src, dst=dst, word=word, acoustic=ac, smalllm=slm)
    # general small-LM order: dictionary expansion (slow path)
    start_hist = (bos,) * k
    node_ids = {(0, start_hist): 0}
    frontier = [start_hist]
    cols = ([], [], [], [], [])
    for pos in range(T):
        nxt_frontier: dict = {}
        for hist in frontier:
            s = node_ids[(pos, hist)]
            for w, a in zip(cand[pos], cac[pos]):
                w = int(w)
                slm = ngram_logprob(small_lm, hist, w)
                nxt = (hist + (w,))[-k:]
                key = (pos + 1, nxt)
                if key not in node_ids:
                    node_ids[key] = len(node_ids)
                for c, v in zip(cols, (s, node_ids[key], w, float(a), slm)):
                    c.append(v)
                nxt_frontier[nxt] = None
        frontier = list(nxt_frontier)
    finals = {node_ids[(T, h)] for h in frontier}
    return Lattice(0, finals, src=cols[0], dst=cols[1], word=cols[2], acoustic=cols[3],
                   smalllm=cols[4])
