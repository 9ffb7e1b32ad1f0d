"""Two-pass rescoring behind the reference's API.

* ``nbest``            -- decoder.py:180-230 (host search in libotflm_b200.so)
* ``rescore_twopass``  -- decoder.py:243-274 (device RNNLM scoring)
* ``nbest_batch`` / ``rescore_twopass_batch`` -- many utterances at once:
  the n-best searches run utterance-parallel on host threads, and all lists
  are scored by one device level loop over their merged prefix tries.

Same names, argument meaning and errors as the reference; ``precision``
selects the recurrent-update arithmetic ("fp64" = the reference's float64
accumulation; "tf32x3" / "bf16" = tcgen05 tensor cores).
"""

from __future__ import annotations

import ctypes as C
import weakref
from typing import Sequence

import numpy as np

from . import _lib
from .device import DeviceModel, DeviceNgram, _p, current_stream_ptr, pack_lattices
from .rescore import PathHypothesis

MODES = {"rnnlm": 0, "hybrid": 1}


class NbestArrays:
    """n-best lists of a lattice batch as flat arrays (hypothesis order =
    search order within each utterance)."""

    def __init__(self, lats, n_hyp, hyp_len, arcs, scores, arc_word, arc_off):
        self.lats = lats
        self.n_hyp = n_hyp                        # [U]
        self.list_off = np.zeros(len(n_hyp) + 1, np.int64)
        self.list_off[1:] = np.cumsum(n_hyp)
        self.hyp_len = hyp_len                    # [n_hyp total]
        self.hyp_off = np.zeros(len(hyp_len) + 1, np.int64)
        self.hyp_off[1:] = np.cumsum(hyp_len)
        self.arcs = arcs                          # lattice-local arc ids
        self.scores = scores                      # [n, 3] combined, acoustic, lm
        # words of every hypothesis, gathered through the batch arc table
        utt_of_arc = np.repeat(np.repeat(np.arange(len(n_hyp)), n_hyp), hyp_len)
        self.words = np.ascontiguousarray(arc_word[arc_off[utt_of_arc] + arcs], np.int32)

    def hypothesis(self, u: int, k: int) -> PathHypothesis:
        j = int(self.list_off[u]) + int(k)
        a0, a1 = int(self.hyp_off[j]), int(self.hyp_off[j + 1])
        return PathHypothesis(tuple(self.arcs[a0:a1].tolist()), tuple(self.words[a0:a1].tolist()),
                              float(self.scores[j, 1]), float(self.scores[j, 2]),
                              float(self.scores[j, 0]))

    def hypotheses(self, u: int) -> list:
        return [self.hypothesis(u, k) for k in range(int(self.n_hyp[u]))]


def nbest_arrays(lattices: Sequence, n: int, lm_weight: float = 1.0, n_threads: int = 0) -> NbestArrays:
    """nbest (decoder.py:180-230) for every lattice, utterance-parallel on
    host threads, returned as flat arrays."""
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    L = _lib.load()
    batch, arrays, lats = pack_lattices(lattices)
    h = C.c_void_p()
    _lib.check(L.otflm_nbest_create(C.byref(batch), n, float(lm_weight), int(n_threads), C.byref(h)),
               "nbest")
    try:
        U = len(lats)
        n_hyp = np.zeros(U, np.int32)
        tot = np.zeros(2, np.int64)
        _lib.check(L.otflm_nbest_sizes(h, _p(n_hyp), _p(tot)), "nbest")
        hl = np.zeros(max(int(tot[0]), 1), np.int32)
        arcs = np.zeros(max(int(tot[1]), 1), np.int32)
        sc = np.zeros((max(int(tot[0]), 1), 3))
        status = np.zeros(U, np.int32)
        _lib.check(L.otflm_nbest_copy(h, _p(hl), _p(arcs), _p(sc), _p(status)), "nbest")
    finally:
        L.otflm_nbest_destroy(h)
    for u in range(U):
        if status[u] == _lib.ERR_NO_PATH:
            raise ValueError("no complete path through the lattice")
        _lib.check(int(status[u]), f"nbest (utterance {u})")
    H, A = int(tot[0]), int(tot[1])
    return NbestArrays(lats, n_hyp, hl[:H], arcs[:A], sc[:H], arrays["arc_word"], arrays["arc_off"])


def nbest_batch(lattices: Sequence, n: int, lm_weight: float = 1.0, n_threads: int = 0):
    """nbest for every lattice; returns one list of PathHypothesis per lattice."""
    r = nbest_arrays(lattices, n, lm_weight, n_threads)
    return [r.hypotheses(u) for u in range(len(r.lats))]


def nbest(lattice, n: int, lm_weight: float = 1.0) -> list:
    """decoder.py:180-230: top-n distinct word sequences by first-pass score."""
    return nbest_batch([lattice], n, lm_weight, n_threads=1)[0]


class TwopassPlan:
    """Prefix tries of a batch of n-best lists, uploaded; reusable runs.

    ``hyp_lists``: lists of PathHypothesis, or an ``NbestArrays``."""

    def __init__(self, model, tree, small_lm, hyp_lists, n_threads: int = 0):
        L = _lib.load()
        self.dmodel = DeviceModel.get(model, tree)
        self.ngram = DeviceNgram.get(small_lm, self.dmodel) if small_lm is not None else None
        if isinstance(hyp_lists, NbestArrays):
            r = hyp_lists
            if len(r.n_hyp) == 0 or np.any(r.n_hyp == 0):
                raise ValueError("empty hypothesis list")
            self.lists = None
            self.nb = r
            self.list_off = r.list_off
            self.hyp_off = r.hyp_off
            self.words = r.words
            self.acoustic = np.ascontiguousarray(r.scores[:, 1])
        else:
            if not hyp_lists or any(len(l) == 0 for l in hyp_lists):
                raise ValueError("empty hypothesis list")
            self.nb = None
            self.lists = [list(l) for l in hyp_lists]
            counts = [len(l) for l in self.lists]
            self.list_off = np.zeros(len(counts) + 1, np.int64)
            self.list_off[1:] = np.cumsum(counts)
            flat = [h for l in self.lists for h in l]
            lens = np.array([len(h.words) for h in flat], np.int64)
            self.hyp_off = np.zeros(len(flat) + 1, np.int64)
            self.hyp_off[1:] = np.cumsum(lens)
            self.words = np.ascontiguousarray(
                np.fromiter((w for h in flat for w in h.words), np.int32, int(self.hyp_off[-1])))
            self.acoustic = np.ascontiguousarray([h.acoustic_score for h in flat], np.float64)
        if len(self.words) and (self.words.min() < 0 or self.words.max() >= model.vocab_size):
            raise ValueError("word id out of range")
        self.n_lists = len(self.list_off) - 1
        self.n_hyp = int(self.list_off[-1])
        self._batch = _lib.HypBatch(self.n_lists, _p(self.list_off), _p(self.hyp_off),
                                    _p(self.words), _p(self.acoustic))
        h = C.c_void_p()
        _lib.check(L.otflm_twopass_create(self.dmodel.handle,
                                          self.ngram.handle if self.ngram is not None else None,
                                          C.byref(self._batch), int(n_threads), C.byref(h),
                                          current_stream_ptr()), "rescore_twopass")
        self.handle = h
        self._fin = weakref.finalize(self, L.otflm_twopass_destroy, h)

    def info(self) -> dict:
        o = np.zeros(6, np.int64)
        _lib.check(_lib.load().otflm_twopass_info(self.handle, _p(o)), "twopass info")
        return dict(trie_nodes=int(o[0]), levels=int(o[1]), words=int(o[2]), updates=int(o[3]),
                    widest_level=int(o[4]), hypotheses=int(o[5]))

    def run(self, mode: str = "rnnlm", interp_weight: float = 0.5, lm_weight: float = 1.0,
            precision: str = "fp64", use_graph: bool = True) -> None:
        if mode not in MODES:
            raise ValueError(f"unknown two-pass mode {mode!r}")
        if mode == "hybrid" and self.ngram is None:
            raise ValueError("hybrid mode needs the small LM")
        _lib.check(_lib.load().otflm_twopass_run(self.handle, MODES[mode], float(interp_weight),
                                                 float(lm_weight), _lib.PREC[precision],
                                                 int(bool(use_graph)), current_stream_ptr()),
                   "rescore_twopass")

    def fetch(self):
        lm = np.zeros(self.n_hyp)
        comb = np.zeros(self.n_hyp)
        best = np.zeros(self.n_lists, np.int32)
        _lib.check(_lib.load().otflm_twopass_fetch(self.handle, _p(lm), _p(comb), _p(best),
                                                   current_stream_ptr()), "rescore_twopass")
        return lm, comb, best

    def results(self, lm_weight: float = 1.0):
        """The winning PathHypothesis of every list (decoder.py:264-274)."""
        lm, comb, best = self.fetch()
        out = []
        for l in range(self.n_lists):
            j = int(self.list_off[l]) + int(best[l])
            h = self.lists[l][int(best[l])] if self.lists is not None else \
                self.nb.hypothesis(l, int(best[l]))
            out.append(PathHypothesis(h.arcs, h.words, h.acoustic_score, float(lm[j]),
                                      float(comb[j])))
        return out


def rescore_twopass_batch(hyp_lists, mode: str, model, tree, small_lm, interp_weight: float = 0.5,
                          lm_weight: float = 1.0, precision: str = "fp64") -> list:
    """rescore_twopass for many n-best lists in one device pass."""
    if mode not in MODES:
        raise ValueError(f"unknown two-pass mode {mode!r}")
    plan = TwopassPlan(model, tree, small_lm if mode == "hybrid" else None, hyp_lists)
    plan.run(mode, interp_weight, lm_weight, precision, use_graph=False)
    return plan.results(lm_weight)


def rescore_twopass(hyps, mode: str, model, tree, small_lm, interp_weight: float = 0.5,
                    lm_weight: float = 1.0, precision: str = "fp64") -> PathHypothesis:
    """decoder.py:243-274: re-rank one n-best list with the RNNLM."""
    if mode not in MODES:
        raise ValueError(f"unknown two-pass mode {mode!r}")
    if not hyps:
        raise ValueError("empty hypothesis list")
    return rescore_twopass_batch([hyps], mode, model, tree, small_lm, interp_weight, lm_weight,
                                 precision)[0]
