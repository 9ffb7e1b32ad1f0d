"""ctypes front-end of the CPU oracle (``oracle/otflm_oracle.c``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline leg and ``--impl reference``), never by the
product package ``paper_2007_11794_b200``.

Objects are duck-typed so that both the reference's own ``otflm`` types (in
this container) and the product package's host mirrors can be passed:

* model: ``hidden_size, vocab_size, maxent_order, maxent_size, hash_seed,
  input_weights, recurrent_weights, node_vectors, maxent_table``
  (reference ``rnnlm.py:69-124``);
* tree: ``path_nodes, path_signs, path_offsets`` (``huffman.py:40-51``);
* small LM: ``order, vocab_size, bos_id, probs, backoffs``
  (``ngram.py:34-46``);
* lattice: ``start, finals, arcs`` with ``Arc(id, src, dst, word, acoustic,
  smalllm)`` (``lattice.py:37-60``).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"

ERRORS = {
    -1: ValueError, -2: KeyError, -3: RuntimeError, -4: ValueError,
    -5: KeyError, -6: MemoryError, -7: ValueError, -8: OverflowError,
}
ERROR_NAMES = {
    -1: "ValueError", -2: "UnknownIndexError", -3: "TableFullError",
    -4: "no complete path through the lattice", -5: "word missing from unigram table",
    -6: "out of memory", -7: "lattice contains a cycle", -8: "PackOverflowError",
}


def build(force: bool = False) -> Path:
    """Compile liboracle.so with the committed Makefile (gcc only)."""
    src = _HERE / "otflm_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(_LIB_PATH))
        p = C.c_void_p
        i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double
        L.orc_feature_index.restype = u64
        L.orc_feature_index.argtypes = [u64, i64, p, i64, i64, u64]
        L.orc_word_logprob.restype = f64
        L.orc_word_logprob.argtypes = [p, i32, p, i64, p, p, i64, p, p, i32, u64, u64]
        L.orc_advance_hidden.restype = None
        L.orc_advance_hidden.argtypes = [p, p, p, i32, p]
        L.orc_all_word_logprobs.restype = None
        L.orc_all_word_logprobs.argtypes = [p, i32, p, i64, p, p, p, i32, p, p, i32, u64, u64, p]
        L.orc_ngram_create.restype = p
        L.orc_ngram_create.argtypes = [i32, i32, i32, i64, p, p, p, i64, p, p, p]
        L.orc_ngram_destroy.argtypes = [p]
        L.orc_ngram_logprob.restype = C.c_int
        L.orc_ngram_logprob.argtypes = [p, p, i32, i32, p]
        L.orc_stack_create.restype = p
        L.orc_stack_create.argtypes = [p, i32, u64]
        L.orc_stack_destroy.argtypes = [p]
        L.orc_stack_reset.argtypes = [p, i32]
        L.orc_stack_cache_clear.argtypes = [p]
        L.orc_stack_roll_stats.argtypes = [p]
        L.orc_stack_stats.argtypes = [p, p]
        L.orc_stack_context.restype = C.c_int
        L.orc_stack_context.argtypes = [p, u64, p, p, p]
        L.orc_rnnlm_prob.restype = C.c_int
        L.orc_rnnlm_prob.argtypes = [p, i32, u64, p, p, p]
        L.orc_serve_request.restype = C.c_int
        L.orc_serve_request.argtypes = [p, p, i32, u64, p, p]
        L.orc_rescore_onthefly.restype = C.c_int
        L.orc_rescore_onthefly.argtypes = [p, p, p, f64, i64, p]
        L.orc_path_score.restype = C.c_int
        L.orc_path_score.argtypes = [p, p, p, p, i32, f64, p]
        L.orc_decode_many.restype = C.c_int
        L.orc_decode_many.argtypes = [p, p, p, i32, f64, i64, i32, i32, p, p, p, p, p]
        L.orc_decode_many_t.restype = C.c_int
        L.orc_decode_many_t.argtypes = [p, p, p, i32, f64, i64, i32, i32, p, p, p, p, p, p]
        L.orc_query_batch.restype = None
        L.orc_query_batch.argtypes = [p, i64, p, p, p, p, p, p, i32]
        L.orc_stack_set_capacity.restype = C.c_int
        L.orc_stack_set_capacity.argtypes = [p, i64]
        L.orc_nbest.restype = C.c_int
        L.orc_nbest.argtypes = [p, i32, f64, p, p, p, i64, p, p]
        L.orc_twopass.restype = C.c_int
        L.orc_twopass.argtypes = [p, p, i32, p, p, p, i32, f64, f64, p, p, p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc: int, what: str = "") -> None:
    if rc != 0:
        raise ERRORS.get(rc, RuntimeError)(f"oracle {what}: {ERROR_NAMES.get(rc, rc)}")


# --------------------------------------------------------------------------
# kernels (reference _kernels_nb.py:21-104)
# --------------------------------------------------------------------------

def feature_index(seed, order_k, words, node_id, mask) -> int:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.int64))
    return int(lib().orc_feature_index(int(seed) & (2**64 - 1), int(order_k), _ptr(w),
                                       len(w), int(node_id), int(mask) & (2**64 - 1)))


def word_logprob(hidden, history, nodes, signs, node_vectors, maxent_table,
                 maxent_order, seed, mask) -> float:
    h = np.ascontiguousarray(hidden, dtype=np.float32)
    hist = np.ascontiguousarray(np.asarray(history, dtype=np.int64))
    nd = np.ascontiguousarray(nodes, dtype=np.int32)
    sg = np.ascontiguousarray(signs, dtype=np.float32)
    nv = np.ascontiguousarray(node_vectors, dtype=np.float32)
    me = np.ascontiguousarray(maxent_table, dtype=np.float32)
    return float(lib().orc_word_logprob(_ptr(h), h.shape[0], _ptr(hist), len(hist), _ptr(nd),
                                        _ptr(sg), len(nd), _ptr(nv), _ptr(me), int(maxent_order),
                                        int(seed), int(mask)))


def advance_hidden(input_row, recurrent, hidden) -> np.ndarray:
    u = np.ascontiguousarray(input_row, dtype=np.float32)
    W = np.ascontiguousarray(recurrent, dtype=np.float32)
    h = np.ascontiguousarray(hidden, dtype=np.float32)
    out = np.empty(W.shape[0], dtype=np.float32)
    lib().orc_advance_hidden(_ptr(u), _ptr(W), _ptr(h), W.shape[0], _ptr(out))
    return out


def all_word_logprobs(hidden, history, path_nodes, path_signs, path_offsets,
                      node_vectors, maxent_table, maxent_order, seed, mask) -> np.ndarray:
    h = np.ascontiguousarray(hidden, dtype=np.float32)
    hist = np.ascontiguousarray(np.asarray(history, dtype=np.int64))
    pn = np.ascontiguousarray(path_nodes, dtype=np.int32)
    ps = np.ascontiguousarray(path_signs, dtype=np.float32)
    po = np.ascontiguousarray(path_offsets, dtype=np.int64)
    nv = np.ascontiguousarray(node_vectors, dtype=np.float32)
    me = np.ascontiguousarray(maxent_table, dtype=np.float32)
    V = len(po) - 1
    out = np.empty(V, dtype=np.float64)
    lib().orc_all_word_logprobs(_ptr(h), h.shape[0], _ptr(hist), len(hist), _ptr(pn), _ptr(ps),
                                _ptr(po), V, _ptr(nv), _ptr(me), int(maxent_order), int(seed),
                                int(mask), _ptr(out))
    return out


# --------------------------------------------------------------------------
# model / n-gram / lattice marshalling
# --------------------------------------------------------------------------

class _OrcModel(C.Structure):
    _fields_ = [("H", C.c_int32), ("V", C.c_int32), ("order", C.c_int32),
                ("maxent_size", C.c_uint64), ("seed", C.c_uint64),
                ("U", C.c_void_p), ("W", C.c_void_p), ("NV", C.c_void_p), ("ME", C.c_void_p),
                ("path_nodes", C.c_void_p), ("path_signs", C.c_void_p),
                ("path_offsets", C.c_void_p)]


class OracleModel:
    """Keeps contiguous copies alive for the C struct."""

    def __init__(self, model, tree):
        self.model = model
        self.H = int(model.hidden_size)
        self.V = int(model.vocab_size)
        self.order = int(model.maxent_order)
        self.arrays = [
            np.ascontiguousarray(model.input_weights, dtype=np.float32),
            np.ascontiguousarray(model.recurrent_weights, dtype=np.float32),
            np.ascontiguousarray(model.node_vectors, dtype=np.float32),
            np.ascontiguousarray(model.maxent_table, dtype=np.float32),
            np.ascontiguousarray(tree.path_nodes, dtype=np.int32),
            np.ascontiguousarray(tree.path_signs, dtype=np.float32),
            np.ascontiguousarray(tree.path_offsets, dtype=np.int64),
        ]
        U, W, NV, ME, pn, ps, po = self.arrays
        self.struct = _OrcModel(self.H, self.V, self.order, int(model.maxent_size),
                                int(model.hash_seed), _ptr(U).value, _ptr(W).value,
                                _ptr(NV).value, _ptr(ME).value, _ptr(pn).value,
                                _ptr(ps).value, _ptr(po).value)

    @property
    def ref(self):
        return C.byref(self.struct)


def ngram_flat(ngram):
    """Flatten probs/backoffs dicts (ngram.py:34-46) to padded arrays."""
    order = int(ngram.order)
    width = max(order, 1)

    def flat(d):
        n = len(d)
        keys = np.zeros((max(n, 1), width), dtype=np.int32)
        lens = np.zeros(max(n, 1), dtype=np.int32)
        vals = np.zeros(max(n, 1), dtype=np.float64)
        for i, (k, v) in enumerate(d.items()):
            lens[i] = len(k)
            keys[i, :len(k)] = k
            vals[i] = v
        return n, keys, lens, vals

    return order, flat(ngram.probs), flat(ngram.backoffs)


class OracleNgram:
    def __init__(self, ngram):
        self.order = int(ngram.order)
        order, (n_p, kp, lp, vp), (n_b, kb, lb, vb) = ngram_flat(ngram)
        self._keep = (kp, lp, vp, kb, lb, vb)
        self.handle = lib().orc_ngram_create(order, int(ngram.vocab_size), int(ngram.bos_id),
                                             n_p, _ptr(kp), _ptr(lp), _ptr(vp),
                                             n_b, _ptr(kb), _ptr(lb), _ptr(vb))
        if not self.handle:
            raise ValueError("oracle: bad n-gram model")

    def logprob(self, context, w) -> float:
        ctx = np.ascontiguousarray(np.asarray(list(context), dtype=np.int32))
        out = np.zeros(1, dtype=np.float64)
        _check(lib().orc_ngram_logprob(self.handle, _ptr(ctx), len(ctx), int(w), _ptr(out)),
               "ngram_logprob")
        return float(out[0])

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.orc_ngram_destroy(self.handle)
            self.handle = None


class _OrcLattice(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_arcs", C.c_int32), ("start", C.c_int32),
                ("n_finals", C.c_int32), ("src", C.c_void_p), ("dst", C.c_void_p),
                ("word", C.c_void_p), ("ac", C.c_void_p), ("slm", C.c_void_p),
                ("finals", C.c_void_p)]


def lattice_arrays(lat):
    """Arc arrays in arc-id order with node ids remapped monotonically onto
    0..n-1 (preserves Kahn smallest-id order and sorted finals)."""
    if hasattr(lat, "arc_src"):  # product-package array lattice
        ids = np.asarray(lat.node_ids)
        rm = lambda x: np.searchsorted(ids, np.asarray(x, np.int64)).astype(np.int32)
        return (len(ids), int(rm([lat.start])[0]), rm(lat.arc_src), rm(lat.arc_dst),
                np.asarray(lat.arc_word, np.int32), np.asarray(lat.arc_acoustic, np.float64),
                np.asarray(lat.arc_smalllm, np.float64), rm(sorted(lat.finals)))
    arcs = sorted(lat.arcs, key=lambda a: a.id)
    nodes = sorted({lat.start} | set(lat.finals) | {a.src for a in arcs} | {a.dst for a in arcs})
    remap = {n: i for i, n in enumerate(nodes)}
    src = np.array([remap[a.src] for a in arcs], dtype=np.int32)
    dst = np.array([remap[a.dst] for a in arcs], dtype=np.int32)
    word = np.array([a.word for a in arcs], dtype=np.int32)
    ac = np.array([a.acoustic for a in arcs], dtype=np.float64)
    slm = np.array([a.smalllm for a in arcs], dtype=np.float64)
    finals = np.array(sorted(remap[f] for f in lat.finals), dtype=np.int32)
    return len(nodes), remap[lat.start], src, dst, word, ac, slm, finals


class OracleLattice:
    def __init__(self, lat):
        n_nodes, start, *arrs = lattice_arrays(lat)
        self.arrs = [np.ascontiguousarray(a) for a in arrs]
        src, dst, word, ac, slm, finals = self.arrs
        self.n_arcs = len(src)
        self.struct = _OrcLattice(n_nodes, len(src), start, len(finals), _ptr(src).value,
                                  _ptr(dst).value, _ptr(word).value, _ptr(ac).value,
                                  _ptr(slm).value, _ptr(finals).value)


class _OrcResult(C.Structure):
    _fields_ = [("n_arcs", C.c_int32), ("arcs", C.c_void_p), ("max_arcs", C.c_int32),
                ("acoustic", C.c_double), ("lm", C.c_double), ("combined", C.c_double),
                ("end_ctx", C.c_int64), ("expansions", C.c_int64)]


@dataclass
class OraclePath:
    arcs: tuple
    words: tuple
    acoustic_score: float
    lm_score: float
    combined_score: float
    end_context: int
    expansions: int
    table_len: int = -1       # IndexTable length after the decode (decode_many only)


@dataclass
class OracleStats:
    lookups: int
    hits: int
    misses: int
    evictions: int
    entries: int
    table_len: int
    cum_lookups: int
    cum_hits: int
    cum_misses: int
    requests: int
    bytes_indexed: int
    bytes_full_baseline: int


class OracleStack:
    """Oracle RescoreStack (decoder.py:61-70): table + cache + ledger."""

    def __init__(self, model, tree, enabled: bool = True, max_entries: int = (1 << 64) - 2,
                 capacity_bytes: int = 0):
        self.om = model if isinstance(model, OracleModel) else OracleModel(model, tree)
        self.handle = lib().orc_stack_create(self.om.ref, int(bool(enabled)), int(max_entries))
        if capacity_bytes:
            self.set_capacity(capacity_bytes)

    def set_capacity(self, capacity_bytes: int) -> None:
        """RescoreCache.set_capacity (cache.py:130-137)."""
        _check(lib().orc_stack_set_capacity(self.handle, int(capacity_bytes)), "set_capacity")

    def rnnlm_prob(self, w: int, c: int):
        p = np.zeros(1, np.float64)
        cn = np.zeros(1, np.uint64)
        hit = np.zeros(1, np.int32)
        _check(lib().orc_rnnlm_prob(self.handle, int(w), int(c), _ptr(p), _ptr(cn), _ptr(hit)),
               "rnnlm_prob")
        return float(p[0]), int(cn[0]), bool(hit[0])

    def serve(self, ngram: OracleNgram, w: int, c: int):
        d = np.zeros(1, np.float32)
        cn = np.zeros(1, np.uint64)
        _check(lib().orc_serve_request(self.handle, ngram.handle, int(w), int(c), _ptr(d),
                                       _ptr(cn)), "serve")
        return float(d[0]), int(cn[0])

    def context(self, idx: int):
        h = np.zeros(self.om.H, np.float32)
        hist = np.zeros(8, np.int64)
        L = np.zeros(1, np.int32)
        _check(lib().orc_stack_context(self.handle, int(idx), _ptr(h), _ptr(hist), _ptr(L)),
               "decode")
        return h, tuple(int(x) for x in hist[:L[0]])

    def reset(self, retain: bool) -> None:
        lib().orc_stack_reset(self.handle, int(bool(retain)))

    def cache_clear(self) -> None:
        """RescoreCache.clear (cache.py:136-140): entries only."""
        lib().orc_stack_cache_clear(self.handle)

    def roll_stats(self) -> None:
        """RescoreCache.roll_stats (cache.py:156-158)."""
        lib().orc_stack_roll_stats(self.handle)

    def stats(self) -> OracleStats:
        out = np.zeros(12, np.int64)
        lib().orc_stack_stats(self.handle, _ptr(out))
        return OracleStats(*[int(x) for x in out])

    def rescore_onthefly(self, lattice, ngram, lm_weight: float = 1.0,
                         beam: int = 1 << 30) -> OraclePath:
        ol = lattice if isinstance(lattice, OracleLattice) else OracleLattice(lattice)
        og = ngram if isinstance(ngram, OracleNgram) else OracleNgram(ngram)
        buf = np.zeros(max(ol.n_arcs, 1), np.int32)
        res = _OrcResult(0, _ptr(buf).value, len(buf), 0.0, 0.0, 0.0, 0, 0)
        _check(lib().orc_rescore_onthefly(self.handle, og.handle, C.byref(ol.struct),
                                          float(lm_weight), int(beam), C.byref(res)),
               "rescore_onthefly")
        arcs = tuple(int(a) for a in buf[:res.n_arcs])
        words = tuple(int(ol.arrs[2][a]) for a in arcs)
        return OraclePath(arcs, words, res.acoustic, res.lm, res.combined, int(res.end_ctx),
                          int(res.expansions))

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.orc_stack_destroy(self.handle)
            self.handle = None


def path_score(model, tree, ngram, lattice, arc_ids, lm_weight: float = 1.0) -> float:
    """oracle_path_score (reference tests/conftest.py:65-78)."""
    om = model if isinstance(model, OracleModel) else OracleModel(model, tree)
    og = ngram if isinstance(ngram, OracleNgram) else OracleNgram(ngram)
    ol = lattice if isinstance(lattice, OracleLattice) else OracleLattice(lattice)
    a = np.ascontiguousarray(np.asarray(arc_ids, dtype=np.int32))
    out = np.zeros(1, np.float64)
    _check(lib().orc_path_score(om.ref, og.handle, C.byref(ol.struct), _ptr(a), len(a),
                                float(lm_weight), _ptr(out)), "path_score")
    return float(out[0])


def decode_many(model, tree, ngram, lattices, lm_weight=1.0, beam=8, enabled=True,
                n_threads=None):
    """Independent per-utterance streams (retain=False), utterance-parallel."""
    om = model if isinstance(model, OracleModel) else OracleModel(model, tree)
    og = ngram if isinstance(ngram, OracleNgram) else OracleNgram(ngram)
    ols = [l if isinstance(l, OracleLattice) else OracleLattice(l) for l in lattices]
    n = len(ols)
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    LatArr = _OrcLattice * n
    ResArr = _OrcResult * n
    lat_arr = LatArr(*[l.struct for l in ols])
    bufs = [np.zeros(max(l.n_arcs, 1), np.int32) for l in ols]
    res_arr = ResArr(*[_OrcResult(0, _ptr(b).value, len(b), 0.0, 0.0, 0.0, 0, 0) for b in bufs])
    rcs = np.zeros(n, np.int32)
    lk, hi, mi, tl = (np.zeros(n, np.int64) for _ in range(4))
    _check(lib().orc_decode_many_t(om.ref, og.handle, lat_arr, n, float(lm_weight), int(beam),
                                   int(bool(enabled)), int(n_threads), res_arr, _ptr(rcs),
                                   _ptr(lk), _ptr(hi), _ptr(mi), _ptr(tl)), "decode_many")
    out = []
    for i, l in enumerate(ols):
        r = res_arr[i]
        arcs = tuple(int(a) for a in bufs[i][:r.n_arcs])
        out.append((OraclePath(arcs, tuple(int(l.arrs[2][a]) for a in arcs), r.acoustic, r.lm,
                               r.combined, int(r.end_ctx), int(r.expansions), int(tl[i])),
                    (int(lk[i]), int(hi[i]), int(mi[i]))))
    return out


def query_batch(model, tree, h, hist, hlen, words, want_p=True, want_h=True, n_threads=None):
    """Batched (word_logprob, advance_hidden) for n independent queries."""
    om = model if isinstance(model, OracleModel) else OracleModel(model, tree)
    h = np.ascontiguousarray(h, np.float32)
    n = h.shape[0]
    hist = np.ascontiguousarray(hist, np.int64).reshape(n, om.order)
    hlen = np.ascontiguousarray(hlen, np.int32)
    words = np.ascontiguousarray(words, np.int32)
    p = np.zeros(n, np.float64) if want_p else None
    ho = np.zeros((n, om.H), np.float32) if want_h else None
    if n_threads is None:
        n_threads = len(os.sched_getaffinity(0))
    lib().orc_query_batch(om.ref, n, _ptr(h), _ptr(hist), _ptr(hlen), _ptr(words),
                          _ptr(p) if p is not None else None,
                          _ptr(ho) if ho is not None else None, int(n_threads))
    return p, ho


# --------------------------------------------------------------------------
# two-pass rescoring (decoder.py:180-274)
# --------------------------------------------------------------------------

def nbest(lattice, n: int, lm_weight: float = 1.0) -> list:
    """decoder.py:180-230: top-n distinct word sequences by first-pass score.
    Returns OraclePath records (end_context / expansions = 0)."""
    ol = lattice if isinstance(lattice, OracleLattice) else OracleLattice(lattice)
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    n_out = np.zeros(1, np.int32)
    hl = np.zeros(n, np.int32)
    sc = np.zeros((n, 3), np.float64)
    need = np.zeros(1, np.int64)
    cap = max(16, n * 64)
    while True:
        arcs = np.zeros(cap, np.int32)
        rc = lib().orc_nbest(C.byref(ol.struct), n, float(lm_weight), _ptr(n_out), _ptr(hl),
                             _ptr(arcs), cap, _ptr(sc), _ptr(need))
        if rc == -6 and int(need[0]) > cap:
            cap = int(need[0])
            continue
        _check(rc, "nbest")
        break
    word = ol.arrs[2]
    out, o = [], 0
    for k in range(int(n_out[0])):
        a = tuple(int(x) for x in arcs[o:o + hl[k]])
        o += int(hl[k])
        out.append(OraclePath(a, tuple(int(word[x]) for x in a), float(sc[k, 1]),
                              float(sc[k, 2]), float(sc[k, 0]), 0, 0))
    return out


def twopass(om: "OracleModel", ngram, word_seqs, acoustic, mode: str, interp_weight: float = 0.5,
            lm_weight: float = 1.0):
    """decoder.py:243-274 over one n-best list: (lm [n], combined [n], best)."""
    if mode not in ("rnnlm", "hybrid"):
        raise ValueError(f"unknown two-pass mode {mode!r}")
    if len(word_seqs) == 0:
        raise ValueError("empty hypothesis list")
    og = None
    if ngram is not None:
        og = ngram if isinstance(ngram, OracleNgram) else OracleNgram(ngram)
    off = np.zeros(len(word_seqs) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in word_seqs])
    words = np.ascontiguousarray(np.concatenate([np.asarray(w, np.int32) for w in word_seqs])
                                 if off[-1] else np.zeros(1, np.int32), dtype=np.int32)
    ac = np.ascontiguousarray(np.asarray(acoustic, np.float64))
    lm = np.zeros(len(word_seqs))
    comb = np.zeros(len(word_seqs))
    best = np.zeros(1, np.int32)
    _check(lib().orc_twopass(om.ref, og.handle if og else None, len(word_seqs), _ptr(off),
                             _ptr(words), _ptr(ac), 0 if mode == "rnnlm" else 1,
                             float(interp_weight), float(lm_weight), _ptr(lm), _ptr(comb),
                             _ptr(best)), "twopass")
    return lm, comb, int(best[0])
