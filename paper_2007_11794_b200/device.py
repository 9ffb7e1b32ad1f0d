"""Device-resident objects: model, small LM, decoding streams, decode plans.

Thin owners of the C-ABI handles (include/otflm_b200.h).  torch is used only
for device buffers and the current CUDA stream; the computation is in
libotflm_b200.so.
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .lattice import as_lattice
from .model import ngram_flat


def cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("a CUDA device is required: the product path has no CPU fallback")
    return torch


def current_stream_ptr() -> int:
    torch = cuda()
    return torch.cuda.current_stream().cuda_stream


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class DeviceModel:
    """Uploaded RNNLM (+ Huffman path CSR).  Immutable; shareable."""

    _cache: dict = {}

    def __init__(self, model, tree=None, device: int = 0, *, recurrent: bool = True,
                 output: bool = True):
        cuda()
        L = _lib.load()
        self.H = int(model.hidden_size)
        self.V = int(model.vocab_size)
        self.order = int(model.maxent_order)
        self.maxent_size = int(model.maxent_size)
        keep = []

        def arr(x, dt):
            a = np.ascontiguousarray(x, dtype=dt)
            keep.append(a)
            return a

        U = arr(model.input_weights, np.float32) if recurrent else None
        W = arr(model.recurrent_weights, np.float32) if recurrent else None
        NV = arr(model.node_vectors, np.float32) if output else None
        ME = arr(model.maxent_table, np.float32) if output else None
        if tree is not None:
            pn = arr(tree.path_nodes, np.int32)
            ps = arr(tree.path_signs, np.float32)
            po = arr(tree.path_offsets, np.int64)
            if len(po) != self.V + 1:
                raise ValueError("tree size does not match model vocabulary")
            n_path = int(len(pn))
        else:
            pn = ps = po = None
            n_path = -1
        desc = _lib.ModelDesc(self.H, self.V, self.order, self.maxent_size,
                              int(model.hash_seed) & (2 ** 64 - 1), _p(U), _p(W), _p(NV), _p(ME),
                              _p(pn), _p(ps), _p(po), n_path)
        h = C.c_void_p()
        _lib.check(L.otflm_model_create(C.byref(desc), int(device), C.byref(h)), "model upload")
        self.handle = h
        self.device = device
        self._fin = weakref.finalize(self, L.otflm_model_destroy, h)

    @classmethod
    def get(cls, model, tree=None):
        """Upload once per (model, tree) object pair."""
        key = (id(model), id(tree))
        ent = cls._cache.get(key)
        if ent is None or ent[0] is not model or ent[1] is not tree:
            ent = (model, tree, cls(model, tree))
            cls._cache[key] = ent
        return ent[2]


class DeviceNgram:
    """Small LM tables as device open-addressing hashes."""

    _cache: dict = {}

    def __init__(self, lm, dmodel: DeviceModel | None = None):
        cuda()
        L = _lib.load()
        order, (n_p, kp, lp, vp), (n_b, kb, lb, vb) = ngram_flat(lm)
        self.order = order
        self._keep = (kp, lp, vp, kb, lb, vb)
        desc = _lib.NgramDesc(order, int(lm.vocab_size), int(lm.bos_id), n_p, _p(kp), _p(lp),
                              _p(vp), n_b, _p(kb), _p(lb), _p(vb))
        h = C.c_void_p()
        _lib.check(L.otflm_ngram_create(C.byref(desc), dmodel.handle if dmodel else None,
                                        C.byref(h)), "small LM upload")
        self.handle = h
        self._fin = weakref.finalize(self, L.otflm_ngram_destroy, h)

    @classmethod
    def get(cls, lm, dmodel=None):
        key = id(lm)
        ent = cls._cache.get(key)
        if ent is None or ent[0] is not lm:
            ent = (lm, cls(lm, dmodel))
            cls._cache[key] = ent
        return ent[1]


class DeviceStreams:
    """n independent decoding streams: IndexTable + RescoreCache each."""

    def __init__(self, dmodel: DeviceModel, n_streams: int, enabled: bool = True,
                 max_contexts: int = 1 << 16, cache_slots: int | None = None,
                 arena_rows: int | None = None):
        L = _lib.load()
        self.dmodel = dmodel
        self.n = int(n_streams)
        self.enabled = bool(enabled)
        self.max_contexts = int(max_contexts)
        if cache_slots is None:
            cache_slots = 2 * self.max_contexts + 16
        if arena_rows is None:
            arena_rows = self.n * self.max_contexts + 2
        cfg = _lib.StreamConfig(self.n, int(self.enabled), self.max_contexts, int(cache_slots),
                                int(arena_rows))
        h = C.c_void_p()
        _lib.check(L.otflm_streams_create(dmodel.handle, C.byref(cfg), C.byref(h)),
                   "stream allocation")
        self.handle = h
        self._fin = weakref.finalize(self, L.otflm_streams_destroy, h)

    def reset(self, retain: bool) -> None:
        _lib.check(_lib.load().otflm_streams_reset(self.handle, int(bool(retain)),
                                                   current_stream_ptr()), "reset")

    def stats(self) -> np.ndarray:
        out = np.zeros((self.n, 8), np.int64)
        _lib.check(_lib.load().otflm_streams_stats(self.handle, _p(out), current_stream_ptr()),
                   "stats")
        return out

    def set_capacity(self, capacity_bytes: int) -> None:
        """RescoreCache capacity of every stream (cache.py:61-137); 0 = unbounded."""
        if capacity_bytes < 0:
            raise ValueError("capacity_bytes must be >= 0")
        _lib.check(_lib.load().otflm_streams_set_capacity(self.handle, int(capacity_bytes),
                                                          current_stream_ptr()), "set_capacity")

    def cache_stats(self) -> np.ndarray:
        """[n, 3]: evictions (window), evictions (cumulative), resident entries."""
        out = np.zeros((self.n, 3), np.int64)
        _lib.check(_lib.load().otflm_streams_cache_stats(self.handle, _p(out), current_stream_ptr()),
                   "stats")
        return out

    def context(self, stream_id: int, idx: int):
        h = np.zeros(self.dmodel.H, np.float32)
        hist = np.zeros(8, np.int32)
        n = np.zeros(1, np.int32)
        _lib.check(_lib.load().otflm_streams_context(self.handle, int(stream_id), int(idx), _p(h),
                                                     _p(hist), _p(n), current_stream_ptr()),
                   "decode")
        return h, tuple(int(x) for x in hist[:n[0]])

    def encode(self, stream_id: int, hidden, hist, hist_len):
        """IndexTable.encode of n host contexts on one stream (context_table.py:76-89)."""
        hh = np.ascontiguousarray(hidden, np.float32)
        hs = np.ascontiguousarray(hist, np.uint32)
        hl = np.ascontiguousarray(hist_len, np.int32)
        idx = np.zeros(len(hl), np.uint32)
        _lib.check(_lib.load().otflm_streams_encode(self.handle, int(stream_id), len(hl), _p(hh), _p(hs),
                                                    _p(hl), _p(idx), current_stream_ptr()), "encode")
        return idx

    def cache_get(self, stream_id: int, c, w):
        cc = np.ascontiguousarray(c, np.uint32)
        ww = np.ascontiguousarray(w, np.int32)
        n = len(ww)
        found = np.zeros(n, np.uint8)
        p = np.zeros(n, np.float64)
        cn = np.zeros(n, np.uint32)
        _lib.check(_lib.load().otflm_streams_cache_get(self.handle, int(stream_id), n, _p(cc), _p(ww), _p(found),
                                                       _p(p), _p(cn), current_stream_ptr()), "cache get")
        return found.astype(bool), p, cn

    def roll_stats(self, stream_id: int) -> None:
        _lib.check(_lib.load().otflm_streams_roll_stats(self.handle, int(stream_id), current_stream_ptr()),
                   "roll_stats")

    def cache_clear(self, stream_id: int) -> None:
        _lib.check(_lib.load().otflm_streams_cache_clear(self.handle, int(stream_id), current_stream_ptr()),
                   "cache clear")

    def cache_put(self, stream_id: int, c, w, p, cn) -> None:
        cc = np.ascontiguousarray(c, np.uint32)
        ww = np.ascontiguousarray(w, np.int32)
        pp = np.ascontiguousarray(p, np.float64)
        nn = np.ascontiguousarray(cn, np.uint32)
        _lib.check(_lib.load().otflm_streams_cache_put(self.handle, int(stream_id), len(ww), _p(cc), _p(ww), _p(pp),
                                                       _p(nn), current_stream_ptr()), "cache put")

    def rnnlm_prob_batch(self, stream_ids, c, w, precision: str = "fp64"):
        sid = np.ascontiguousarray(stream_ids, np.int32)
        cc = np.ascontiguousarray(c, np.uint32)
        ww = np.ascontiguousarray(w, np.int32)
        n = len(ww)
        p = np.zeros(n, np.float64)
        cn = np.zeros(n, np.uint32)
        hit = np.zeros(n, np.uint8)
        _lib.check(_lib.load().otflm_rnnlm_prob_batch(self.handle, n, _p(sid), _p(cc), _p(ww),
                                                      _lib.PREC[precision], _p(p), _p(cn), _p(hit),
                                                      current_stream_ptr()), "rnnlm_prob")
        return p, cn, hit.astype(bool)


def pack_lattices(lattices, stream_ids=None):
    """Flatten lattices into the C-ABI batch (node ids remapped monotonically
    onto 0..n-1, which keeps Kahn smallest-id order and sorted finals)."""
    lats = [as_lattice(l) for l in lattices]
    U = len(lats)
    n_nodes = np.zeros(U, np.int32)
    start = np.zeros(U, np.int32)
    arc_off = np.zeros(U + 1, np.int64)
    final_off = np.zeros(U + 1, np.int64)
    src, dst, word, ac, slm, finals = [], [], [], [], [], []
    for i, lat in enumerate(lats):
        ids = lat.node_ids
        n_nodes[i] = len(ids)
        if len(ids) and ids[0] == 0 and ids[-1] == len(ids) - 1:     # already 0..n-1 (sorted unique)
            start[i] = lat.start
            src.append(lat.arc_src.astype(np.int32, copy=False))
            dst.append(lat.arc_dst.astype(np.int32, copy=False))
        else:
            start[i] = np.searchsorted(ids, lat.start)
            src.append(np.searchsorted(ids, lat.arc_src).astype(np.int32))
            dst.append(np.searchsorted(ids, lat.arc_dst).astype(np.int32))
        word.append(lat.arc_word.astype(np.int32))
        ac.append(lat.arc_acoustic)
        slm.append(lat.arc_smalllm)
        f = np.searchsorted(ids, np.array(sorted(lat.finals), np.int64)).astype(np.int32)
        finals.append(f)
        arc_off[i + 1] = arc_off[i] + lat.n_arcs
        final_off[i + 1] = final_off[i] + len(f)
    cat = lambda xs, dt: np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0), dt)
    arrays = dict(n_nodes=n_nodes, start=start, arc_off=arc_off, arc_src=cat(src, np.int32),
                  arc_dst=cat(dst, np.int32), arc_word=cat(word, np.int32),
                  arc_ac=cat(ac, np.float64), arc_slm=cat(slm, np.float64), final_off=final_off,
                  finals=cat(finals, np.int32),
                  stream_ids=np.ascontiguousarray(
                      np.arange(U) if stream_ids is None else stream_ids, np.int32))
    batch = _lib.LatticeBatch(U, *[_p(arrays[k]) for k in (
        "n_nodes", "start", "arc_off", "arc_src", "arc_dst", "arc_word", "arc_ac", "arc_slm",
        "final_off", "finals", "stream_ids")])
    return batch, arrays, lats


class Plan:
    """A compiled, uploaded lattice batch (reusable across runs)."""

    def __init__(self, streams: DeviceStreams, lattices, beam: int, stream_ids=None):
        L = _lib.load()
        self.streams = streams
        self.batch, self.arrays, self.lats = pack_lattices(lattices, stream_ids)
        self.n_utt = len(self.lats)
        h = C.c_void_p()
        _lib.check(L.otflm_plan_create(streams.handle, C.byref(self.batch), int(beam), C.byref(h),
                                       current_stream_ptr()), "lattice compile")
        self.handle = h
        self._fin = weakref.finalize(self, L.otflm_plan_destroy, h)
        info = self.info()
        self.n_levels = int(info[0])
        self.max_path = max(self.n_levels, 1)

    def info(self) -> np.ndarray:
        out = np.zeros(8, np.int64)
        _lib.check(_lib.load().otflm_plan_info(self.handle, _p(out)), "plan info")
        return out

    def wide(self) -> int:
        """Bit 0: nodes with more than 64 arrival slots (CTA-per-node expand);
        bit 1: request ranges above 4096 per (level, stream) (multi-CTA
        assign).  Both are level-schedule kernels."""
        f = C.c_int32(0)
        _lib.check(_lib.load().otflm_plan_wide(self.handle, C.byref(f)), "plan wide")
        return int(f.value)

    def refresh(self, lattices, stream_ids=None) -> bool:
        """Load another batch with the same compiled structure into this plan
        (same buffers, captured graphs stay valid).  False: structure differs."""
        batch, arrays, lats = pack_lattices(lattices, stream_ids)
        same = C.c_int32(0)
        rc = _lib.load().otflm_plan_refresh(self.handle, C.byref(batch), C.byref(same),
                                            current_stream_ptr())
        if not same.value:
            return False
        _lib.check(rc, "plan refresh")
        self.batch, self.arrays, self.lats = batch, arrays, lats
        return True

    def set_arena(self, start: int, end: int) -> None:
        _lib.check(_lib.load().otflm_plan_set_arena(self.handle, int(start), int(end)), "arena")

    def phase_ns(self) -> dict:
        """Stream schedule, after ``profile``: device ns per phase summed over
        CTAs (utterance streams)."""
        o = np.zeros(32, np.int64)
        _lib.check(_lib.load().otflm_plan_phase_ns(self.handle, o.ctypes.data, current_stream_ptr()),
                   "phase_ns")
        names = ("expand", "update_kloop", "update_drain", "update_epilogue", "hs_setup", "hs_pairs",
                 "hs_group_total", "assign", "control_waits_for_update", "mma_wait_operands",
                 "update_fallback")
        # (EXACT profiling: index 5 on rank 1 is also used for the digitize
        # row table and 6 for the digitize body -- see exact_update.cuh)
        # (EXACT: update_kloop = digitize the context rows, update_drain = the
        # digit-pair K loops, update_fallback = the uncertified elements' loop)
        out = {k: int(o[i]) for i, k in enumerate(names)}
        for i, k in enumerate(("assign_probe", "assign_dedup_scan", "assign_numbering", "assign_values",
                               "assign_arrivals")):
            out[k] = int(o[12 + i])
        out["ctas"] = int(o[11])
        out["x_row_table"] = int(o[17])
        out["x_digitize"] = int(o[18])
        out["x_epi_tmem"] = int(o[19])
        out["x_epi_certify"] = int(o[20])
        out["x_hs_wait_digits"] = int(o[21])
        out["x_hs_kloop"] = int(o[9])
        out["x_hs_gemm_epilogue"] = int(o[22])
        out["x_hs_maxent_lsig"] = int(o[23])
        out["x_plane_rows"] = int(o[24])
        out["x_plane_copy"] = int(o[25])
        out["x_update_mma"] = int(o[26])       # the MMA warp's K loops (issue to completion)
        out["x_epi_rest"] = int(o[27])         # epilogue stores / digests / U loads between row groups
        # warp 2 under the update K loops (solo kernel): HS tail, row stores, fallbacks, U staging
        for i, k in enumerate(("w2_hs_tail", "w2_rows_out", "w2_fallbacks", "w2_u_stage")):
            out[k] = int(o[28 + i])
        return out

    def set_schedule(self, schedule: str) -> None:
        """"level" (level-synchronous kernels, CUDA graph) or "stream"
        (persistent kernel, one CTA per utterance stream)."""
        _lib.check(_lib.load().otflm_plan_set_schedule(self.handle, _lib.SCHED[schedule]), "schedule")
        self.schedule = schedule

    def counters(self) -> dict:
        out = np.zeros(6, np.int64)
        _lib.check(_lib.load().otflm_plan_counters(self.handle, _p(out), current_stream_ptr()),
                   "plan counters")
        return dict(sum_path=int(out[0]), sum_path_k=int(out[1]), hs_queries=int(out[2]),
                    h2d_bytes=int(out[3]), exact_fallbacks=int(out[4]), exact_rows_digitized_late=int(out[5]))

    def run(self, ngram: DeviceNgram, lm_weight: float = 1.0, precision: str = "fp64",
            use_graph: bool = True, stream: int | None = None) -> None:
        _lib.check(_lib.load().otflm_decode_run(
            self.handle, ngram.handle, float(lm_weight), _lib.PREC[precision], int(use_graph),
            current_stream_ptr() if stream is None else stream), "decode")

    def profile(self, ngram: DeviceNgram, lm_weight: float = 1.0, precision: str = "fp64") -> dict:
        """One run replayed from a graph with event nodes around every kernel:
        {category: (total device ms, launches)}."""
        ms = np.zeros(len(_lib.PROFILE_CATEGORIES))
        n = np.zeros(len(_lib.PROFILE_CATEGORIES), np.int64)
        _lib.check(_lib.load().otflm_decode_profile(self.handle, ngram.handle, float(lm_weight),
                                                    _lib.PREC[precision], current_stream_ptr(),
                                                    _p(ms), _p(n)), "profile")
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(_lib.PROFILE_CATEGORIES)}

    def set_lattice_out(self, enable: bool = True) -> None:
        _lib.check(_lib.load().otflm_plan_set_lattice_out(self.handle, int(bool(enable))), "lattice-out")

    def fetch_lattice_records(self, stream: int | None = None):
        """Per utterance the rescored, pruned state lattice of the last run as
        a structured array (score, state, parent, arc) -- see
        otflm_decode_lattice_fetch."""
        L = _lib.load()
        st = current_stream_ptr() if stream is None else stream
        cnt = np.zeros(self.n_utt, np.int64)
        _lib.check(L.otflm_decode_lattice_fetch(self.handle, _p(cnt), None, 0, st), "lattice-out")
        dt = np.dtype([("score", "<f8"), ("state", "<u4"), ("parent", "<u4"), ("arc", "<u4"), ("pad", "<u4")])
        rec = np.zeros(max(int(cnt.sum()), 1), dt)
        _lib.check(L.otflm_decode_lattice_fetch(self.handle, _p(cnt), rec.ctypes.data_as(C.c_void_p),
                                                len(rec), st), "lattice-out")
        off = np.concatenate([[0], np.cumsum(cnt)])
        return [rec[off[u]:off[u + 1]] for u in range(self.n_utt)]

    def fetch(self, stream: int | None = None):
        U, MP = self.n_utt, self.max_path
        out = dict(path_len=np.zeros(U, np.int32), path_arcs=np.zeros((U, MP), np.int32),
                   combined=np.zeros(U), acoustic=np.zeros(U), lm=np.zeros(U),
                   end_ctx=np.zeros(U, np.int64), expansions=np.zeros(U, np.int64),
                   status=np.zeros(U, np.int32))
        res = _lib.DecodeResult(_p(out["path_len"]), _p(out["path_arcs"]), MP, _p(out["combined"]),
                                _p(out["acoustic"]), _p(out["lm"]), _p(out["end_ctx"]),
                                _p(out["expansions"]), _p(out["status"]))
        _lib.check(_lib.load().otflm_decode_fetch(self.handle, C.byref(res),
                                                  current_stream_ptr() if stream is None else stream),
                   "decode")
        return out


class PlanGroup:
    """Plans over disjoint utterance subsets replayed as parallel chains of
    one CUDA graph; each plan owns an arena partition."""

    def __init__(self, plans):
        L = _lib.load()
        self.plans = plans
        arr = (C.c_void_p * len(plans))(*[p.handle.value for p in plans])
        h = C.c_void_p()
        _lib.check(L.otflm_group_create(arr, len(plans), C.byref(h)), "group")
        self.handle = h
        self._fin = weakref.finalize(self, L.otflm_group_destroy, h)

    def run(self, ngram: DeviceNgram, lm_weight: float = 1.0, precision: str = "fp64") -> None:
        _lib.check(_lib.load().otflm_group_run(self.handle, ngram.handle, float(lm_weight),
                                               _lib.PREC[precision], current_stream_ptr()), "decode")

    def profile(self, ngram: DeviceNgram, lm_weight: float = 1.0, precision: str = "fp64") -> dict:
        ms = np.zeros(len(_lib.PROFILE_CATEGORIES))
        n = np.zeros(len(_lib.PROFILE_CATEGORIES), np.int64)
        _lib.check(_lib.load().otflm_group_profile(self.handle, ngram.handle, float(lm_weight),
                                                   _lib.PREC[precision], current_stream_ptr(),
                                                   _p(ms), _p(n)), "profile")
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(_lib.PROFILE_CATEGORIES)}


def last_launch_count() -> int:
    return int(_lib.load().otflm_last_launch_count())
