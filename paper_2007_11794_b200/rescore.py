"""Drop-in mirror of the reference decoder/LM API, executed on the B200.

Same names, argument meaning and error behaviour as the reference
(``otflm.cache``, ``otflm.context_table``, ``otflm.codec``,
``otflm.decoder``); the numeric work, the IndexTable and the result cache
live on the device (libotflm_b200.so), never on the host.

* ``IndexTable``      -- context_table.py:48-119 (device content table)
* ``RescoreCache``    -- cache.py:61-162 (device (c, w) -> (p, c') table;
                         capacity 0 = unbounded is the device mode)
* ``rnnlm_prob``      -- cache.py:165-182
* ``reset_utterance`` -- cache.py:185-191
* ``RescoreStack``    -- decoder.py:61-70
* ``rescore_onthefly``-- decoder.py:114-173
* ``rescore_batch``   -- many utterances, one stream each
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _lib
from .device import DeviceModel, DeviceNgram, DeviceStreams, Plan, PlanGroup, cuda
from .model import RnnlmContext

ENTRY_BYTES = 32          # cache.py:26
REQUEST_BYTES = 16        # codec.py:23
RESPONSE_BYTES = 16
DEFAULT_RNN_BITS = 32
DEFAULT_DEVICE_CONTEXTS = 1 << 18
_HISTORY_SENTINEL = 0xFFFFFFFFFFFFFFFF   # context_table.py: empty history slot


@dataclass(frozen=True)
class CacheValue:
    p: float
    c_next: int


@dataclass
class CacheStats:
    """cache.py:37-58"""

    lookups: int = 0
    hits: int = 0
    misses: int = 0
    evictions: int = 0
    resident_bytes: int = 0

    @property
    def hit_ratio(self) -> float:
        return self.hits / self.lookups if self.lookups else 0.0

    def line(self) -> str:
        return (f"lookups={self.lookups} hits={self.hits} "
                f"hit_ratio={self.hit_ratio:.6f} "
                f"resident_bytes={self.resident_bytes} evictions={self.evictions}")

    def add(self, other: "CacheStats") -> None:
        self.lookups += other.lookups
        self.hits += other.hits
        self.misses += other.misses
        self.evictions += other.evictions


@dataclass
class TransferLedger:
    """codec.py:95-110 -- per-stream byte accounting of the (now on-device)
    request/response exchange; counts are derived from device counters."""

    requests: int = 0
    bytes_indexed: int = 0
    bytes_full_baseline: int = 0
    request_bytes: int = field(default=REQUEST_BYTES, repr=False)
    response_bytes: int = field(default=RESPONSE_BYTES, repr=False)

    def record(self, context_bytes: int, n: int = 1) -> None:
        self.requests += n
        self.bytes_indexed += n * (self.request_bytes + self.response_bytes)
        self.bytes_full_baseline += n * 2 * context_bytes


def reduction_ratio(ledger: TransferLedger, context_bytes: int) -> float:
    if ledger.requests == 0:
        raise ValueError("no requests recorded")
    return ledger.requests * 2 * context_bytes / ledger.bytes_indexed


def pack(rnnlm_index: int, smalllm_index: int, rnn_bits: int = DEFAULT_RNN_BITS) -> int:
    """codec.py:35-46"""
    if not 1 <= rnn_bits <= 63:
        raise ValueError(f"rnn_bits must be in 1..63, got {rnn_bits}")
    small_bits = 64 - rnn_bits
    if not 0 <= rnnlm_index < (1 << rnn_bits):
        raise _lib.PackOverflowError(f"rnnlm_index {rnnlm_index} does not fit in {rnn_bits} bits")
    if not 0 <= smalllm_index < (1 << small_bits):
        raise _lib.PackOverflowError(
            f"smalllm_index {smalllm_index} does not fit in {small_bits} bits")
    return (rnnlm_index << small_bits) | smalllm_index


def unpack(value: int, rnn_bits: int = DEFAULT_RNN_BITS) -> tuple:
    if not 1 <= rnn_bits <= 63:
        raise ValueError(f"rnn_bits must be in 1..63, got {rnn_bits}")
    small_bits = 64 - rnn_bits
    return value >> small_bits, value & ((1 << small_bits) - 1)


# --------------------------------------------------------------------------
class _Binding:
    """One device stream shared by an (IndexTable, RescoreCache) pair."""

    def __init__(self, model, tree, table: "IndexTable", cache: "RescoreCache"):
        self.dmodel = DeviceModel.get(model, tree)
        cap = int(min(table.max_entries, table.device_capacity))
        self.streams = DeviceStreams(self.dmodel, 1, enabled=cache.enabled, max_contexts=cap,
                                     cache_slots=2 * cap + 16, arena_rows=cap + 2)
        if cache.capacity_bytes:
            self.streams.set_capacity(cache.capacity_bytes)
        self.model, self.tree = model, tree


class IndexTable:
    """Device IndexTable (context_table.py:48-119).  Index 0 is the zero
    context; fresh contexts get len + 1; dedup is bit-exact on the f32
    hidden state + history."""

    def __init__(self, hidden_size: int, maxent_order: int, max_entries: int = (1 << 64) - 2,
                 device_capacity: int = DEFAULT_DEVICE_CONTEXTS):
        self.hidden_size = hidden_size
        self.maxent_order = maxent_order
        self.max_entries = max_entries
        self.device_capacity = device_capacity
        self._bind: _Binding | None = None

    @property
    def element_bytes(self) -> int:
        return 4 * self.hidden_size + 8 * self.maxent_order + 8

    def __len__(self) -> int:
        if self._bind is None:
            return 0
        return int(self._bind.streams.stats()[0, 3])

    def decode(self, idx: int) -> RnnlmContext:
        idx = int(idx)
        if idx == 0:
            return RnnlmContext(np.zeros(self.hidden_size, np.float32), ())
        if self._bind is None or not 1 <= idx <= len(self):
            raise _lib.UnknownIndexError(f"index {idx} not in table (length {len(self)})")
        h, hist = self._bind.streams.context(0, idx)
        return RnnlmContext(h, hist)

    def bind(self, model, tree, cache: "RescoreCache | None" = None) -> "IndexTable":
        """Attach the table to a model's device stream (rnnlm_prob and
        RescoreStack do this on first use)."""
        _binding(cache if cache is not None else RescoreCache(), self, model, tree)
        return self

    def encode(self, ctx: RnnlmContext) -> int:
        """context_table.py:76-89 on the device: the index of an equal stored
        context (bit-exact hidden bytes + history), else len + 1."""
        self._key_bytes(ctx)                                   # the reference's ValueErrors
        if self._bind is None:
            raise ValueError("IndexTable has no device stream yet: call bind(model, tree) "
                             "or use it through rnnlm_prob / a RescoreStack first")
        hist = np.zeros((1, self.maxent_order), np.uint32)
        hist[0, :len(ctx.history)] = ctx.history
        return int(self._bind.streams.encode(0, ctx.hidden[None, :], hist, [len(ctx.history)])[0])

    def _key_bytes(self, ctx: RnnlmContext) -> bytes:
        """context_table.py:64-74: f32 hidden + history slots (u64, sentinel-padded)."""
        if ctx.hidden.shape != (self.hidden_size,):
            raise ValueError(f"context hidden size {ctx.hidden.shape} does not match table "
                             f"H={self.hidden_size}")
        if len(ctx.history) > self.maxent_order:
            raise ValueError("context history longer than table maxent order")
        slots = np.full(self.maxent_order, _HISTORY_SENTINEL, dtype="<u8")
        slots[:len(ctx.history)] = ctx.history
        return np.ascontiguousarray(ctx.hidden, dtype="<f4").tobytes() + slots.tobytes()

    def serialized(self, idx: int) -> bytes:
        """context_table.py:107-111: the stored element bytes of index idx
        (key bytes + u32 order + u32 index), read back from the device row."""
        idx = int(idx)
        if self._bind is None or not 1 <= idx <= len(self):
            raise _lib.UnknownIndexError(f"index {idx} not in table")
        return self._key_bytes(self.decode(idx)) + struct.pack("<II", self.maxent_order, idx)

    def memory_report(self) -> tuple:
        n = len(self)
        return n, self.element_bytes, n * self.element_bytes

    def clear(self) -> None:
        if self._bind is not None:
            self._bind.streams.reset(retain=False)


class RescoreCache:
    """Device result cache (cache.py:61-162).  capacity_bytes = 0: unbounded
    (per-utterance clear via reset_utterance); > 0: at most capacity_bytes /
    ENTRY_BYTES resident entries under the reference's LFU + LRU-tie-break
    eviction (cache.py:98-137), replayed on the device over every lookup in
    reference order -- hits, misses, evictions and resident bytes equal the
    reference's."""

    def __init__(self, capacity_bytes: int = 0, enabled: bool = True):
        if capacity_bytes < 0:
            raise ValueError("capacity_bytes must be >= 0")
        self.capacity_bytes = capacity_bytes
        self.enabled = enabled
        self._bind: _Binding | None = None
        self._rolled = CacheStats()

    def _raw(self):
        return self._bind.streams.stats()[0] if self._bind else np.zeros(8, np.int64)

    def _ev(self):
        if self._bind is None or not self.capacity_bytes:
            return np.zeros(3, np.int64)
        return self._bind.streams.cache_stats()[0]

    def __len__(self) -> int:
        return int(self._raw()[7])

    @property
    def resident_bytes(self) -> int:
        return len(self) * ENTRY_BYTES

    def _direct(self):
        if self._bind is None:
            raise ValueError("RescoreCache has no device stream yet: use it through rnnlm_prob / "
                             "a RescoreStack first (or IndexTable.bind(model, tree, cache))")
        return self._bind.streams

    def get(self, key) -> "CacheValue | None":
        """cache.py:80-94 on the device: counts the lookup; None on a miss
        (and always when the cache is disabled)."""
        c, w = (int(x) for x in key)
        found, p, cn = self._direct().cache_get(0, [c], [w])
        return CacheValue(float(p[0]), int(cn[0])) if found[0] else None

    def clear(self) -> None:
        """cache.py:136-140: drop every entry (and, when bounded, the LFU state); counters are kept."""
        if self._bind is not None:
            self._bind.streams.cache_clear(0)

    def roll_stats(self) -> None:
        """cache.py:156-158: the window counters (and evictions) move into the cumulative ones."""
        if self._bind is not None:
            self._bind.streams.roll_stats(0)

    def put(self, key, value: CacheValue) -> None:
        """cache.py:96-108 on the device: first value wins; no-op when disabled."""
        c, w = (int(x) for x in key)
        self._direct().cache_put(0, [c], [w], [float(value.p)], [int(value.c_next)])

    def set_capacity(self, capacity_bytes: int) -> None:
        """cache.py:130-137: 0 removes the bound; shrinking evicts at once."""
        if capacity_bytes < 0:
            raise ValueError("capacity_bytes must be >= 0")
        self.capacity_bytes = capacity_bytes
        if self._bind is not None:
            self._bind.streams.set_capacity(capacity_bytes)

    def stats(self) -> CacheStats:
        r = self._raw()
        return CacheStats(int(r[0]), int(r[1]), int(r[2]), int(self._ev()[0]), int(r[7]) * ENTRY_BYTES)

    def cumulative_stats(self) -> CacheStats:
        r = self._raw()
        return CacheStats(int(r[4]), int(r[5]), int(r[6]), int(self._ev()[1]), int(r[7]) * ENTRY_BYTES)


def _binding(cache: RescoreCache, table: IndexTable, model, tree) -> _Binding:
    b = table._bind or cache._bind
    if b is None:
        b = _Binding(model, tree, table, cache)
        table._bind = cache._bind = b
    elif table._bind is not cache._bind:
        if cache._bind is None:
            cache._bind = b
        elif table._bind is None:
            table._bind = b
        else:
            raise ValueError("table and cache are bound to different device streams")
    if b.model is not model or b.tree is not tree:
        raise ValueError("stream already bound to a different model")
    return b


def rnnlm_prob(cache: RescoreCache, table: IndexTable, model, tree, w: int, c: int,
               precision: str = "fp64") -> CacheValue:
    """cache.py:165-182 -- one Table-1 lookup on the device."""
    w = int(w)
    if not 0 <= w < model.vocab_size:
        raise ValueError(f"word id {w} out of range 0..{model.vocab_size - 1}")
    b = _binding(cache, table, model, tree)
    p, cn, _ = b.streams.rnnlm_prob_batch([0], [int(c)], [w], precision)
    return CacheValue(float(p[0]), int(cn[0]))


def rnnlm_prob_trace(cache: RescoreCache, table: IndexTable, model, tree, trace,
                     precision: str = "fp64"):
    """Replay a (w, parent_step) trace (reference tests/test_cache.py:60-97)
    in dependency waves: every request whose parent is resolved goes in one
    device batch, with the batch's array order equal to trace order, which
    keeps hit/miss and index numbering identical to one-by-one replay."""
    b = _binding(cache, table, model, tree)
    n = len(trace)
    ws = np.array([t[0] for t in trace], np.int64)
    par = np.array([t[1] for t in trace], np.int64)
    if np.any((ws < 0) | (ws >= model.vocab_size)):
        raise ValueError("word id out of range")
    depth = np.zeros(n, np.int64)
    for i in range(n):
        depth[i] = 0 if par[i] < 0 else depth[par[i]] + 1
    succ = np.zeros(n, np.int64)
    p_out = np.zeros(n)
    hit = np.zeros(n, bool)
    # waves must also respect order: a request may only run after all
    # earlier requests (it could hit their entries), so a wave is a maximal
    # run of consecutive trace entries whose parents lie before the run
    i = 0
    while i < n:
        j = i
        while j < n and (par[j] < i):
            j += 1
        if j == i:
            raise ValueError("trace parent must precede the request")
        cs = np.where(par[i:j] < 0, 0, succ[np.maximum(par[i:j], 0)])
        p, cn, h = b.streams.rnnlm_prob_batch(np.zeros(j - i, np.int32), cs, ws[i:j], precision)
        succ[i:j] = cn
        p_out[i:j] = p
        hit[i:j] = h
        i = j
    return p_out, succ, hit


def reset_utterance(cache: RescoreCache, table: IndexTable, retain: bool) -> None:
    """cache.py:185-191"""
    b = table._bind or cache._bind
    if b is not None:
        b.streams.reset(retain)


@dataclass
class RescoreStack:
    """decoder.py:61-70"""

    model: object
    tree: object
    table: IndexTable
    cache: RescoreCache
    ledger: TransferLedger = field(default_factory=TransferLedger)
    rnn_bits: int = 32


# --------------------------------------------------------------------------
# the paper's search <-> rescorer boundary (codec.py:23-92, decoder.py:73-104):
# 16-byte requests in, 16-byte responses out; the LM work behind serve() is the
# device Table-1 lookup (rnnlm_prob), the small-LM term is the host n-gram
_REQUEST = struct.Struct("<QII")     # packed (c, small idx), word, frame
_RESPONSE = struct.Struct("<fQ4x")   # f32 delta, packed (c', small idx)


def quantize_delta(delta: float) -> float:
    """codec.py:57-60 -- the response carries the delta as an f32."""
    return float(np.float32(delta))


@dataclass(frozen=True)
class RescoreRequest:
    """codec.py:63-75"""

    packed: int
    w: int
    frame: int

    def to_bytes(self) -> bytes:
        return _REQUEST.pack(self.packed, self.w, self.frame)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "RescoreRequest":
        return cls(*_REQUEST.unpack(raw))


@dataclass(frozen=True)
class RescoreResponse:
    """codec.py:78-92"""

    delta: float
    c_next_packed: int

    @classmethod
    def build(cls, delta: float, c_next_packed: int) -> "RescoreResponse":
        return cls(quantize_delta(delta), c_next_packed)

    def to_bytes(self) -> bytes:
        return _RESPONSE.pack(self.delta, self.c_next_packed)

    @classmethod
    def from_bytes(cls, raw: bytes) -> "RescoreResponse":
        return cls(*_RESPONSE.unpack(raw))


def small_context(history: Sequence[int], small_lm) -> list:
    """decoder.py:73-80 -- stored history, left-padded with <s>."""
    hist = list(history)
    pad = small_lm.order - 1 - len(hist)
    return [small_lm.bos_id] * pad + hist if pad > 0 else hist


class RescoreServer:
    """decoder.py:83-104: consumes request bytes, returns response bytes.

    ``serve`` answers one request exactly as the reference does; ``serve_batch``
    answers a concatenation of requests with one device batch (array order =
    reference order for cache claims and index numbering), for clients that
    pipeline a frame's requests."""

    def __init__(self, stack: "RescoreStack", small_lm):
        if small_lm.order - 1 > stack.model.maxent_order:
            raise ValueError("small LM order exceeds the stored context history; "
                             f"need maxent_order >= {small_lm.order - 1}")
        self.stack = stack
        self.small_lm = small_lm
        self.precision = "fp64"

    def serve(self, raw: bytes) -> bytes:
        return self.serve_batch(raw)

    def serve_batch(self, raw: bytes) -> bytes:
        from .model import ngram_logprob
        st = self.stack
        n, rem = divmod(len(raw), REQUEST_BYTES)
        if rem or n == 0:
            raise ValueError(f"request buffer of {len(raw)} bytes is not a whole number of "
                             f"{REQUEST_BYTES}-byte requests")
        reqs = np.frombuffer(raw, dtype=np.dtype([("packed", "<u8"), ("w", "<u4"), ("frame", "<u4")]))
        small_bits = 64 - st.rnn_bits
        if not 1 <= st.rnn_bits <= 63:
            raise ValueError(f"rnn_bits must be in 1..63, got {st.rnn_bits}")
        c = (reqs["packed"] >> np.uint64(small_bits)).astype(np.int64)
        small = reqs["packed"] & np.uint64((1 << small_bits) - 1)
        w = reqs["w"].astype(np.int64)
        if np.any(w >= st.model.vocab_size):
            raise ValueError(f"word id out of range 0..{st.model.vocab_size - 1}")
        if np.any(c >= (1 << 32)):
            raise _lib.UnknownIndexError("context index beyond the device table")
        b = _binding(st.cache, st.table, st.model, st.tree)
        p, cn, _ = b.streams.rnnlm_prob_batch(np.zeros(n, np.int32), c, w, self.precision)
        hist = {}
        out = bytearray()
        for i in range(n):
            ci = int(c[i])
            if ci not in hist:
                hist[ci] = st.table.decode(ci).history
            p_small = ngram_logprob(self.small_lm, small_context(hist[ci], self.small_lm), int(w[i]))
            out += RescoreResponse.build(float(p[i]) - p_small,
                                         pack(int(cn[i]), int(small[i]), st.rnn_bits)).to_bytes()
        st.ledger.record(st.table.element_bytes, n)
        return bytes(out)


def first_pass_weight(arc, lm_weight: float) -> float:
    """decoder.py:176-177"""
    return arc.acoustic + lm_weight * arc.smalllm


def rescored_path_score(lattice, arc_ids: Sequence[int], model, tree, small_lm,
                        lm_weight: float = 1.0) -> float:
    """decoder.py:277-292 -- one path under the on-the-fly objective, straight
    from the model (device word_logprob / advance_context, exact f64 mode)."""
    from . import advance_context, word_logprob
    from .model import ngram_logprob
    ctx = model.zero_context()
    score = 0.0
    for a in arc_ids:
        arc = lattice.arcs[a]
        p = word_logprob(model, tree, ctx, arc.word)
        p_small = ngram_logprob(small_lm, small_context(ctx.history, small_lm), arc.word)
        score = score + arc.acoustic + lm_weight * (arc.smalllm + quantize_delta(p - p_small))
        ctx = advance_context(model, ctx, arc.word)
    return score


def edit_distance(ref: Sequence, hyp: Sequence) -> int:
    """decoder.py:295-303 -- Levenshtein distance (word error counts)."""
    row = np.arange(len(hyp) + 1)
    for i, r in enumerate(ref, 1):
        nxt = np.empty_like(row)
        nxt[0] = i
        for j, h in enumerate(hyp, 1):
            nxt[j] = min(row[j] + 1, nxt[j - 1] + 1, row[j - 1] + (r != h))
        row = nxt
    return int(row[-1])


@dataclass
class PathHypothesis:
    """decoder.py:49-58"""

    arcs: tuple
    words: tuple
    acoustic_score: float
    lm_score: float
    combined_score: float
    end_context: int = 0


@dataclass
class TraversalReport:
    """decoder.py:107-111"""

    expansions: int
    cache_stats: object
    transfer: TransferLedger


def _hyp(out, u, lat, arc_base: int = 0) -> PathHypothesis:
    n = int(out["path_len"][u])
    a = out["path_arcs"][u, :n].astype(np.int64) - arc_base            # batch -> lattice arc ids
    arcs = tuple(a.tolist())
    words = tuple(np.asarray(lat.arc_word)[a].tolist())
    return PathHypothesis(arcs, words, float(out["acoustic"][u]), float(out["lm"][u]),
                          float(out["combined"][u]), int(out["end_ctx"][u]))


def rescore_onthefly(lattice, small_lm, stack: RescoreStack, lm_weight: float = 1.0,
                     beam: int = 1 << 30, precision: str = "fp64"):
    """decoder.py:114-173 -- one utterance on the stack's device stream."""
    if beam < 1:
        raise ValueError("beam must be >= 1")
    if small_lm.order - 1 > stack.model.maxent_order:
        raise ValueError("small LM order exceeds the stored context history; "
                         f"need maxent_order >= {small_lm.order - 1}")
    b = _binding(stack.cache, stack.table, stack.model, stack.tree)
    g = DeviceNgram.get(small_lm, b.dmodel)
    plan = Plan(b.streams, [lattice], beam)
    plan.run(g, lm_weight, precision, use_graph=False)
    out = plan.fetch()
    hyp = _hyp(out, 0, plan.lats[0])
    exp = int(out["expansions"][0])
    stack.ledger.record(stack.table.element_bytes, exp)
    return hyp, TraversalReport(expansions=exp, cache_stats=stack.cache.stats(),
                                transfer=stack.ledger)


class BatchDecoder:
    """Decode many utterances at once, one independent stream each
    (retain=False semantics between batches), on one GPU.

    ``prepare`` compiles and uploads the lattices (host->device), ``run``
    decodes with the inputs resident in HBM (replaying a CUDA graph of the
    level loop), ``fetch`` copies the 1-best paths back.  With ``n_groups``
    > 1 the utterances are split into groups whose level loops run as
    parallel chains of the same graph (each with its own arena partition).
    """

    def __init__(self, model, tree, small_lm, n_streams: int, max_contexts: int,
                 enabled: bool = True, precision: str = "fp64", n_groups: int = 1,
                 schedule: str = "auto", n_buffers: int = 1, capacity_bytes: int = 0,
                 lattice_out: bool = False):
        self.model, self.tree = model, tree
        self.dmodel = DeviceModel.get(model, tree)
        self.ngram = DeviceNgram.get(small_lm, self.dmodel)
        self.precision = precision
        # "auto": the persistent kernels for ordinary beams; a batch with wide
        # levels (big beams: nodes of more than 64 arrival slots) is moved to
        # the level schedule when it is prepared (k_expand_big / k_asg_*)
        self._auto = schedule == "auto"
        if schedule == "auto":
            schedule = auto_schedule(self.dmodel, precision, n_streams)
        if schedule not in _lib.SCHED:
            raise ValueError(f"unknown schedule {schedule!r}")
        if schedule != "level" and not schedule_supported(self.dmodel, schedule, precision):
            raise ValueError(f"the {schedule} schedule does not support precision {precision!r} / this model")
        self.schedule = schedule
        # concurrent groups only help the level-synchronous schedule
        self.n_groups = 1 if schedule != "level" else max(1, min(int(n_groups), n_streams))
        self.arena_rows = n_streams * max_contexts + 2
        self.streams = DeviceStreams(self.dmodel, n_streams, enabled=enabled,
                                     max_contexts=max_contexts,
                                     cache_slots=2 * max_contexts + 16,
                                     arena_rows=self.arena_rows)
        if capacity_bytes:
            self.streams.set_capacity(capacity_bytes)
        self.lattice_out = bool(lattice_out)
        self.plans = []
        self.group = None
        self.plan = None
        # n_buffers = 2: two plan sets used alternately, so the host compile +
        # upload of batch i+1 (prepare) overlaps the decode of batch i
        self.n_buffers = max(1, int(n_buffers))
        self._slots = [dict(plans=[], spans=[], group=None, plan=None, beam=None, done=None)
                       for _ in range(self.n_buffers)]
        self._side = None            # copy stream for fetch (waits only for its own batch)
        self._cur = 0
        self._next = 0

    def _activate(self, slot: int) -> None:
        st = self._slots[slot]
        self.plans, self.spans, self.group, self.plan = st["plans"], st["spans"], st["group"], st["plan"]
        self.beam = st["beam"]
        self._cur = slot

    def _store(self, slot: int) -> None:
        self._slots[slot].update(plans=self.plans, spans=self.spans, group=self.group, plan=self.plan,
                                 beam=getattr(self, "beam", None))

    @staticmethod
    def contexts_needed(lattices, beam: int) -> int:
        """Upper bound on new contexts per utterance: every request may
        create one (sum over nodes of min(beam, capacity) * out-degree)."""
        from .lattice import as_lattice
        worst = 0
        for lat in lattices:
            l = as_lattice(lat)
            worst = max(worst, int(min(beam, 1 << 20)) * l.n_arcs)
        return worst + 1

    def prepare(self, lattices, beam: int):
        """Compile + upload a batch into the next plan buffer and make it the
        current one (returns the buffer index for run / fetch).  A batch with
        the same compiled structure as the buffer's previous one is loaded
        into the existing plans (captured graphs are replayed); otherwise new
        plans are built."""
        slot = self._next
        self._next = (self._next + 1) % self.n_buffers
        self._activate(slot)
        self._prepare(lattices, beam)
        self._store(slot)
        return slot

    def _prepare(self, lattices, beam: int):
        lattices = list(lattices)
        G = min(self.n_groups, len(lattices))
        bounds = np.linspace(0, len(lattices), G + 1).astype(int)
        if self.plans and getattr(self, "beam", None) == beam and len(self.plans) == G and \
                all(len(ids) == b1 - b0 for ids, b0, b1 in zip(self.spans, bounds[:-1], bounds[1:])):
            if all(p.refresh([lattices[i] for i in ids], stream_ids=ids)
                   for p, ids in zip(self.plans, self.spans)):
                return self.plans
        self.beam = beam
        self.plans = []
        self.spans = []
        rows = (self.arena_rows - 1) // G
        for g in range(G):
            ids = np.arange(bounds[g], bounds[g + 1])
            p = Plan(self.streams, [lattices[i] for i in ids], beam, stream_ids=ids)
            if self._auto and self.schedule != "level" and p.wide():
                self.schedule = "level"
            p.set_schedule(self.schedule)
            if self.lattice_out:
                p.set_lattice_out(True)
            if G > 1:
                p.set_arena(1 + g * rows, 1 + (g + 1) * rows)
            self.plans.append(p)
            self.spans.append(ids)
        self.group = PlanGroup(self.plans) if G > 1 else None
        self.plan = self.plans[0]
        return self.plans

    def run(self, lm_weight: float = 1.0, use_graph: bool = True, slot: int | None = None,
            retain: bool = False) -> None:
        """Decode the current batch (one utterance per stream).  retain=True
        keeps every stream's IndexTable and (bounded) cache from its previous
        utterance (reset_utterance(retain=True), cache.py:185-191) -- the
        paper's Table-4 setting; False starts fresh streams."""
        if slot is not None:
            self._activate(slot)
        self._lm_weight = lm_weight
        self.streams.reset(retain=bool(retain))
        if self.group is not None:
            self.group.run(self.ngram, lm_weight, self.precision)
        else:
            self.plan.run(self.ngram, lm_weight, self.precision, use_graph=use_graph)
        if self.n_buffers > 1:           # completion of this batch, for fetch on the copy stream
            torch = cuda()
            ev = torch.cuda.Event()
            ev.record()
            self._slots[self._cur]["done"] = ev

    def profile(self, lm_weight: float = 1.0) -> dict:
        self.streams.reset(retain=False)
        if self.group is not None:
            return self.group.profile(self.ngram, lm_weight, self.precision)
        return self.plan.profile(self.ngram, lm_weight, self.precision)

    def counters(self) -> dict:
        tot = {}
        for p in self.plans:
            for k, v in p.counters().items():
                tot[k] = tot.get(k, 0) + v
        return tot

    def fetch(self, slot: int | None = None):
        if slot is not None:
            self._activate(slot)
        stream = None
        done = self._slots[self._cur].get("done") if self.n_buffers > 1 else None
        if done is not None:
            # read this batch's results on a copy stream that waits only for
            # its own decode, not for a later batch already queued behind it
            torch = cuda()
            if self._side is None:
                self._side = torch.cuda.Stream()
            self._side.wait_event(done)
            stream = self._side.cuda_stream
        hyps, outs = [], []
        for p in self.plans:
            out = p.fetch(stream=stream)
            offs = p.arrays["arc_off"]
            hyps += [_hyp(out, u, p.lats[u], int(offs[u])) for u in range(p.n_utt)]
            outs.append(out)
        merged = {}
        for k in outs[0]:
            if k == "path_arcs":
                w = max(o[k].shape[1] for o in outs)
                merged[k] = np.concatenate([np.pad(o[k], ((0, 0), (0, w - o[k].shape[1])))
                                            for o in outs])
            else:
                merged[k] = np.concatenate([o[k] for o in outs])
        return hyps, merged


    def fetch_lattices(self, slot: int | None = None) -> list:
        """Lattice-out (BatchDecoder(lattice_out=True)): per utterance the
        RNNLM-rescored, beam-pruned state lattice of the last run as a
        ``Lattice``.  States are the kept tokens (node, context); an arc
        carries the original arc's word and acoustic score and, as its
        small-LM field, the rescored LM term (smalllm + delta), so that
        acoustic + lm_weight * smalllm is the arc's on-the-fly weight and the
        best path under first-pass weights is the on-the-fly 1-best."""
        from .lattice import Lattice
        if not self.lattice_out:
            raise ValueError("BatchDecoder(lattice_out=True) is required")
        if slot is not None:
            self._activate(slot)
        lm_w = getattr(self, "_lm_weight", 1.0)
        out = []
        for p in self.plans:
            recs = p.fetch_lattice_records()
            A = p.arrays
            for u, r in enumerate(recs):
                a0 = int(A["arc_off"][u])
                lat = p.lats[u]
                st = r["state"].astype(np.int64)
                score = dict(zip(st.tolist(), r["score"].tolist()))
                child = r["parent"] != 0xFFFFFFFF
                start = int(st[~child][0])
                arc = r["arc"][child].astype(np.int64) - a0
                par = r["parent"][child].astype(np.int64)
                sc = r["score"][child]
                psc = np.array([score[int(x)] for x in par], np.float64)
                ac = np.asarray(lat.arc_acoustic, np.float64)[arc]
                lmv = (sc - psc - ac) / lm_w if lm_w != 0 else np.zeros(len(arc))
                fin_nodes = set(int(x) for x in lat.finals)
                dst_node = np.asarray(lat.arc_dst)[arc]
                finals = sorted(int(s_) for s_, d in zip(st[child].tolist(), dst_node.tolist())
                                if int(d) in fin_nodes)
                if lat.start in fin_nodes:
                    finals = sorted(set(finals) | {start})
                lo = Lattice(start, finals, src=par, dst=st[child],
                             word=np.asarray(lat.arc_word)[arc], acoustic=ac, smalllm=lmv)
                lo.arc_ref = arc          # arc id in the input lattice, per output arc
                out.append(lo)
        return out


def auto_schedule(dmodel, precision: str, n_streams: int) -> str:
    """The persistent per-stream kernel where the precision has one: in
    EXACT, one CTA per stream ("stream1") once the batch has more streams
    than half the SMs (a 2-CTA cluster per stream would need a second wave),
    else the 2-CTA cluster ("stream"); otherwise the level schedule."""
    if schedule_supported(dmodel, "stream", precision):
        if schedule_supported(dmodel, "stream1", precision):
            torch = cuda()
            n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            if 2 * n_streams > n_sm:
                return "stream1"
        return "stream"
    return "level"


def schedule_supported(dmodel, schedule: str, precision: str) -> bool:
    return bool(_lib.load().otflm_schedule_supported(dmodel.handle, _lib.SCHED[schedule],
                                                     _lib.PREC[precision]))


def rescore_batch(lattices: Sequence, small_lm, model, tree, lm_weight: float = 1.0,
                  beam: int = 8, precision: str = "fp64", enabled: bool = True,
                  max_contexts: int | None = None, schedule: str = "auto"):
    """Many utterances, independent fresh streams (retain=False)."""
    if max_contexts is None:
        max_contexts = BatchDecoder.contexts_needed(lattices, beam)
    dec = BatchDecoder(model, tree, small_lm, len(lattices), max_contexts, enabled, precision,
                       schedule=schedule)
    dec.prepare(lattices, beam)
    dec.run(lm_weight, use_graph=False)
    hyps, out = dec.fetch()
    return hyps, out
