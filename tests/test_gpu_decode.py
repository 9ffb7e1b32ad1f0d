"""Decoder / Table-1 parity on the B200 (FP64 mode = exact mode).

Against the reference's own outputs (golden fixtures) and the CPU oracle:
1-best arc sequence identical, context ids / end context identical, cache
hit/miss and IndexTable counts bit-exact, combined score within 1e-9
(float64 path scores; the only source of difference is the f32 rounding of
a delta whose float64 value differs from the reference's by ~1e-16).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import small_results
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9
EXHAUSTIVE = 1 << 30


def _stack(gm, enabled=True):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack
    m = gm.model
    return RescoreStack(model=m, tree=gm.tree, table=IndexTable(m.hidden_size, m.maxent_order,
                                                                device_capacity=1 << 17),
                        cache=RescoreCache(enabled=enabled))


def test_small_decodes_match_reference_golden(small):
    from paper_2007_11794_b200 import rescore_onthefly
    d, gm, lats = small
    beams = [int(b) for b in d["beams"]]
    for row in small_results(d):
        li, bi, en = int(row[0]), int(row[1]), int(row[2])
        st = _stack(gm, enabled=bool(en))
        lm_w = 1.0 if li % 2 else 0.7
        hyp, rep = rescore_onthefly(lats[li], gm.lm, st, lm_weight=lm_w, beam=beams[bi])
        assert hyp.arcs == tuple(d[f"l{li}_b{bi}_e{en}_arcs"]), (li, bi, en)
        assert abs(hyp.combined_score - row[3]) <= TOL
        assert abs(hyp.acoustic_score - row[4]) <= TOL
        assert abs(hyp.lm_score - row[5]) <= TOL
        assert hyp.end_context == int(row[6])
        assert rep.expansions == int(row[7])
        s = st.cache.stats()
        assert (s.lookups, s.hits, s.misses) == tuple(int(x) for x in row[8:11])
        assert len(st.table) == int(row[11])
        # test_decoder.py:100-107 accounting
        assert st.ledger.requests == rep.expansions == s.lookups
        assert st.ledger.bytes_indexed == 32 * rep.expansions == int(row[12])
        assert st.ledger.bytes_full_baseline == int(row[13])


def test_config_a_matches_reference_golden(config_a):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack, rescore_onthefly
    d, model, tree, lm, lat = config_a
    st = RescoreStack(model=model, tree=tree, table=IndexTable(64, 3, device_capacity=1 << 16),
                      cache=RescoreCache())
    hyp, rep = rescore_onthefly(lat, lm, st, beam=8)
    res = d["result"]
    assert hyp.arcs == tuple(d["arcs"])
    assert abs(hyp.combined_score - res[0]) <= TOL
    assert hyp.end_context == int(res[3])
    assert rep.expansions == int(res[4])
    s = st.cache.stats()
    assert (s.lookups, s.hits, s.misses) == tuple(int(x) for x in res[5:8])
    assert len(st.table) == int(res[8])


def test_trace_replay_matches_reference_golden(small):
    """tests/test_cache.py:60-97 and acceptance crit 3: p / c' / hidden."""
    from paper_2007_11794_b200 import IndexTable, RescoreCache, rnnlm_prob_trace
    d, gm, _ = small
    for enabled in (True, False):
        table = IndexTable(16, 3, device_capacity=1 << 13)
        cache = RescoreCache(enabled=enabled)
        p, succ, hit = rnnlm_prob_trace(cache, table, gm.model, gm.tree,
                                        [tuple(int(x) for x in t) for t in d["trace"]])
        assert np.max(np.abs(p - d["trace_p"])) <= 1e-12
        assert np.array_equal(succ, d["trace_c"])
        for i in range(0, len(succ), 37):
            assert table.decode(int(succ[i])).hidden.tobytes() == d["trace_h"][i].tobytes()
        s = cache.stats()
        if enabled:
            assert [s.lookups, s.hits, s.misses, len(table)] == list(d["trace_stats"])
        else:
            assert s.hits == 0 and s.misses == s.lookups == len(d["trace"])
            assert len(table) == int(d["trace_stats"][3])


def test_single_rnnlm_prob_calls(small):
    """test_cache.py:32-57 / :100-110 shapes on the device API."""
    from paper_2007_11794_b200 import IndexTable, RescoreCache, reset_utterance, rnnlm_prob
    d, gm, _ = small
    table, cache = IndexTable(16, 3, device_capacity=1024), RescoreCache()
    v1 = rnnlm_prob(cache, table, gm.model, gm.tree, 5, 0)
    v2 = rnnlm_prob(cache, table, gm.model, gm.tree, 5, 0)
    assert v1 == v2 and v1.c_next == 1
    s = cache.stats()
    assert (s.lookups, s.hits, s.misses) == (2, 1, 1)
    st = O.OracleStack(gm.model, gm.tree)
    p, cn, _ = st.rnnlm_prob(5, 0)
    assert abs(v1.p - p) <= 1e-12
    h, hist = st.context(cn)
    ctx = table.decode(v1.c_next)
    assert ctx.hidden.tobytes() == h.tobytes() and ctx.history == hist
    reset_utterance(cache, table, retain=False)
    assert len(table) == 0 and len(cache) == 0
    assert cache.stats().lookups == 0 and cache.cumulative_stats().lookups == 2
    v = rnnlm_prob(cache, table, gm.model, gm.tree, 3, 0)
    assert v.c_next == 1 and cache.stats().misses == 1
    with pytest.raises(KeyError):
        rnnlm_prob(cache, table, gm.model, gm.tree, 3, 99)     # UnknownIndexError
    with pytest.raises(ValueError):
        rnnlm_prob(cache, table, gm.model, gm.tree, gm.model.vocab_size, 0)


def test_retained_second_pass_computes_nothing(small):
    """test_decoder.py:110-120."""
    from paper_2007_11794_b200 import rescore_onthefly, reset_utterance
    d, gm, lats = small
    st = _stack(gm)
    h1, _ = rescore_onthefly(lats[10], gm.lm, st, beam=8)
    first = st.cache.stats().misses
    reset_utterance(st.cache, st.table, retain=True)
    h2, _ = rescore_onthefly(lats[10], gm.lm, st, beam=8)
    assert st.cache.stats().misses == 0 < first
    assert h1.arcs == h2.arcs and h1.combined_score == h2.combined_score


def test_exhaustive_beam_equals_brute_force(small):
    """test_decoder.py:40-51 / acceptance crit 6 (oracle path score)."""
    from paper_2007_11794_b200 import rescore_onthefly
    d, gm, lats = small
    for li in (0, 3, 6, 9):
        lat = lats[li]
        st = _stack(gm)
        hyp, _ = rescore_onthefly(lat, gm.lm, st, beam=EXHAUSTIVE)
        ol = O.OracleLattice(lat)
        best, best_s = None, -math.inf
        for path in _paths(lat):
            s = O.path_score(gm.model, gm.tree, gm.lm, ol, path)
            if s > best_s:
                best, best_s = path, s
        assert hyp.arcs == best
        assert abs(hyp.combined_score - best_s) <= TOL


def _paths(lat, limit=5000):
    out = []
    outs = {}
    for a in lat.arcs:
        outs.setdefault(a.src, []).append(a)

    def dfs(n, acc):
        assert len(out) < limit
        if n in lat.finals:
            out.append(tuple(acc))
        for a in outs.get(n, []):
            dfs(a.dst, acc + [a.id])

    dfs(lat.start, [])
    return out


@pytest.mark.parametrize("groups", [1, 3])
def test_batch_decode_matches_oracle(groups):
    """Many utterances, one stream each (the bench path), vs the oracle;
    groups > 1 replays the utterance groups as parallel graph chains."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("a", n_utt=12, T=60, seed=3)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=s.beam, n_threads=4)
    need = BatchDecoder.contexts_needed(s.lattices, s.beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, n_groups=groups)
    dec.prepare(s.lattices, s.beam)
    for use_graph in (False, True, True):
        dec.run(1.0, use_graph=use_graph)
        hyps, out = dec.fetch()
        for u, (r, (lk, hi, mi)) in enumerate(ref):
            assert hyps[u].arcs == r.arcs
            assert abs(hyps[u].combined_score - r.combined_score) <= TOL
            assert hyps[u].end_context == r.end_context
            assert int(out["expansions"][u]) == r.expansions
        st = dec.streams.stats()
        assert [int(x) for x in st[:, 0]] == [x[1][0] for x in ref]
        assert [int(x) for x in st[:, 2]] == [x[1][2] for x in ref]


def test_degenerate_zero_model_dedups_contexts(small):
    """test_decoder.py:61-89: zero recurrent weights -> identical hidden
    states, so the IndexTable dedups on history alone; every delta is 0 and
    the best path is the small-LM Viterbi path."""
    from paper_2007_11794_b200 import RnnlmModel, rescore_onthefly
    from paper_2007_11794_b200.lattice import generate_lattice
    from paper_2007_11794_b200.model import log_half_path_unigram
    d, gm, lats = small
    V = gm.model.vocab_size
    model = RnnlmModel.new(V, hidden_size=8, maxent_order=3, maxent_table_bits=6, seed=1)
    model.input_weights[:] = 0
    model.recurrent_weights[:] = 0
    uni = log_half_path_unigram(gm.tree, V, 1, 2)
    ref = [5, 9, 4, 12, 7]
    lat = generate_lattice(ref, V, uni, 3, noise_seed=3)
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack
    st = RescoreStack(model=model, tree=gm.tree, table=IndexTable(8, 3, device_capacity=4096),
                      cache=RescoreCache())
    hyp, _ = rescore_onthefly(lat, uni, st, beam=EXHAUSTIVE)
    ost = O.OracleStack(model, gm.tree)
    r = ost.rescore_onthefly(lat, uni, beam=EXHAUSTIVE)
    assert hyp.arcs == r.arcs and hyp.combined_score == r.combined_score
    assert len(st.table) == ost.stats().table_len
    assert st.cache.stats().hits == ost.stats().hits
    best = max(_paths(lat), key=lambda p: sum(lat.arcs[a].acoustic + lat.arcs[a].smalllm for a in p))
    assert hyp.arcs == best


def test_errors_map_to_reference_exceptions(small):
    from paper_2007_11794_b200 import Lattice, rescore_onthefly
    d, gm, lats = small
    st = _stack(gm)
    with pytest.raises(ValueError):
        rescore_onthefly(lats[0], gm.lm, st, beam=0)
    cyc = Lattice(0, [2], src=[0, 1, 1], dst=[1, 0, 2], word=[3, 4, 5], acoustic=[0, 0, 0],
                  smalllm=[-1.0, -1.0, -1.0])
    with pytest.raises(ValueError):
        rescore_onthefly(cyc, gm.lm, st, beam=4)
    dead = Lattice(0, [3], src=[0, 1], dst=[1, 2], word=[3, 4], acoustic=[0, 0],
                   smalllm=[-1.0, -1.0])
    with pytest.raises(ValueError, match="no complete path"):
        rescore_onthefly(dead, gm.lm, st, beam=4)
    bad = Lattice(0, [1], src=[0], dst=[1], word=[gm.model.vocab_size + 5], acoustic=[0.0],
                  smalllm=[-1.0])
    with pytest.raises(ValueError):
        rescore_onthefly(bad, gm.lm, st, beam=4)


def _decode(s, precision, schedule, beam, enabled=True):
    from paper_2007_11794_b200.rescore import BatchDecoder
    need = BatchDecoder.contexts_needed(s.lattices, beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, enabled=enabled,
                       precision=precision, schedule=schedule)
    assert dec.schedule == schedule
    dec.prepare(s.lattices, beam)
    dec.run(1.0)
    hyps, out = dec.fetch()
    return hyps, out, dec.streams.stats()


# (config, n_utt, frames, beam, cache): H = 64 and 256; cache off and a wide
# beam push a level past one 128-row tile and one 512-request assign chunk
STREAM_CASES = [("a", 12, 60, 8, True), ("a", 6, 30, 32, False), ("b", 4, 40, 8, True)]


@pytest.mark.parametrize("case", STREAM_CASES)
def test_stream_schedule_matches_level_schedule(case):
    """The persistent per-stream kernel and the level-synchronous kernels in
    TF32X3: same 1-best paths, expansions and cache lookups; scores within
    the fp32 bound.  (The stream kernel puts W in the MMA A operand, so h'
    can differ in the last f32 bit and the byte-exact content dedup may
    merge a few contexts differently: table lengths agree to 0.5 %.)"""
    from paper_2007_11794_b200 import synth
    name, n_utt, T, beam, enabled = case
    s = synth.build_setup(name, n_utt=n_utt, T=T, seed=5)
    hl, ol, sl = _decode(s, "tf32x3", "level", beam, enabled)
    hs, os_, ss = _decode(s, "tf32x3", "stream", beam, enabled)
    assert np.array_equal(ol["expansions"], os_["expansions"])
    assert np.array_equal(sl[:, 0], ss[:, 0])                      # lookups
    assert np.all(np.abs(sl[:, 3] - ss[:, 3]) <= 0.005 * sl[:, 3] + 1)
    for a, b in zip(hl, hs):
        assert a.arcs == b.arcs
        assert abs(a.combined_score - b.combined_score) <= 1e-4 * T


@pytest.mark.parametrize("case", STREAM_CASES)
def test_stream_schedule_tf32x3_matches_oracle(case):
    """TF32X3 (fp32-faithful) stream decode vs the exact CPU oracle: same
    1-best arcs, expansions and lookups; combined score within 1e-4 per
    frame (north star: per-query log-probs within 1e-4)."""
    from paper_2007_11794_b200 import synth
    name, n_utt, T, beam, enabled = case
    s = synth.build_setup(name, n_utt=n_utt, T=T, seed=5)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=beam, enabled=enabled, n_threads=4)
    hyps, out, st = _decode(s, "tf32x3", "stream", beam, enabled)
    for u, (r, (lk, hi, mi)) in enumerate(ref):
        assert hyps[u].arcs == r.arcs
        assert abs(hyps[u].combined_score - r.combined_score) <= 1e-4 * T
        assert int(out["expansions"][u]) == r.expansions
    assert [int(x) for x in st[:, 0]] == [x[1][0] for x in ref]


def test_stream_schedule_tf32_single_pass():
    """Single-pass TF32 (the looser mode): runs the same traversal; scores
    within 2e-3 per frame of the oracle."""
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("a", n_utt=6, T=40, seed=5)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=8, n_threads=4)
    hyps, out, st = _decode(s, "tf32", "stream", 8)
    for u, (r, _) in enumerate(ref):
        assert abs(hyps[u].combined_score - r.combined_score) <= 2e-3 * 40
        assert int(out["expansions"][u]) == r.expansions


def test_double_buffered_pipeline_matches_single_batches():
    """BatchDecoder(n_buffers=2): prepare(i+1) / run(i+1) are queued while
    batch i is fetched on the copy stream; every batch's results equal a
    fresh single-buffer decode of the same batch."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("a", n_utt=6, T=40, seed=5)
    batches = [s.lattices] + [synth.more_lattices(s, 6, 40, seed=20 + i) for i in range(3)]
    need = max(BatchDecoder.contexts_needed(b, 8) for b in batches)
    ref = []
    for b in batches:
        d1 = BatchDecoder(s.model, s.tree, s.small_lm, 6, need, precision="tf32x3")
        d1.prepare(b, 8)
        d1.run(1.0)
        ref.append(d1.fetch()[0])
    dec = BatchDecoder(s.model, s.tree, s.small_lm, 6, need, precision="tf32x3", n_buffers=2)
    prev = dec.prepare(batches[0], 8)
    dec.run(1.0, slot=prev)
    got = []
    for b in batches[1:]:
        cur = dec.prepare(b, 8)
        dec.run(1.0, slot=cur)
        got.append(dec.fetch(slot=prev)[0])
        prev = cur
    got.append(dec.fetch(slot=prev)[0])
    for r, g in zip(ref, got):
        assert [h.arcs for h in r] == [h.arcs for h in g]
        assert [h.combined_score for h in r] == [h.combined_score for h in g]


def _random_dag(rng, n_nodes, V, lm, max_skip=3, out_deg=(1, 4)):
    """A non-layered lattice: arcs i -> j > i with skips of up to max_skip
    nodes, several finals, ids not in time order of a sausage (Kahn order
    interleaves frames), arc small-LM scores from the bigram on a random
    predecessor word (any weight is legal for the decoder)."""
    from paper_2007_11794_b200.lattice import Lattice
    from paper_2007_11794_b200.model import ngram_logprob
    src, dst, word, ac, slm = [], [], [], [], []
    for i in range(n_nodes - 1):
        for _ in range(int(rng.randint(out_deg[0], out_deg[1] + 1))):
            j = min(n_nodes - 1, i + int(rng.randint(1, max_skip + 1)))
            w = int(rng.randint(3, V))
            src.append(i); dst.append(j); word.append(w)
            ac.append(-abs(float(rng.normal(1.0, 0.7))))
            slm.append(ngram_logprob(lm, [int(rng.randint(1, V))], w))
    finals = sorted({n_nodes - 1, n_nodes - 2})
    return Lattice(0, finals, src=np.array(src), dst=np.array(dst), word=np.array(word),
                   acoustic=np.array(ac), smalllm=np.array(slm))


@pytest.mark.parametrize("schedule,precision", [("level", "fp64"), ("stream", "tf32x3")])
def test_ragged_and_non_layered_batch_vs_oracle(schedule, precision):
    """Edge cases in one batch: utterances of 1, 2, 5, 17 and 40 frames next
    to random non-layered DAGs (skip arcs, several finals, out-degree up to
    4).  fp64 level schedule: exact 1-best / counters, scores within 1e-9;
    TF32X3 stream schedule: same 1-best, scores within 1e-4 per arc."""
    from paper_2007_11794_b200 import synth
    base = synth.build_setup("a", n_utt=1, T=5, seed=2)
    rng = np.random.RandomState(12)
    lats = []
    for T in (1, 2, 5, 17, 40):
        lats += synth.more_lattices(base, 1, T, seed=100 + T)
    for n in (6, 15, 33):
        lats.append(_random_dag(rng, n, base.model.vocab_size, base.small_lm))
    s = synth.Setup("ragged", base.model, base.tree, base.small_lm, lats, 8, 3)
    for beam in (3, 8):
        ref = O.decode_many(s.model, s.tree, s.small_lm, lats, beam=beam, n_threads=4)
        hyps, out, st = _decode(s, precision, schedule, beam)
        for u, (r, (lk, hi, mi)) in enumerate(ref):
            assert hyps[u].arcs == r.arcs, (u, beam)
            tol = TOL if precision == "fp64" else 1e-4 * max(1, len(r.arcs))
            assert abs(hyps[u].combined_score - r.combined_score) <= tol
            assert int(out["expansions"][u]) == r.expansions
            if precision == "fp64":
                assert hyps[u].end_context == r.end_context
        assert [int(x) for x in st[:, 0]] == [x[1][0] for x in ref]
        if precision == "fp64":
            assert [int(x) for x in st[:, 2]] == [x[1][2] for x in ref]


def test_config_c_geometry_stream_decode_vs_oracle():
    """H = 512, V = 65,536 (config c/e geometry): stream schedule TF32X3 vs
    the exact oracle on 3 utterances x 25 frames."""
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("c", n_utt=3, T=25, seed=9)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=8, n_threads=3)
    hyps, out, st = _decode(s, "tf32x3", "stream", 8)
    for u, (r, (lk, hi, mi)) in enumerate(ref):
        assert hyps[u].arcs == r.arcs
        assert abs(hyps[u].combined_score - r.combined_score) <= 1e-4 * 25
        assert int(out["expansions"][u]) == r.expansions


@pytest.mark.parametrize("schedule,precision", [("level", "fp64"), ("stream", "tf32x3")])
def test_lattice_out_contains_the_onthefly_best_path(schedule, precision):
    """Lattice-out: the rescored pruned state lattice is a
    DAG whose best path under first-pass weights (acoustic + lm_weight *
    rescored LM) is the on-the-fly 1-best -- same input arcs, same score --
    and every state's score is its parent's plus the arc weight."""
    from paper_2007_11794_b200 import nbest, synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("a", n_utt=5, T=30, seed=21)
    lm_w = 0.8
    need = BatchDecoder.contexts_needed(s.lattices, s.beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision=precision,
                       schedule=schedule, lattice_out=True)
    dec.prepare(s.lattices, s.beam)
    dec.run(lm_w)
    hyps, _ = dec.fetch()
    lats = dec.fetch_lattices()
    for u, (h, lo) in enumerate(zip(hyps, lats)):
        assert lo.n_arcs > len(h.arcs)
        assert lo.n_arcs <= s.beam * s.lattices[u].n_arcs
        best = nbest(lo, 1, lm_weight=lm_w)[0]
        assert abs(best.combined_score - h.combined_score) <= 1e-9 * max(1.0, abs(h.combined_score))
        assert tuple(int(lo.arc_ref[a]) for a in best.arcs) == h.arcs
