"""Capacity-bounded RescoreCache on the device (cache.py:61-137, LFU with LRU
tie-break) against the reference's own outputs (tests/golden/lfu.npz, the
acceptance crit-8 recipe tests/test_acceptance.py:227-282) and the oracle:
per-utterance lookups / hits / misses / evictions / resident entries exact,
decodes unchanged (fp64: combined score within 1e-9, same end context)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_lattice
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _stack(gm, cap):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack
    m = gm.model
    return RescoreStack(model=m, tree=gm.tree,
                        table=IndexTable(m.hidden_size, m.maxent_order, device_capacity=1 << 14),
                        cache=RescoreCache(capacity_bytes=cap))


def test_bounded_cache_decode_matches_reference(golden, small):
    from paper_2007_11794_b200 import rescore_onthefly, reset_utterance
    _, gm, _ = small
    d = golden("lfu")
    lats = {int(i): golden_lattice(d, f"t{int(i)}_") for i in set(d["utt_template"].tolist())}
    for ci, cap in enumerate(d["capacities"]):
        for retain in (True, False):
            st = _stack(gm, int(cap))
            want = d[f"c{ci}_r{int(retain)}"]
            for i, t in enumerate(d["utt_template"]):
                hyp, rep = rescore_onthefly(lats[int(t)], gm.lm, st, beam=6)
                s = st.cache.stats()
                got = (s.lookups, s.hits, s.misses, s.evictions, len(st.cache), len(st.table))
                assert got == tuple(int(x) for x in want[i, :6]), (int(cap), retain, i, got, want[i])
                assert abs(hyp.combined_score - want[i, 6]) <= 1e-9
                assert hyp.end_context == int(want[i, 7])
                assert st.cache.resident_bytes == len(st.cache) * 32
                reset_utterance(st.cache, st.table, retain=retain)
            cum = st.cache.cumulative_stats()
            assert [cum.lookups, cum.hits, cum.misses, cum.evictions] == \
                list(d[f"c{ci}_r{int(retain)}_cum"])


def test_bounded_cache_trace_matches_reference(golden, small):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, rnnlm_prob_trace
    _, gm, _ = small
    d = golden("lfu")
    trace = [(int(w), int(p)) for w, p in d["trace"]]
    for cap in (32 * 40, 32 * 300):
        table = IndexTable(16, 3, device_capacity=4096)
        cache = RescoreCache(capacity_bytes=cap)
        p, succ, hit = rnnlm_prob_trace(cache, table, gm.model, gm.tree, trace)
        s = cache.stats()
        assert [s.lookups, s.hits, s.misses, s.evictions, len(cache), len(table)] == \
            list(d[f"trace_cap{cap}"])
        assert list(hit.astype(int)) == list(d[f"trace_cap{cap}_hits"])
        assert list(succ) == list(d[f"trace_cap{cap}_succ"])


def test_set_capacity_shrinks_like_reference(golden, small):
    """cache.py:130-137: shrinking evicts at once; 0 removes the bound."""
    from paper_2007_11794_b200 import rescore_onthefly, reset_utterance
    _, gm, lats = small
    st = _stack(gm, 32 * 200)
    ost = O.OracleStack(gm.model, gm.tree, capacity_bytes=32 * 200)
    og = O.OracleNgram(gm.lm)
    for i, cap in enumerate((None, 32 * 50, None, 32 * 10, 32 * 400, None)):
        if cap is not None:
            st.cache.set_capacity(cap)
            ost.set_capacity(cap)
        lat = lats[i]
        hyp, _ = rescore_onthefly(lat, gm.lm, st, beam=4)
        r = ost.rescore_onthefly(lat, og, beam=4)
        s, o = st.cache.stats(), ost.stats()
        assert (s.lookups, s.hits, s.misses, s.evictions, len(st.cache)) == \
            (o.lookups, o.hits, o.misses, o.evictions, o.entries), i
        assert hyp.arcs == r.arcs
        reset_utterance(st.cache, st.table, retain=True)
        ost.reset(True)


@pytest.mark.parametrize("schedule,precision", [("level", "fp64"), ("stream", "tf32x3")])
def test_bounded_cache_batch_decoder_vs_oracle(schedule, precision):
    """Many utterances at once (one stream each, fresh per run), bounded
    cache: counters per stream equal the oracle's."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("a", n_utt=6, T=40, seed=8)
    cap = 32 * 300
    need = BatchDecoder.contexts_needed(s.lattices, s.beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision=precision,
                       schedule=schedule, capacity_bytes=cap)
    dec.prepare(s.lattices, s.beam)
    og = O.OracleNgram(s.small_lm)
    om = O.OracleModel(s.model, s.tree)
    for _ in range(2):                       # runs are independent (retain=False between runs)
        dec.run(1.0)
        hyps, out = dec.fetch()
        st = dec.streams.stats()
        cs = dec.streams.cache_stats()
        for u, lat in enumerate(s.lattices):
            ost = O.OracleStack(om, None, capacity_bytes=cap)
            r = ost.rescore_onthefly(lat, og, beam=s.beam)
            o = ost.stats()
            assert hyps[u].arcs == r.arcs
            assert (int(st[u, 0]), int(st[u, 1]), int(st[u, 2]), int(cs[u, 0]), int(cs[u, 2])) == \
                (o.lookups, o.hits, o.misses, o.evictions, o.entries), u


def test_bounded_cache_roll_and_clear_match_oracle(small):
    """roll_stats and clear on a capacity-bounded cache (cache.py:156-158,
    :136-140): decode, roll, decode (table and cache retained), clear the
    cache only, decode -- window / cumulative counters, evictions, resident
    entries and table length after every step equal the oracle's."""
    from paper_2007_11794_b200 import rescore_onthefly
    s, gm, lats = small
    for cap in (32 * 40, 32 * 400):
        st = _stack(gm, cap)
        ref = O.OracleStack(gm.model, gm.tree, capacity_bytes=cap)
        og = O.OracleNgram(gm.lm)
        for step, lat in enumerate([lats[0], lats[0], lats[0]]):
            hyp, _ = rescore_onthefly(lat, gm.lm, st, beam=6)
            r = ref.rescore_onthefly(lat, og, beam=6)
            assert hyp.arcs == r.arcs and abs(hyp.combined_score - r.combined_score) <= 1e-9
            a, c, o = st.cache.stats(), st.cache.cumulative_stats(), ref.stats()
            got = (a.lookups, a.hits, a.misses, len(st.cache), len(st.table), c.lookups, c.hits, c.misses)
            assert got == (o.lookups, o.hits, o.misses, o.entries, o.table_len,
                           o.cum_lookups, o.cum_hits, o.cum_misses), (cap, step, got, o)
            assert a.evictions == o.evictions, (cap, step)
            if step == 0:
                st.cache.roll_stats()
                ref.roll_stats()
                assert st.cache.stats().lookups == 0 and st.cache.stats().evictions == 0
            elif step == 1:
                ev_before = st.cache.cumulative_stats().evictions
                st.cache.clear()
                ref.cache_clear()
                assert len(st.cache) == 0 and st.cache.cumulative_stats().evictions == ev_before
