"""Big beams and wide lattices on the level schedule: the CTA-per-node expand
(k_expand_big: hash recombination + CTA ranking, decoder.py:131-149) and the
multi-CTA ordered assign (k_asg_*: len+1 numbering over chunks,
context_table.py:83-86; cache claims cache.py:99-109).

Both are checked for identity with the reference: (1) forced onto every node
and every (level, stream) range of the reference's own golden decodes
(OTFLM_EXPAND_BIG_MIN=0, OTFLM_ASSIGN_BIG=0 -- the thresholds are read at
plan creation); (2) at their default thresholds on beam-64 decodes against
the oracle (arcs, expansions, end context, cache counters, table length;
scores within 1e-9), FP64 and EXACT precision.  The fat variant
(test_gpu_fullsize.py) runs both paths by default."""

from __future__ import annotations

import pytest

from conftest import small_results
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture
def forced_big(monkeypatch):
    monkeypatch.setenv("OTFLM_EXPAND_BIG_MIN", "0")
    monkeypatch.setenv("OTFLM_ASSIGN_BIG", "0")


def test_forced_big_paths_match_reference_golden(small, forced_big):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack, rescore_onthefly
    d, gm, lats = small
    beams = [int(b) for b in d["beams"]]
    n = 0
    for row in small_results(d):
        li, bi, en = int(row[0]), int(row[1]), int(row[2])
        m = gm.model
        st = RescoreStack(model=m, tree=gm.tree, table=IndexTable(m.hidden_size, m.maxent_order,
                                                                  device_capacity=1 << 17),
                          cache=RescoreCache(enabled=bool(en)))
        hyp, rep = rescore_onthefly(lats[li], gm.lm, st, lm_weight=1.0 if li % 2 else 0.7, beam=beams[bi])
        assert hyp.arcs == tuple(d[f"l{li}_b{bi}_e{en}_arcs"]), (li, bi, en)
        assert abs(hyp.combined_score - row[3]) <= TOL
        assert hyp.end_context == int(row[6])
        assert rep.expansions == int(row[7])
        s = st.cache.stats()
        assert (s.lookups, s.hits, s.misses) == tuple(int(x) for x in row[8:11])
        assert len(st.table) == int(row[11])
        n += 1
    assert n >= 200


def test_forced_big_paths_config_a_golden(config_a, forced_big):
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


def _decode_vs_oracle(s, beam, precision, schedule="level"):
    from paper_2007_11794_b200.rescore import BatchDecoder
    need = BatchDecoder.contexts_needed(s.lattices, beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision=precision, schedule=schedule)
    dec.prepare(s.lattices, beam)
    dec.run(1.0)
    hyps, out = dec.fetch()
    st = dec.streams.stats()
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=beam)
    for u, (r, (lk, hi, mi)) in enumerate(ref):
        assert hyps[u].arcs == r.arcs, (precision, u)
        assert abs(hyps[u].combined_score - r.combined_score) <= TOL
        assert int(out["expansions"][u]) == r.expansions and hyps[u].end_context == r.end_context
        assert (int(st[u, 0]), int(st[u, 1]), int(st[u, 2]), int(st[u, 3])) == (lk, hi, mi, r.table_len)
    return dec


@pytest.mark.parametrize("precision", ["fp64", "exact"])
def test_beam64_level_schedule_vs_oracle(precision):
    """Config-b geometry, beam 64 (192 arrival slots per node -> k_expand_big
    at its default threshold)."""
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("b", n_utt=6, T=60, seed=11)
    _decode_vs_oracle(s, 64, precision)


@pytest.mark.parametrize("precision", ["fp64", "exact"])
def test_wide_lattice_multi_cta_assign_vs_oracle(precision, monkeypatch):
    """Breadth 8, beam 32 (8 x 32 x 8 = 2k requests per stream level) with
    the multi-CTA assign at a lowered threshold (1024), so every range of the
    level spans several chunks."""
    from paper_2007_11794_b200 import synth
    monkeypatch.setenv("OTFLM_ASSIGN_BIG", "1024")
    import dataclasses
    s = synth.build_setup("b", n_utt=1, T=4, seed=5)
    s = dataclasses.replace(s, breadth=8)
    s = dataclasses.replace(s, lattices=synth.more_lattices(s, 3, 30, seed=5), beam=32)
    _decode_vs_oracle(s, 32, precision)
