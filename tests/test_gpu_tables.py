"""Container-level IndexTable / RescoreCache operations on the device tables
(tables.cuh) against the reference (tests/golden/tables.npz, made by
tests/golden/make_golden_tables.py): IndexTable.encode (context_table.py:
76-89), rnnlm_prob from encoded indices (cache.py:165-182), RescoreCache.get
/ put (cache.py:80-108) on enabled and disabled caches."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_encode_then_rnnlm_prob_matches_reference(golden, small):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, rnnlm_prob
    from paper_2007_11794_b200.model import RnnlmContext
    d = golden("tables")
    _, gm, _ = small
    table, cache = IndexTable(16, 3), RescoreCache()
    table.bind(gm.model, gm.tree, cache)
    got = [table.encode(RnnlmContext(h, tuple(int(x) for x in hh[:L])))
           for h, hh, L in zip(d["enc_h"], d["enc_hist"], d["enc_len"])]
    assert got == [int(x) for x in d["enc_idx"]]
    assert len(table) == int(d["table_len"])
    for i in (0, 5, len(got) - 1):                       # stored bytes come back
        ctx = table.decode(got[i])
        assert np.array_equal(ctx.hidden.view(np.uint32), d["enc_h"][i].view(np.uint32))
        assert ctx.history == tuple(int(x) for x in d["enc_hist"][i][:d["enc_len"][i]])
    for (w, c), p, cn in zip(d["probe"], d["probe_p"], d["probe_c"]):
        v = rnnlm_prob(cache, table, gm.model, gm.tree, int(w), int(c))
        assert abs(v.p - p) <= 1e-12
        assert v.c_next == int(cn)
    assert len(table) == int(d["table_len2"])


def test_encode_validation(small):
    from paper_2007_11794_b200 import IndexTable
    from paper_2007_11794_b200.model import RnnlmContext
    _, gm, _ = small
    t = IndexTable(16, 3)
    with pytest.raises(ValueError, match="bind"):
        t.encode(RnnlmContext(np.zeros(16, np.float32), ()))
    t.bind(gm.model, gm.tree)
    with pytest.raises(ValueError):
        t.encode(RnnlmContext(np.zeros(8, np.float32), ()))
    with pytest.raises(ValueError):
        t.encode(RnnlmContext(np.zeros(16, np.float32), (1, 2, 3, 4)))
    assert t.encode(RnnlmContext(np.zeros(16, np.float32), ())) == 1      # the zero context is not index 0


@pytest.mark.parametrize("tag", ["on", "off"])
def test_cache_get_put_sequence_matches_reference(golden, small, tag):
    from paper_2007_11794_b200 import CacheValue, IndexTable, RescoreCache
    d = golden("tables")
    _, gm, _ = small
    cache = RescoreCache(enabled=tag == "on")
    IndexTable(16, 3).bind(gm.model, gm.tree, cache)
    for (op, c, w, cn), p, rp, rc in zip(d[f"ops_{tag}"], d[f"ops_{tag}_p"], d[f"res_{tag}_p"], d[f"res_{tag}_c"]):
        if op == 0:
            v = cache.get((int(c), int(w)))
            if rc < 0:
                assert v is None
            else:
                assert v is not None and v.p == rp and v.c_next == int(rc)
        else:
            cache.put((int(c), int(w)), CacheValue(float(p), int(cn)))
    s = cache.stats()
    assert [s.lookups, s.hits, s.misses, len(cache)] == [int(x) for x in d[f"stats_{tag}"]]


def test_direct_get_put_refused_on_bounded_cache(small):
    from paper_2007_11794_b200 import CacheValue, IndexTable, RescoreCache
    _, gm, _ = small
    cache = RescoreCache(capacity_bytes=32 * 8)
    IndexTable(16, 3).bind(gm.model, gm.tree, cache)
    with pytest.raises(ValueError, match="capacity-bounded"):
        cache.get((0, 5))
    with pytest.raises(ValueError, match="capacity-bounded"):
        cache.put((0, 5), CacheValue(-1.0, 1))


def test_roll_stats_and_clear_match_reference(golden, small):
    from paper_2007_11794_b200 import CacheValue, IndexTable, RescoreCache
    d = golden("tables")
    _, gm, _ = small
    cache = RescoreCache()
    IndexTable(16, 3).bind(gm.model, gm.tree, cache)
    for (op, c, w, cn), p in zip(d["ops_on"], d["ops_on_p"]):
        if op == 0:
            cache.get((int(c), int(w)))
        else:
            cache.put((int(c), int(w)), CacheValue(float(p), int(cn)))
    cache.roll_stats()
    s1, cu = cache.stats(), cache.cumulative_stats()
    cache.clear()
    n_after = len(cache)
    a = d["after_ops"]
    assert [s1.lookups, s1.hits, s1.misses, cu.lookups, cu.hits, cu.misses, n_after] == [int(x) for x in a[:7]]
    k = (int(d["ops_on"][0][1]), int(d["ops_on"][0][2]))
    assert (cache.get(k) is None) == bool(a[7])
    s2 = cache.stats()
    assert [s2.lookups, s2.misses] == [int(a[8]), int(a[9])]
