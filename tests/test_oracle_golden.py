"""Pin the CPU oracle (oracle/otflm_oracle.c) against vectors produced by the
reference implementation itself (tests/golden/make_golden.py).  The oracle
reproduces the reference's float64 arithmetic order, so everything here is
exact equality."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np
import pytest

from conftest import GoldenModel, golden_lattice, small_results
from oracle import oracle as O
from paper_2007_11794_b200.model import build_huffman_from_counts
from paper_2007_11794_b200 import synth


def test_feature_index_matches_reference(golden):
    fi = golden("kernels")["fi"]
    for row in fi:
        seed, k = int(row[0]), int(row[1])
        words = [int(x) for x in row[2:6]][:k]
        node, mask, want = int(row[6]), int(row[7]), int(row[8])
        assert O.feature_index(seed, k, words, node, mask) == want


def test_word_logprob_advance_all_exact(golden):
    d = golden("kernels")
    gm = GoldenModel(d)
    m, t = gm.model, gm.tree
    for i in range(len(d["q_w"])):
        L = int(d["q_hl"][i])
        hist = d["q_hist"][i, :L]
        w = int(d["q_w"][i])
        o0, o1 = t.path_offsets[w], t.path_offsets[w + 1]
        lp = O.word_logprob(d["q_h"][i], hist, t.path_nodes[o0:o1], t.path_signs[o0:o1],
                            m.node_vectors, m.maxent_table, m.maxent_order, m.hash_seed,
                            m.maxent_size - 1)
        assert lp == d["q_lp"][i]
        adv = O.advance_hidden(m.input_weights[w], m.recurrent_weights, d["q_h"][i])
        assert adv.tobytes() == d["q_adv"][i].tobytes()
    for i in range(d["q_all"].shape[0]):
        L = int(d["q_hl"][i])
        allw = O.all_word_logprobs(d["q_h"][i], d["q_hist"][i, :L], t.path_nodes, t.path_signs,
                                   t.path_offsets, m.node_vectors, m.maxent_table,
                                   m.maxent_order, m.hash_seed, m.maxent_size - 1)
        assert np.array_equal(allw, d["q_all"][i])


def test_huffman_builder_matches_reference(golden):
    d = golden("huffman")
    t = build_huffman_from_counts([5, 2, 1, 1])
    assert np.array_equal(t.path_nodes, d["pn_5211"])
    assert np.array_equal(t.path_signs, d["ps_5211"])
    assert np.array_equal(t.path_offsets, d["po_5211"])
    assert [t.code_length(w) for w in range(4)] == [1, 2, 3, 3]   # test_huffman.py:39-45
    for V in (1000, 20000, 65536):
        t = build_huffman_from_counts(synth.zipf_counts(V))
        h = hashlib.sha256()
        for a in (t.path_nodes, t.path_signs, t.path_offsets):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(d[f"sha_{V}"]), V
        if V == 1000:
            assert np.array_equal(t.path_nodes, d["pn_1000"])


def test_small_decodes_match_reference(small):
    d, gm, lats = small
    om = O.OracleModel(gm.model, gm.tree)
    og = O.OracleNgram(gm.lm)
    beams = [int(b) for b in d["beams"]]
    for row in small_results(d):
        li, bi, en = int(row[0]), int(row[1]), int(row[2])
        st = O.OracleStack(om, None, enabled=bool(en))
        lm_w = 1.0 if li % 2 else 0.7
        r = st.rescore_onthefly(lats[li], og, lm_weight=lm_w, beam=beams[bi])
        s = st.stats()
        assert r.arcs == tuple(d[f"l{li}_b{bi}_e{en}_arcs"])
        assert r.combined_score == row[3]
        assert r.acoustic_score == row[4]
        assert r.lm_score == row[5]
        assert r.end_context == int(row[6])
        assert r.expansions == int(row[7])
        assert (s.lookups, s.hits, s.misses, s.table_len) == tuple(int(x) for x in row[8:12])
        assert (s.bytes_indexed, s.bytes_full_baseline) == (int(row[12]), int(row[13]))


def test_trace_replay_matches_reference(small):
    d, gm, _ = small
    st = O.OracleStack(gm.model, gm.tree)
    succ = []
    for i, (w, parent) in enumerate(d["trace"]):
        c = 0 if parent < 0 else succ[parent]
        p, cn, _ = st.rnnlm_prob(int(w), int(c))
        succ.append(cn)
        assert p == d["trace_p"][i]
        assert cn == d["trace_c"][i]
        h, _ = st.context(cn)
        assert h.tobytes() == d["trace_h"][i].tobytes()
    s = st.stats()
    assert [s.lookups, s.hits, s.misses, s.table_len] == list(d["trace_stats"])


def test_config_a_decode_matches_reference(config_a):
    d, model, tree, lm, lat = config_a
    st = O.OracleStack(model, tree)
    r = st.rescore_onthefly(lat, lm, beam=8)
    s = st.stats()
    res = d["result"]
    assert r.arcs == tuple(d["arcs"])
    assert r.combined_score == res[0]
    assert r.end_context == int(res[3])
    assert r.expansions == int(res[4])
    assert (s.lookups, s.hits, s.misses, s.table_len) == tuple(int(x) for x in res[5:9])


def test_oracle_path_score_equals_decode_score(small):
    """decoder.py:277-292 composes to the traversal score (test_decoder.py:53-58)."""
    d, gm, lats = small
    st = O.OracleStack(gm.model, gm.tree)
    r = st.rescore_onthefly(lats[6], gm.lm, beam=1 << 30)
    assert O.path_score(gm.model, gm.tree, gm.lm, lats[6], r.arcs) == r.combined_score


def _lfu_lattices(golden):
    d = golden("lfu")
    lats = {int(i): golden_lattice(d, f"t{int(i)}_") for i in set(d["utt_template"].tolist())}
    return d, lats


def test_oracle_lfu_cache_matches_reference(golden, small):
    """Capacity-bounded RescoreCache (cache.py:61-134): the crit-8 recipe
    (tests/test_acceptance.py:227-282) -- 80 command utterances, beam 6,
    retained and reset caches -- per-utterance lookups / hits / misses /
    evictions / resident entries / table length and the decode itself."""
    _, gm, _ = small
    d, lats = _lfu_lattices(golden)
    og = O.OracleNgram(gm.lm)
    om = O.OracleModel(gm.model, gm.tree)
    for ci, cap in enumerate(d["capacities"]):
        for retain in (True, False):
            st = O.OracleStack(om, None, capacity_bytes=int(cap))
            want = d[f"c{ci}_r{int(retain)}"]
            for i, t in enumerate(d["utt_template"]):
                r = st.rescore_onthefly(lats[int(t)], og, beam=6)
                s = st.stats()
                got = (s.lookups, s.hits, s.misses, s.evictions, s.entries, s.table_len)
                assert got == tuple(int(x) for x in want[i, :6]), (cap, retain, i, got, want[i])
                assert r.combined_score == want[i, 6] and r.end_context == int(want[i, 7])
                st.reset(retain)


def test_oracle_lfu_trace_matches_reference(golden, small):
    _, gm, _ = small
    d, _ = _lfu_lattices(golden)
    for cap in (32 * 40, 32 * 300):
        st = O.OracleStack(gm.model, gm.tree, capacity_bytes=cap)
        succ, hits = [], []
        for w, parent in d["trace"]:
            c = 0 if parent < 0 else succ[parent]
            _, cn, hit = st.rnnlm_prob(int(w), int(c))
            succ.append(cn)
            hits.append(int(hit))
        s = st.stats()
        assert [s.lookups, s.hits, s.misses, s.evictions, s.entries, s.table_len] == \
            list(d[f"trace_cap{cap}"])
        assert hits == list(d[f"trace_cap{cap}_hits"])
        assert succ == list(d[f"trace_cap{cap}_succ"])


def test_oracle_and_host_ngram_with_trigram_small_lm():
    """tests/golden/ngram3.npz (reference train_ngram + ARPA round trip,
    order 3, missing back-offs): the host ngram_logprob equals the
    reference's on all 4000 queries, and the C oracle's decode with the
    trigram as small LM equals the reference's rescore_onthefly (1-best,
    score, counters, IndexTable length)."""
    from paper_2007_11794_b200.lattice import Lattice
    from paper_2007_11794_b200.model import (RnnlmModel, build_huffman_from_counts, ngram_from_arrays,
                                             ngram_logprob)
    G = np.load(Path(__file__).parent / "golden" / "ngram3.npz")
    lm = ngram_from_arrays(G["order"], G["V"], G["bos"], G["eos"], G["pk"], G["pl"], G["pv"],
                           G["bk"], G["bl"], G["bv"])
    got = [ngram_logprob(lm, [int(a), int(b)], int(w)) for (a, b), w in zip(G["q_ctx"], G["q_w"])]
    assert np.array_equal(np.array(got), G["q_expect"])
    U = G["U"]
    m = RnnlmModel(U.shape[1], U.shape[0], 3, G["ME"].shape[0], int(G["seed"]), U, G["W"], G["NV"], G["ME"])
    tree = build_huffman_from_counts(G["counts"])
    lat = Lattice(int(G["lat_start"]), G["lat_finals"].tolist(), src=G["lat_src"], dst=G["lat_dst"],
                  word=G["lat_word"], acoustic=G["lat_ac"], smalllm=G["lat_slm"])
    (r, (lk, hi, mi)), = O.decode_many(m, tree, lm, [lat], beam=8, n_threads=1)
    comb, ac, lms, end_ctx, exp_, look, hit, miss, tlen = G["result"]
    assert list(r.arcs) == G["arcs"].tolist() and r.combined_score == comb
    assert (r.end_context, r.expansions, lk, hi, mi, r.table_len) == \
        (int(end_ctx), int(exp_), int(look), int(hit), int(miss), int(tlen))
