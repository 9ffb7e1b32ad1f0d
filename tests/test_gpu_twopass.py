"""Two-pass rescoring on the B200 (decoder.py:180-274) against the
reference's outputs (tests/golden/twopass.npz) and the CPU oracle.

Bounds (written here):
* fp64 mode: per-hypothesis LM score |d| <= 1e-9 (HS float64 sums differ from
  the reference only in summation order, ~1e-13 per word; the hybrid
  interpolation uses CUDA exp/log), winner index identical.
* tf32x3 mode (tcgen05 recurrent update, f32 HS partials): per-hypothesis
  |d| <= 2e-5 per scored word; the winner is identical unless the reference's
  top two are closer than that bound.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O
from test_twopass import MODES, _blocks

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _lists(tp, small, config_a):
    from paper_2007_11794_b200 import nbest
    out = []
    for key, lat, model, tree, lm in _blocks(tp, small, config_a):
        hyps = nbest(lat, int(tp[f"{key}_n"]), float(tp[f"{key}_lmw"]))
        ns = tp[f"{key}_per_hyp_lm"].shape[0]
        out.append((key, hyps[:ns], model, tree, lm))
    return out


def test_twopass_matches_reference_golden(tp, small, config_a):
    from paper_2007_11794_b200 import TwopassPlan
    for key, hyps, model, tree, lm in _lists(tp, small, config_a):
        lmw = float(tp[f"{key}_lmw"])
        plan = TwopassPlan(model, tree, lm, [hyps])
        for mi, (mode, lam) in enumerate(MODES):
            plan.run(mode, lam, lmw, "fp64", use_graph=(mi % 2 == 0))
            lmv, comb, best = plan.fetch()
            row = tp[f"{key}_best"][mi]
            assert int(best[0]) == int(row[0]), (key, mode, lam)
            assert abs(lmv[best[0]] - row[1]) <= TOL and abs(comb[best[0]] - row[2]) <= TOL
            if (mode, lam) == ("rnnlm", 0.5):
                assert np.abs(lmv - tp[f"{key}_per_hyp_lm"][:, 0]).max() <= TOL, key
            if (mode, lam) == ("hybrid", 0.3):
                assert np.abs(lmv - tp[f"{key}_per_hyp_lm"][:, 1]).max() <= TOL, key


def test_twopass_batch_equals_single_lists(tp, small, config_a):
    """All lists in one device pass (merged tries, one level loop) give the
    per-list results; the drop-in entry point agrees too."""
    from paper_2007_11794_b200 import rescore_twopass, rescore_twopass_batch
    groups = {}
    for key, hyps, model, tree, lm in _lists(tp, small, config_a):
        groups.setdefault(id(model), []).append((key, hyps, model, tree, lm))
    for items in groups.values():
        _, _, model, tree, lm = items[0]
        lists = [h for _, h, *_ in items]
        for mode, lam in MODES:
            batch = rescore_twopass_batch(lists, mode, model, tree, lm, lam, 1.0)
            for (key, hyps, *_), b in zip(items, batch):
                one = rescore_twopass(hyps, mode, model, tree, lm, lam, 1.0)
                assert b.arcs == one.arcs and b.lm_score == one.lm_score, key


def test_twopass_reference_properties(small):
    """tests/test_decoder.py:167-212 on the device path."""
    from paper_2007_11794_b200 import nbest, rescore_twopass
    d, gm, lats = small
    model, tree, bigram = gm.model, gm.tree, gm.lm
    single = nbest(lats[3], 1)
    best = rescore_twopass(single, "rnnlm", model, tree, bigram)
    assert best.arcs == single[0].arcs and best.words == single[0].words
    hyps = nbest(lats[4], 8)
    best = rescore_twopass(hyps, "hybrid", model, tree, bigram, interp_weight=1.0)
    assert best.words == hyps[0].words
    assert abs(best.combined_score - hyps[0].combined_score) <= 1e-9
    hyps = nbest(lats[5], 5)
    for lam in (0.0, 0.3, 1.0):
        b = rescore_twopass(hyps, "hybrid", model, tree, bigram, interp_weight=lam)
        assert b.words in {h.words for h in hyps}
    with pytest.raises(ValueError):
        rescore_twopass([], "rnnlm", model, tree, bigram)
    with pytest.raises(ValueError):
        rescore_twopass(hyps, "bogus", model, tree, bigram)


def _oracle_lists(setup, n):
    from paper_2007_11794_b200 import nbest_batch
    lists = nbest_batch(setup.lattices, n, 1.0)
    om, og = O.OracleModel(setup.model, setup.tree), O.OracleNgram(setup.small_lm)
    return lists, om, og


@pytest.mark.parametrize("cfg", ["b", "c"])
def test_twopass_config_sizes_vs_oracle(cfg):
    """Config (b) / (c) models (V=20k H=256 / V=64k H=512), 4 utterances x 40
    frames, 30-best: fp64 mode vs the oracle, tensor-core mode within bound."""
    from paper_2007_11794_b200 import TwopassPlan, synth
    s = synth.build_setup(cfg, n_utt=4, T=40, seed=7)
    lists, om, og = _oracle_lists(s, 30)
    plan = TwopassPlan(s.model, s.tree, s.small_lm, lists)
    info = plan.info()
    assert info["trie_nodes"] < info["words"]          # prefixes are shared
    for mode, lam in (("rnnlm", 0.5), ("hybrid", 0.4)):
        want = [O.twopass(om, og, [h.words for h in l], [h.acoustic_score for h in l], mode, lam)
                for l in lists]
        plan.run(mode, lam, 1.0, "fp64")
        lmv, comb, best = plan.fetch()
        ref_lm = np.concatenate([w[0] for w in want])
        assert np.abs(lmv - ref_lm).max() <= TOL
        assert [int(b) for b in best] == [w[2] for w in want]
        plan.run(mode, lam, 1.0, "tf32x3")
        lm3, comb3, best3 = plan.fetch()
        words = np.array([len(h.words) for l in lists for h in l])
        assert np.all(np.abs(lm3 - ref_lm) <= 2e-5 * np.maximum(words, 1))
        for u, w in enumerate(want):
            c = np.sort(w[1])[::-1]
            if len(c) < 2 or c[0] - c[1] > 4e-5 * words.max():
                assert int(best3[u]) == w[2]
