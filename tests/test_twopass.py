"""Two-pass rescoring: nbest (decoder.py:180-230) and
rescore_twopass (decoder.py:243-274).

CPU tests pin the oracle restatement bit-exactly against the reference's
own outputs (tests/golden/twopass.npz, made by tests/golden/make_golden.py)
and mirror the reference's nbest / twopass tests (tests/test_decoder.py:
134-225).  GPU tests run the product path (host n-best search in
libotflm_b200.so + the device trie-level RNNLM scorer) against the same
vectors and the oracle."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GoldenModel, golden_lattice
from oracle import oracle as O

MODES = [("rnnlm", 0.5), ("hybrid", 0.0), ("hybrid", 0.3), ("hybrid", 1.0)]


def _blocks(tp, small, config_a):
    d, gm, lats = small
    for li in range(12):
        yield f"l{li}", lats[li], gm.model, gm.tree, gm.lm
    _, model, tree, lm, lat = config_a
    yield "a", lat, model, tree, lm


def _check_nbest(tp, key, hyps):
    assert len(hyps) == len(tp[f"{key}_hyp_len"])
    assert [len(h.arcs) for h in hyps] == list(tp[f"{key}_hyp_len"])
    assert np.array_equal(np.concatenate([np.asarray(h.arcs) for h in hyps]), tp[f"{key}_hyp_arcs"])
    sc = np.array([[h.combined_score, h.acoustic_score, h.lm_score] for h in hyps])
    assert np.array_equal(sc, tp[f"{key}_hyp_scores"])


def test_oracle_nbest_matches_reference(tp, small, config_a):
    for key, lat, *_ in _blocks(tp, small, config_a):
        hyps = O.nbest(lat, int(tp[f"{key}_n"]), float(tp[f"{key}_lmw"]))
        _check_nbest(tp, key, hyps)
        # a shorter list is a prefix of a longer one (same search order)
        short = O.nbest(lat, 3, float(tp[f"{key}_lmw"]))
        assert [h.arcs for h in short] == [h.arcs for h in hyps[:3]]


def test_oracle_twopass_matches_reference(tp, small, config_a):
    for key, lat, model, tree, lm in _blocks(tp, small, config_a):
        om, og = O.OracleModel(model, tree), O.OracleNgram(lm)
        lmw = float(tp[f"{key}_lmw"])
        hyps = O.nbest(lat, int(tp[f"{key}_n"]), lmw)
        ns = tp[f"{key}_per_hyp_lm"].shape[0]
        ws = [h.words for h in hyps[:ns]]
        ac = [h.acoustic_score for h in hyps[:ns]]
        for mi, (mode, lam) in enumerate(MODES):
            lmv, comb, b = O.twopass(om, og, ws, ac, mode, lam, lmw)
            row = tp[f"{key}_best"][mi]
            assert (b, lmv[b], comb[b]) == (int(row[0]), row[1], row[2]), (key, mode, lam)
            if (mode, lam) == ("rnnlm", 0.5):
                assert np.array_equal(lmv, tp[f"{key}_per_hyp_lm"][:, 0])
            if (mode, lam) == ("hybrid", 0.3):
                assert np.array_equal(lmv, tp[f"{key}_per_hyp_lm"][:, 1])


def test_oracle_nbest_errors(small):
    _, _, lats = small
    with pytest.raises(ValueError):
        O.nbest(lats[0], 0)


def test_product_nbest_matches_reference(tp, small, config_a):
    """The product n-best search (host C++ in libotflm_b200.so; no GPU needed)."""
    from paper_2007_11794_b200 import nbest, nbest_batch
    blocks = list(_blocks(tp, small, config_a))
    for key, lat, *_ in blocks:
        _check_nbest(tp, key, nbest(lat, int(tp[f"{key}_n"]), float(tp[f"{key}_lmw"])))
    # batch form: utterance-parallel threads, same lists
    small_blocks = [b for b in blocks if b[0] != "a" and float(tp[f"{b[0]}_lmw"]) == 1.0]
    lists = nbest_batch([b[1] for b in small_blocks], 60, 1.0, n_threads=4)
    for (key, *_), hyps in zip(small_blocks, lists):
        _check_nbest(tp, key, hyps)


def test_product_nbest_errors(small):
    from paper_2007_11794_b200 import nbest
    from paper_2007_11794_b200.lattice import Lattice
    _, _, lats = small
    with pytest.raises(ValueError):
        nbest(lats[0], 0)
    dead = Lattice(0, [5], src=np.array([0, 1]), dst=np.array([1, 2]), word=np.array([3, 4]),
                   acoustic=np.array([-1.0, -1.0]), smalllm=np.array([-1.0, -1.0]))
    with pytest.raises(ValueError):
        nbest(dead, 3)
