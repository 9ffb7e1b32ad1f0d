"""An ORDER-3 small LM on the device (reference ngram.py:161-179, decoder.py:
86-90): the device open-addressing n-gram hash against the reference's own
``ngram_logprob`` values, and a whole decode with the trigram small LM
against the reference's ``rescore_onthefly`` -- both from
tests/golden/ngram3.npz (tests/golden/make_golden_ngram3.py: a Kneser-Ney
trigram trained and ARPA-round-tripped by the reference, some back-offs
removed; seen, unseen and partially seen contexts)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
G = np.load(Path(__file__).parent / "golden" / "ngram3.npz")


def _lm():
    from paper_2007_11794_b200.model import ngram_from_arrays
    return ngram_from_arrays(G["order"], G["V"], G["bos"], G["eos"], G["pk"], G["pl"], G["pv"],
                             G["bk"], G["bl"], G["bv"])


def _model():
    from paper_2007_11794_b200.model import RnnlmModel, build_huffman_from_counts
    U = G["U"]
    m = RnnlmModel(U.shape[1], U.shape[0], 3, G["ME"].shape[0], int(G["seed"]), U, G["W"], G["NV"], G["ME"])
    return m, build_huffman_from_counts(G["counts"])


def test_device_trigram_logprob_equals_reference():
    import torch
    from paper_2007_11794_b200 import kernels
    from paper_2007_11794_b200.device import DeviceModel, DeviceNgram
    lm = _lm()
    m, tree = _model()
    dn = DeviceNgram(lm, DeviceModel(m, tree))
    got = kernels.ngram_logprob_batch(dn, torch.from_numpy(G["q_ctx"]).cuda(),
                                      torch.from_numpy(G["q_w"]).cuda()).cpu().numpy()
    assert np.array_equal(got, G["q_expect"]), np.abs(got - G["q_expect"]).max()


@pytest.mark.parametrize("precision,schedule", [("exact", "stream"), ("fp64", "level")])
def test_decode_with_trigram_small_lm_equals_reference(precision, schedule):
    from paper_2007_11794_b200.lattice import Lattice
    from paper_2007_11794_b200.rescore import BatchDecoder
    lm = _lm()
    m, tree = _model()
    lat = Lattice(int(G["lat_start"]), G["lat_finals"].tolist(), src=G["lat_src"], dst=G["lat_dst"],
                  word=G["lat_word"], acoustic=G["lat_ac"], smalllm=G["lat_slm"])
    need = BatchDecoder.contexts_needed([lat], 8)
    dec = BatchDecoder(m, tree, lm, 1, need, precision=precision, schedule=schedule)
    dec.prepare([lat], 8)
    dec.run(1.0)
    hyps, out = dec.fetch()
    st = dec.streams.stats()
    comb, ac, lmsc, end_ctx, exp_, look, hit, miss, tlen = G["result"]
    assert list(hyps[0].arcs) == G["arcs"].tolist()
    assert abs(hyps[0].combined_score - comb) <= 1e-9 and abs(hyps[0].lm_score - lmsc) <= 1e-9
    assert hyps[0].end_context == int(end_ctx) and int(out["expansions"][0]) == int(exp_)
    assert [int(x) for x in st[0, :4]] == [int(look), int(hit), int(miss), int(tlen)]
    # and the CPU oracle agrees on the same inputs
    r = O.decode_many(m, tree, lm, [lat], beam=8, n_threads=1)[0][0]
    assert list(r.arcs) == G["arcs"].tolist()
