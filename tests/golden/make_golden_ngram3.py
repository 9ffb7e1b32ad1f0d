"""Golden fixture for an ORDER-3 small LM on the device (verdict r01 item 7),
generated from the REFERENCE implementation (otflm) in the build container:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ngram3.py

ngram3.npz
  * a Kneser-Ney trigram trained by ``train_ngram`` (ngram.py) on a Zipfian
    corpus (synth.py), round-tripped through ``save_arpa`` / ``load_arpa``
    (so back-off weights that the ARPA file omits are missing), and some
    back-off entries deleted on purpose; its tables flattened;
  * 4000 (<s>-padded 2-word context, word) queries -- seen, unseen and
    partially seen contexts -- with ``ngram_logprob``'s float64 result
    (ngram.py:161-179);
  * a decode with that trigram as the small LM (decoder.py:86-90 allows
    order - 1 <= maxent_order = 3): a breadth-3 ``generate_lattice`` over a
    40-word reference sentence, a ``RnnlmModel.new`` model with a random
    output layer, ``rescore_onthefly`` at beam 8: the 1-best, scores, end
    context, expansions and cache / table counters.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from otflm.cache import RescoreCache  # noqa: E402
from otflm.codec import TransferLedger  # noqa: E402
from otflm.context_table import IndexTable  # noqa: E402
from otflm.decoder import RescoreStack, rescore_onthefly  # noqa: E402
from otflm.huffman import build_huffman  # noqa: E402
from otflm.lattice import generate_lattice  # noqa: E402
from otflm.ngram import load_arpa, ngram_logprob, save_arpa, train_ngram  # noqa: E402
from otflm.rnnlm import RnnlmModel  # noqa: E402
from otflm.synth import zipfian_corpus  # noqa: E402
from otflm.vocab import build_vocabulary  # noqa: E402

from oracle.oracle import ngram_flat  # noqa: E402  (flattening only; test infrastructure)

OUT = Path(__file__).resolve().parent / "ngram3.npz"


def main():
    corpus = zipfian_corpus(3000, 300, seed=11)
    vocab = build_vocabulary(corpus)
    lm = train_ngram(corpus, vocab, 3, smoothing="kneser-ney")
    with tempfile.TemporaryDirectory() as d:
        save_arpa(lm, vocab, Path(d) / "lm.arpa")
        lm = load_arpa(Path(d) / "lm.arpa", vocab)
    # missing back-offs: drop every 7th order-2 back-off entry
    bo2 = sorted(k for k in lm.backoffs if len(k) == 2)
    for k in bo2[::7]:
        del lm.backoffs[k]
    V = len(vocab)
    bos = vocab.sentence_begin_id
    rng = np.random.default_rng(5)
    seen = sorted(k for k in lm.probs if len(k) == 3)
    ctx = np.empty((4000, 2), np.int32)
    w = np.empty(4000, np.int32)
    for i in range(4000):
        kind = i % 4
        if kind == 0:                     # a stored trigram
            k = seen[int(rng.integers(len(seen)))]
            ctx[i] = k[:2]; w[i] = k[2]
        elif kind == 1:                   # <s>-padded short history
            ctx[i] = (bos, int(rng.integers(3, V))); w[i] = int(rng.integers(3, V))
        elif kind == 2:                   # stored context, unseen continuation
            k = seen[int(rng.integers(len(seen)))]
            ctx[i] = k[:2]; w[i] = int(rng.integers(3, V))
        else:                             # random context
            ctx[i] = rng.integers(3, V, size=2); w[i] = int(rng.integers(3, V))
    expect = np.array([ngram_logprob(lm, [int(a), int(b)], int(x)) for (a, b), x in zip(ctx, w)])
    order, (n_p, kp, lp, vp), (n_b, kb, lb, vb) = ngram_flat(lm)
    # a decode with the trigram small LM
    model = RnnlmModel.new(V, hidden_size=48, maxent_order=3, maxent_table_bits=16, seed=4)
    r = np.random.RandomState(8)
    model.node_vectors[:] = r.uniform(-0.3, 0.3, model.node_vectors.shape).astype(np.float32)
    model.maxent_table[:] = r.uniform(-0.1, 0.1, model.maxent_size).astype(np.float32)
    tree = build_huffman(vocab)
    ref_words = [int(x) for x in rng.integers(3, V, size=40)]
    lat = generate_lattice(ref_words, vocab, lm, 3, noise_seed=9)
    st = RescoreStack(model=model, tree=tree, table=IndexTable(model.hidden_size, 3), cache=RescoreCache(),
                      ledger=TransferLedger())
    hyp, rep = rescore_onthefly(lat, lm, st, beam=8)
    s = st.cache.stats()
    arcs = sorted(lat.arcs, key=lambda a: a.id)
    np.savez_compressed(
        OUT, order=np.int32(order), V=np.int32(V), bos=np.int32(bos), eos=np.int32(vocab.sentence_end_id),
        pk=kp[:n_p], pl=lp[:n_p], pv=vp[:n_p], bk=kb[:n_b], bl=lb[:n_b], bv=vb[:n_b],
        q_ctx=ctx, q_w=w, q_expect=expect,
        U=model.input_weights, W=model.recurrent_weights, NV=model.node_vectors, ME=model.maxent_table,
        seed=np.uint64(model.hash_seed), counts=np.array(vocab.counts, np.int64),
        lat_src=np.array([a.src for a in arcs], np.int64), lat_dst=np.array([a.dst for a in arcs], np.int64),
        lat_word=np.array([a.word for a in arcs], np.int32), lat_ac=np.array([a.acoustic for a in arcs]),
        lat_slm=np.array([a.smalllm for a in arcs]), lat_start=np.int64(lat.start),
        lat_finals=np.array(sorted(lat.finals), np.int64),
        arcs=np.array(hyp.arcs, np.int32),
        result=np.array([hyp.combined_score, hyp.acoustic_score, hyp.lm_score, hyp.end_context,
                         rep.expansions, s.lookups, s.hits, s.misses, len(st.table)], np.float64),
        produced_by=np.array("otflm.ngram.train_ngram/save_arpa/load_arpa/ngram_logprob + "
                             "otflm.decoder.rescore_onthefly (order-3 small LM)"))
    print(f"ngram3: {n_p} n-grams, {n_b} back-offs, V={V}; decode {rep.expansions} requests, "
          f"1-best {len(hyp.arcs)} arcs")


if __name__ == "__main__":
    main()
