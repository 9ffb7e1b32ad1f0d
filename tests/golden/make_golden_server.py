"""Golden fixture for the paper's search <-> rescorer boundary, produced by
the REFERENCE (otflm) in the build container:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_server.py

Writes tests/golden/server.npz: on the decode_small model and KN bigram
(same recipe as make_golden.make_decode_small, checked against
decode_small.npz), a 1500-request RescoreServer.serve session
(decoder.py:83-104): request bytes in, response bytes out (codec.py:23-28
layouts), the ledger after the session, the cache/table counters, IndexTable.serialized
(context_table.py:107-111) of five indices; plus
rescored_path_score (decoder.py:277-292) of the beam-8 1-best of the first
8 decode_small lattices.
"""
import sys
import zlib
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as G  # noqa: E402  (puts the reference on sys.path)
from otflm.codec import RescoreRequest, pack  # noqa: E402
from otflm.decoder import RescoreServer, rescored_path_score  # noqa: E402


def main():
    lines = G.zipfian_corpus(400, 60, seed=91)
    vocab = G.build_vocabulary(lines)
    tree = G.build_huffman(vocab)
    bigram = G.train_ngram(lines, vocab, 2, smoothing="kneser-ney")
    model = G.RnnlmModel.new(vocab.size, hidden_size=16, maxent_order=3, maxent_table_bits=12, seed=17)
    G.rnnlm_mod.train(model, lines[:150], vocab, tree, epochs=1, learn_rate=0.1)
    ds = np.load(G.OUT / "decode_small.npz")
    assert np.array_equal(ds["U"], model.input_weights) and np.array_equal(ds["NV"], model.node_vectors)

    st = G.RescoreStack(model=model, tree=tree, table=G.IndexTable(16, 3), cache=G.RescoreCache(),
                        ledger=G.TransferLedger())
    srv = RescoreServer(st, bigram)
    rng = np.random.RandomState(21)
    known = [0]
    reqs, resps = [], []
    for i in range(1500):
        c = known[int(rng.randint(len(known)))] if rng.rand() < 0.8 else 0
        w = int(rng.randint(3, model.vocab_size))
        small = int(rng.randint(0, 1 << 31))
        raw = RescoreRequest(pack(c, small), w, i).to_bytes()
        out = srv.serve(raw)
        reqs.append(np.frombuffer(raw, np.uint8))
        resps.append(np.frombuffer(out, np.uint8))
        known.append(int.from_bytes(out[4:12], "little") >> 32)
    s = st.cache.stats()
    ser_idx = [1, 2, 10, 100, len(st.table)]
    ser = np.stack([np.frombuffer(st.table.serialized(i), np.uint8) for i in ser_idx])
    d = dict(ser_idx=np.array(ser_idx, np.int64), serialized=ser, requests=np.stack(reqs), responses=np.stack(resps),
             ledger=np.array([st.ledger.requests, st.ledger.bytes_indexed, st.ledger.bytes_full_baseline], np.int64),
             stats=np.array([s.lookups, s.hits, s.misses, len(st.table)], np.int64))
    # rescored_path_score of reference 1-best paths
    scores, arcs_all, lens = [], [], []
    for li in range(8):
        line = lines[li]
        lat = G.generate_lattice(vocab.tokenize(line), vocab, bigram, 2 if li % 3 == 0 else 3,
                                 zlib.crc32(line.encode()))
        st2 = G.RescoreStack(model=model, tree=tree, table=G.IndexTable(16, 3), cache=G.RescoreCache(),
                             ledger=G.TransferLedger())
        hyp, _ = G.rescore_onthefly(lat, bigram, st2, lm_weight=1.0 if li % 2 else 0.7, beam=8)
        assert list(hyp.arcs) == list(ds[f"l{li}_b3_e1_arcs"])
        scores.append(rescored_path_score(lat, hyp.arcs, model, tree, bigram, 1.0 if li % 2 else 0.7))
        arcs_all += list(hyp.arcs)
        lens.append(len(hyp.arcs))
    d.update(path_scores=np.array(scores), path_arcs=np.array(arcs_all, np.int32), path_lens=np.array(lens, np.int32))
    d["produced_by"] = np.array("otflm.decoder.RescoreServer.serve; otflm.decoder.rescored_path_score")
    np.savez_compressed(G.OUT / "server.npz", **d)
    print("wrote server.npz", (G.OUT / "server.npz").stat().st_size, "bytes; stats", d["stats"], "ledger", d["ledger"])


if __name__ == "__main__":
    main()
