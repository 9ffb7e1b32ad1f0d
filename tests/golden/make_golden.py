"""Generate golden fixtures from the REFERENCE implementation (otflm).

Run in the build container, where /root/reference is mounted:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz`` (committed).  Nothing at test time reads
/root/reference; the fixtures carry the reference's inputs and outputs.
Each fixture names the reference functions that produced it.

Fixtures
--------
kernels.npz    feature_index vectors (tests/test_rnnlm.py:162-171 recipe),
               word_logprob / advance_hidden / all_word_logprobs on the
               reference "toy" model (tests/test_rnnlm.py:14-24).
huffman.npz    build_huffman_from_counts CSR arrays (huffman.py:40-104) for
               the synthetic Zipf counts at V=1000 plus sha256 digests at
               V=20000 / 65536.
decode_small.npz  the reference small_setup stack (tests/conftest.py:86-99):
               trained model, KN bigram, 24 generator lattices; per
               (lattice, beam): rescore_onthefly 1-best, scores, end context,
               expansions, cache/table counters; plus a 2000-step
               rnnlm_prob trace replay (tests/test_cache.py:60-97).
twopass.npz    nbest (decoder.py:180-230) and rescore_twopass (decoder.py:243-274)
               on the decode_small lattices (model regenerated and checked
               against decode_small.npz) and on the config (a) lattice:
               n-best arcs and scores, two-pass winners, per-hypothesis LM
               scores (rnnlm and hybrid modes).
lfu.npz        capacity-bounded RescoreCache (cache.py:61-134, LFU with LRU
               tie-break): the acceptance crit-8 recipe (tests/test_acceptance.py:
               227-282; command corpus, retained cache, beam 6) at several
               capacities, per-utterance lookups/hits/misses/evictions/entries,
               plus a bounded 2000-step rnnlm_prob trace replay.
decode_a.npz   config (a) geometry (V=1000, H=64, MaxEnt 2^20; one 300-step
               breadth-3 lattice, beam 8): model regenerated from seeds at
               test time (sha256-checked), lattice arcs and the bigram
               entries it touches stored, reference 1-best and counters.
"""

from __future__ import annotations

import hashlib
import sys
import time
import zlib
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from otflm import _kernels_nb as knb  # noqa: E402
from otflm import rnnlm as rnnlm_mod  # noqa: E402
from otflm.cache import RescoreCache, rnnlm_prob  # noqa: E402
from otflm.codec import TransferLedger  # noqa: E402
from otflm.context_table import IndexTable  # noqa: E402
from otflm.decoder import RescoreStack, nbest, rescore_onthefly, rescore_twopass  # noqa: E402
from otflm.huffman import build_huffman, build_huffman_from_counts  # noqa: E402
from otflm.lattice import generate_lattice  # noqa: E402
from otflm.ngram import ngram_logprob, train_ngram  # noqa: E402
from otflm.rnnlm import RnnlmContext, RnnlmModel  # noqa: E402
from otflm.synth import command_corpus, zipfian_corpus  # noqa: E402
from otflm.cache import reset_utterance  # noqa: E402
from otflm.vocab import Vocabulary, build_vocabulary  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def zipf_counts(V: int) -> list[int]:
    """Synthetic vocabulary counts used by every config."""
    r = np.arange(1, V + 1, dtype=np.float64)
    return [int(c) for c in np.maximum(1, np.floor(1e7 / r ** 1.05)).astype(np.int64)]


def synth_model(V: int, H: int, bits: int) -> RnnlmModel:
    """benchmarks/kernel_speed.py:29-38 recipe on RnnlmModel.new(seed=2)."""
    m = RnnlmModel.new(V, hidden_size=H, maxent_order=3, maxent_table_bits=bits, seed=2)
    rng = np.random.RandomState(3)
    m.node_vectors[:] = rng.uniform(-0.3, 0.3, m.node_vectors.shape).astype(np.float32)
    m.maxent_table[:] = rng.uniform(-0.1, 0.1, m.maxent_size).astype(np.float32)
    return m


def ngram_tables(ng, keys_needed=None):
    items_p = list(ng.probs.items())
    items_b = list(ng.backoffs.items())
    if keys_needed is not None:
        items_p = [(k, v) for k, v in items_p if k in keys_needed]
        items_b = [(k, v) for k, v in items_b if k in keys_needed]
    W = max(ng.order, 1)

    def pack(items):
        keys = np.zeros((len(items), W), np.int32)
        lens = np.zeros(len(items), np.int32)
        vals = np.zeros(len(items), np.float64)
        for i, (k, v) in enumerate(items):
            keys[i, :len(k)] = k
            lens[i] = len(k)
            vals[i] = v
        return keys, lens, vals

    pk, pl, pv = pack(items_p)
    bk, bl, bv = pack(items_b)
    return dict(ng_order=ng.order, ng_V=ng.vocab_size, ng_bos=ng.bos_id, ng_eos=ng.eos_id,
                ng_pk=pk, ng_pl=pl, ng_pv=pv, ng_bk=bk, ng_bl=bl, ng_bv=bv)


def lattice_arrays(lat, prefix: str):
    arcs = sorted(lat.arcs, key=lambda a: a.id)
    return {
        f"{prefix}src": np.array([a.src for a in arcs], np.int32),
        f"{prefix}dst": np.array([a.dst for a in arcs], np.int32),
        f"{prefix}word": np.array([a.word for a in arcs], np.int32),
        f"{prefix}ac": np.array([a.acoustic for a in arcs], np.float64),
        f"{prefix}slm": np.array([a.smalllm for a in arcs], np.float64),
        f"{prefix}start": np.int32(lat.start),
        f"{prefix}finals": np.array(sorted(lat.finals), np.int32),
    }


def make_kernels():
    rng = np.random.RandomState(8)
    fi = []
    for _ in range(300):
        seed = int(rng.randint(0, 1 << 31))
        k = int(rng.randint(1, 5))
        words = rng.randint(0, 10 ** 6, size=4).astype(np.int64)
        node = int(rng.randint(0, 10 ** 5))
        mask = (1 << int(rng.randint(4, 24))) - 1
        got = int(knb.feature_index(np.uint64(seed), k, words[:k], node, np.uint64(mask)))
        fi.append((seed, k, *words, node, mask, got))
    fi = np.array(fi, dtype=np.uint64)

    lines = zipfian_corpus(120, 30, seed=11)
    vocab = build_vocabulary(lines)
    tree = build_huffman(vocab)
    model = RnnlmModel.new(vocab.size, hidden_size=12, maxent_order=3, maxent_table_bits=10, seed=2)
    r = np.random.RandomState(1)
    model.node_vectors[:] = r.uniform(-0.3, 0.3, model.node_vectors.shape).astype(np.float32)
    model.maxent_table[:] = r.uniform(-0.2, 0.2, model.maxent_size).astype(np.float32)
    q = np.random.RandomState(4)
    n = 200
    H, order = model.hidden_size, model.maxent_order
    hs = q.uniform(0.001, 0.999, (n, H)).astype(np.float32)
    hl = q.randint(0, order + 1, size=n).astype(np.int32)
    hist = np.full((n, order), -1, np.int64)
    ws = q.randint(0, model.vocab_size, size=n).astype(np.int32)
    lp = np.zeros(n, np.float64)
    adv = np.zeros((n, H), np.float32)
    for i in range(n):
        hist[i, :hl[i]] = q.randint(0, model.vocab_size, size=hl[i])
        ctx = RnnlmContext(hs[i], tuple(int(x) for x in hist[i, :hl[i]]))
        lp[i] = rnnlm_mod.word_logprob(model, tree, ctx, int(ws[i]))
        adv[i] = rnnlm_mod.advance_context(model, ctx, int(ws[i])).hidden
    allw = np.stack([rnnlm_mod.all_word_logprobs(
        model, tree, RnnlmContext(hs[i], tuple(int(x) for x in hist[i, :hl[i]])))
        for i in range(8)])
    np.savez_compressed(
        OUT / "kernels.npz", fi=fi,
        U=model.input_weights, W=model.recurrent_weights, NV=model.node_vectors,
        ME=model.maxent_table, seed=np.uint64(model.hash_seed), order=np.int32(order),
        pn=tree.path_nodes, ps=tree.path_signs, po=tree.path_offsets,
        q_h=hs, q_hist=hist, q_hl=hl, q_w=ws, q_lp=lp, q_adv=adv, q_all=allw,
        produced_by=np.array("otflm._kernels_nb.feature_index; otflm.rnnlm.word_logprob/"
                             "advance_context/all_word_logprobs (numba backend)"))


def make_huffman():
    out = {}
    for V in (1000, 20000, 65536):
        t = build_huffman_from_counts(zipf_counts(V))
        out[f"sha_{V}"] = np.array(sha(t.path_nodes, t.path_signs, t.path_offsets))
        if V == 1000:
            out["pn_1000"], out["ps_1000"], out["po_1000"] = t.path_nodes, t.path_signs, t.path_offsets
    # reference test vectors (tests/test_huffman.py:39-45)
    t = build_huffman_from_counts([5, 2, 1, 1])
    out["pn_5211"], out["ps_5211"], out["po_5211"] = t.path_nodes, t.path_signs, t.path_offsets
    np.savez_compressed(OUT / "huffman.npz", **out,
                        produced_by=np.array("otflm.huffman.build_huffman_from_counts"))


def make_decode_small():
    lines = zipfian_corpus(400, 60, seed=91)
    vocab = build_vocabulary(lines)
    tree = build_huffman(vocab)
    bigram = train_ngram(lines, vocab, 2, smoothing="kneser-ney")
    model = RnnlmModel.new(vocab.size, hidden_size=16, maxent_order=3, maxent_table_bits=12, seed=17)
    rnnlm_mod.train(model, lines[:150], vocab, tree, epochs=1, learn_rate=0.1)
    d = dict(U=model.input_weights, W=model.recurrent_weights, NV=model.node_vectors,
             ME=model.maxent_table, seed=np.uint64(model.hash_seed), order=np.int32(3),
             pn=tree.path_nodes, ps=tree.path_signs, po=tree.path_offsets,
             counts=np.array(vocab.counts, np.int64))
    d.update(ngram_tables(bigram))
    beams = [1, 2, 4, 8, 1 << 30]
    res = []
    nlat = 24
    for li in range(nlat):
        line = lines[li]
        breadth = 2 if li % 3 == 0 else 3
        lat = generate_lattice(vocab.tokenize(line), vocab, bigram, breadth,
                               zlib.crc32(line.encode()))
        d.update(lattice_arrays(lat, f"l{li}_"))
        for bi, beam in enumerate(beams):
            for enabled in (True, False):
                st = RescoreStack(model=model, tree=tree, table=IndexTable(16, 3),
                                  cache=RescoreCache(enabled=enabled), ledger=TransferLedger())
                hyp, rep = rescore_onthefly(lat, bigram, st, lm_weight=1.0 if li % 2 else 0.7,
                                            beam=beam)
                s = st.cache.stats()
                d[f"l{li}_b{bi}_e{int(enabled)}_arcs"] = np.array(hyp.arcs, np.int32)
                res.append((li, bi, int(enabled), hyp.combined_score, hyp.acoustic_score,
                            hyp.lm_score, hyp.end_context, rep.expansions, s.lookups, s.hits,
                            s.misses, len(st.table), st.ledger.bytes_indexed,
                            st.ledger.bytes_full_baseline))
    d["results"] = np.array(res, dtype=np.float64)
    d["beams"] = np.array(beams, np.int64)
    # retained-cache second pass (tests/test_decoder.py:110-120)
    # and trace replay (tests/test_cache.py:60-97)
    rng = np.random.RandomState(13)
    trace = []
    for i in range(2000):
        w = int(rng.randint(0, model.vocab_size))
        parent = int(rng.randint(-1, i)) if i > 0 else -1
        if rng.rand() < 0.3:
            parent = -1
        trace.append((w, parent))
    table = IndexTable(16, 3)
    cache = RescoreCache()
    succ, tp, tc, th = [], [], [], []
    for w, parent in trace:
        c = 0 if parent < 0 else succ[parent]
        v = rnnlm_prob(cache, table, model, tree, w, c)
        succ.append(v.c_next)
        tp.append(v.p)
        tc.append(v.c_next)
        th.append(table.decode(v.c_next).hidden)
    s = cache.stats()
    d.update(trace=np.array(trace, np.int64), trace_p=np.array(tp), trace_c=np.array(tc, np.int64),
             trace_h=np.array(th, np.float32),
             trace_stats=np.array([s.lookups, s.hits, s.misses, len(table)], np.int64))
    d["produced_by"] = np.array("otflm.decoder.rescore_onthefly; otflm.cache.rnnlm_prob")
    np.savez_compressed(OUT / "decode_small.npz", **d)


def make_decode_a():
    V, H, bits = 1000, 64, 20
    counts = zipf_counts(V)
    words = ["<unk>", "<s>", "</s>"] + [f"w{i}" for i in range(3, V)]
    vocab = Vocabulary(words, counts)
    tree = build_huffman(vocab)
    model = synth_model(V, H, bits)
    corpus = [" ".join(f"w{int(x) + 3}" for x in s.replace("w", "").split())
              for s in zipfian_corpus(20000, V - 3, seed=1)]
    bigram = train_ngram(corpus, vocab, 2, smoothing="kneser-ney")
    rng = np.random.RandomState(21)
    ref = [int(x) for x in rng.randint(3, V, size=300)]
    lat = generate_lattice(ref, vocab, bigram, 3, noise_seed=5)
    needed = set()
    # every n-gram lookup the decoder can make: contexts are lattice-path
    # histories, so for the bigram only (h, w) with h a predecessor word.
    for a in lat.arcs:
        for k in ((a.word,),):
            needed.add(k)
    preds = {}
    for a in lat.arcs:
        preds.setdefault(a.dst, set()).add(a.word)
    for a in lat.arcs:
        hs = preds.get(a.src, {vocab.sentence_begin_id})
        for h in hs:
            needed.add((h, a.word))
            needed.add((h,))
    t0 = time.time()
    st = RescoreStack(model=model, tree=tree, table=IndexTable(H, 3), cache=RescoreCache(),
                      ledger=TransferLedger())
    hyp, rep = rescore_onthefly(lat, bigram, st, beam=8)
    dt = time.time() - t0
    s = st.cache.stats()
    # check the subset reproduces every lookup the decode made
    d = dict(V=np.int32(V), H=np.int32(H), bits=np.int32(bits),
             model_sha=np.array(sha(model.input_weights, model.recurrent_weights,
                                    model.node_vectors, model.maxent_table)),
             tree_sha=np.array(sha(tree.path_nodes, tree.path_signs, tree.path_offsets)),
             arcs=np.array(hyp.arcs, np.int32),
             result=np.array([hyp.combined_score, hyp.acoustic_score, hyp.lm_score,
                              hyp.end_context, rep.expansions, s.lookups, s.hits, s.misses,
                              len(st.table)], np.float64),
             ref_seconds=np.float64(dt))
    d.update(ngram_tables(bigram, needed))
    d.update(lattice_arrays(lat, "lat_"))
    d["produced_by"] = np.array("otflm.decoder.rescore_onthefly (config a geometry)")
    np.savez_compressed(OUT / "decode_a.npz", **d)
    print(f"decode_a: {rep.expansions} requests in {dt:.2f}s on the reference")


def _twopass_block(d, key, lat, model, tree, bigram, n, lm_w, n_score):
    hyps = nbest(lat, n, lm_weight=lm_w)
    d[f"{key}_n"] = np.int32(n)
    d[f"{key}_lmw"] = np.float64(lm_w)
    d[f"{key}_hyp_len"] = np.array([len(h.arcs) for h in hyps], np.int32)
    d[f"{key}_hyp_arcs"] = np.array([a for h in hyps for a in h.arcs], np.int32)
    d[f"{key}_hyp_scores"] = np.array([[h.combined_score, h.acoustic_score, h.lm_score]
                                       for h in hyps], np.float64)
    modes = [("rnnlm", 0.5), ("hybrid", 0.0), ("hybrid", 0.3), ("hybrid", 1.0)]
    best = []
    for mode, lam in modes:
        b = rescore_twopass(hyps[:n_score], mode, model, tree, bigram, interp_weight=lam,
                            lm_weight=lm_w)
        idx = [h.arcs for h in hyps].index(b.arcs)
        best.append((idx, b.lm_score, b.combined_score))
    d[f"{key}_best"] = np.array(best, np.float64)
    per = np.zeros((min(n_score, len(hyps)), 2))
    for j, h in enumerate(hyps[:n_score]):
        per[j, 0] = rescore_twopass([h], "rnnlm", model, tree, bigram, lm_weight=lm_w).lm_score
        per[j, 1] = rescore_twopass([h], "hybrid", model, tree, bigram, interp_weight=0.3,
                                    lm_weight=lm_w).lm_score
    d[f"{key}_per_hyp_lm"] = per


def make_twopass():
    lines = zipfian_corpus(400, 60, seed=91)
    vocab = build_vocabulary(lines)
    tree = build_huffman(vocab)
    bigram = train_ngram(lines, vocab, 2, smoothing="kneser-ney")
    model = RnnlmModel.new(vocab.size, hidden_size=16, maxent_order=3, maxent_table_bits=12, seed=17)
    rnnlm_mod.train(model, lines[:150], vocab, tree, epochs=1, learn_rate=0.1)
    small = np.load(OUT / "decode_small.npz")
    assert np.array_equal(small["U"], model.input_weights), "small setup drifted"
    assert np.array_equal(small["W"], model.recurrent_weights)
    d = {}
    for li in range(12):
        line = lines[li]
        breadth = 2 if li % 3 == 0 else 3
        lat = generate_lattice(vocab.tokenize(line), vocab, bigram, breadth,
                               zlib.crc32(line.encode()))
        assert np.array_equal(small[f"l{li}_word"],
                              np.array([a.word for a in sorted(lat.arcs, key=lambda a: a.id)]))
        _twopass_block(d, f"l{li}", lat, model, tree, bigram, n=60 if li % 2 else 25,
                       lm_w=1.0 if li % 2 else 0.7, n_score=20)
    # config (a) lattice: 300 frames, V=1000, H=64
    a = np.load(OUT / "decode_a.npz")
    V, H, bits = 1000, 64, 20
    words = ["<unk>", "<s>", "</s>"] + [f"w{i}" for i in range(3, V)]
    vocab = Vocabulary(words, zipf_counts(V))
    tree = build_huffman(vocab)
    model = synth_model(V, H, bits)
    corpus = [" ".join(f"w{int(x) + 3}" for x in s.replace("w", "").split())
              for s in zipfian_corpus(20000, V - 3, seed=1)]
    bigram = train_ngram(corpus, vocab, 2, smoothing="kneser-ney")
    rng = np.random.RandomState(21)
    ref = [int(x) for x in rng.randint(3, V, size=300)]
    lat = generate_lattice(ref, vocab, bigram, 3, noise_seed=5)
    assert np.array_equal(a["lat_word"], np.array([x.word for x in sorted(lat.arcs, key=lambda x: x.id)]))
    t0 = time.time()
    _twopass_block(d, "a", lat, model, tree, bigram, n=100, lm_w=1.0, n_score=40)
    print(f"twopass config a: {time.time() - t0:.1f}s")
    d["produced_by"] = np.array("otflm.decoder.nbest; otflm.decoder.rescore_twopass")
    np.savez_compressed(OUT / "twopass.npz", **d)


def make_lfu():
    lines = zipfian_corpus(400, 60, seed=91)
    vocab = build_vocabulary(lines)
    tree = build_huffman(vocab)
    bigram = train_ngram(lines, vocab, 2, smoothing="kneser-ney")
    model = RnnlmModel.new(vocab.size, hidden_size=16, maxent_order=3, maxent_table_bits=12, seed=17)
    rnnlm_mod.train(model, lines[:150], vocab, tree, epochs=1, learn_rate=0.1)
    small = np.load(OUT / "decode_small.npz")
    assert np.array_equal(small["U"], model.input_weights), "small setup drifted"
    templates, utts = command_corpus(n_templates=15, n_utterances=80, seed=31, vocab_size=50)
    d = {}
    lat_of = {}
    order = []
    for tid, line in utts:
        if tid not in lat_of:
            lat = generate_lattice(vocab.tokenize(line), vocab, bigram, 2,
                                   noise_seed=zlib.crc32(line.encode()))
            lat_of[tid] = len(lat_of)
            d.update(lattice_arrays(lat, f"t{lat_of[tid]}_"))
            lat_of[("lat", tid)] = lat
        order.append(lat_of[tid])
    d["utt_template"] = np.array(order, np.int32)
    d["n_templates"] = np.int32(len([k for k in lat_of if not isinstance(k, tuple)]))
    caps = [0, 32 * 16, 32 * 64, 32 * 256, 250 * 1024]
    d["capacities"] = np.array(caps, np.int64)
    for ci, cap in enumerate(caps):
        for retain in (True, False):
            st = RescoreStack(model=model, tree=tree, table=IndexTable(16, 3),
                              cache=RescoreCache(capacity_bytes=cap), ledger=TransferLedger())
            rec = []
            for i, (tid, _) in enumerate(utts):
                hyp, rep = rescore_onthefly(lat_of[("lat", tid)], bigram, st, beam=6)
                s_ = st.cache.stats()
                rec.append((s_.lookups, s_.hits, s_.misses, s_.evictions, len(st.cache),
                            len(st.table), hyp.combined_score, hyp.end_context))
                reset_utterance(st.cache, st.table, retain=retain)
            cum = st.cache.cumulative_stats()
            d[f"c{ci}_r{int(retain)}"] = np.array(rec, np.float64)
            d[f"c{ci}_r{int(retain)}_cum"] = np.array([cum.lookups, cum.hits, cum.misses, cum.evictions],
                                                     np.int64)
    # bounded trace replay (tests/test_cache.py:60-97 recipe with capacity)
    rng = np.random.RandomState(13)
    trace = []
    for i in range(2000):
        w = int(rng.randint(0, model.vocab_size))
        parent = int(rng.randint(-1, i)) if i > 0 else -1
        if rng.rand() < 0.3:
            parent = -1
        trace.append((w, parent))
    for cap in (32 * 40, 32 * 300):
        table = IndexTable(16, 3)
        cache = RescoreCache(capacity_bytes=cap)
        succ, hits = [], []
        for w, parent in trace:
            c = 0 if parent < 0 else succ[parent]
            h0 = cache.stats().hits
            v = rnnlm_prob(cache, table, model, tree, w, c)
            succ.append(v.c_next)
            hits.append(cache.stats().hits - h0)
        s_ = cache.stats()
        d[f"trace_cap{cap}"] = np.array([s_.lookups, s_.hits, s_.misses, s_.evictions, len(cache),
                                         len(table)], np.int64)
        d[f"trace_cap{cap}_hits"] = np.array(hits, np.int8)
        d[f"trace_cap{cap}_succ"] = np.array(succ, np.int64)
    d["trace"] = np.array(trace, np.int64)
    d["produced_by"] = np.array("otflm.cache.RescoreCache(capacity_bytes>0) via rescore_onthefly / rnnlm_prob")
    np.savez_compressed(OUT / "lfu.npz", **d)


if __name__ == "__main__":
    if sys.argv[1:] == ["twopass"]:
        make_twopass()
        sys.exit(0)
    if sys.argv[1:] == ["lfu"]:
        make_lfu()
        sys.exit(0)
    make_kernels()
    make_huffman()
    make_decode_small()
    make_decode_a()
    make_twopass()
    make_lfu()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
