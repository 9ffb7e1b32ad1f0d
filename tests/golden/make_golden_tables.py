"""Golden fixture for the container-level table API, produced by the
REFERENCE (otflm) in the build container:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_tables.py

Writes tests/golden/tables.npz on the decode_small model (H=16, order 3):
IndexTable.encode (context_table.py:76-89) of 60 contexts with repeats,
history-only and one-bit hidden differences; then rnnlm_prob
(cache.py:165-182) from some encoded indices (successors may dedup against
the encoded ones); RescoreCache.get / put (cache.py:80-108) op sequences on
an enabled and a disabled cache with their results and counters.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
import make_golden as G  # noqa: E402
from otflm.cache import CacheValue  # noqa: E402


def main():
    lines = G.zipfian_corpus(400, 60, seed=91)
    vocab = G.build_vocabulary(lines)
    tree = G.build_huffman(vocab)
    model = G.RnnlmModel.new(vocab.size, hidden_size=16, maxent_order=3, maxent_table_bits=12, seed=17)
    G.rnnlm_mod.train(model, lines[:150], vocab, tree, epochs=1, learn_rate=0.1)
    ds = np.load(G.OUT / "decode_small.npz")
    assert np.array_equal(ds["U"], model.input_weights)
    rng = np.random.RandomState(31)
    H = 16
    hs, hists, lens = [], [], []
    base = [rng.uniform(0, 1, H).astype(np.float32) for _ in range(20)]
    for i in range(60):
        r = rng.rand()
        if r < 0.3 and hs:                                  # exact repeat
            j = rng.randint(len(hs)); h = hs[j].copy(); hist = [int(x) for x in hists[j][:lens[j]]]
        elif r < 0.45 and hs:                               # same hidden, other history
            j = rng.randint(len(hs)); h = hs[j].copy()
            hist = [int(x) for x in rng.randint(3, vocab.size, rng.randint(0, 4))]
        elif r < 0.55 and hs:                               # one f32 bit flipped
            j = rng.randint(len(hs)); h = hs[j].copy(); h.view(np.uint32)[rng.randint(H)] ^= 1
            hist = [int(x) for x in hists[j][:lens[j]]]
        else:
            h = base[rng.randint(20)].copy() * np.float32(rng.rand())
            hist = [int(x) for x in rng.randint(3, vocab.size, rng.randint(0, 4))]
        hs.append(h)
        lens.append(len(hist))
        hists.append(np.array(hist + [0] * (3 - len(hist)), np.uint32))
    table = G.IndexTable(16, 3)
    cache = G.RescoreCache()
    idx = [table.encode(G.RnnlmContext(h, tuple(int(x) for x in hh[:L]))) for h, hh, L in zip(hs, hists, lens)]
    tl1 = len(table)
    probe = [(int(rng.randint(3, vocab.size)), int(idx[rng.randint(len(idx))])) for _ in range(40)]
    pv = [G.rnnlm_prob(cache, table, model, tree, w, c) for w, c in probe]
    d = dict(enc_h=np.stack(hs), enc_hist=np.stack(hists), enc_len=np.array(lens, np.int32),
             enc_idx=np.array(idx, np.int64), table_len=np.int64(tl1),
             probe=np.array(probe, np.int64), probe_p=np.array([v.p for v in pv]),
             probe_c=np.array([v.c_next for v in pv], np.int64), table_len2=np.int64(len(table)))
    for enabled in (True, False):
        c2 = G.RescoreCache(enabled=enabled)
        ops, res = [], []
        keys = [(int(rng.randint(0, 30)), int(rng.randint(3, 50))) for _ in range(25)]
        for i in range(300):
            k = keys[rng.randint(len(keys))]
            if rng.rand() < 0.5:
                v = c2.get(k)
                ops.append((0, k[0], k[1], 0.0, 0))
                res.append((-1.0, -1) if v is None else (v.p, v.c_next))
            else:
                val = CacheValue(float(rng.normal()), int(rng.randint(1, 1000)))
                c2.put(k, val)
                ops.append((1, k[0], k[1], val.p, val.c_next))
                res.append((0.0, 0))
        s = c2.stats()
        tag = "on" if enabled else "off"
        d[f"ops_{tag}"] = np.array([(o[0], o[1], o[2], o[4]) for o in ops], np.int64)
        d[f"ops_{tag}_p"] = np.array([o[3] for o in ops])
        d[f"res_{tag}_p"] = np.array([r[0] for r in res])
        d[f"res_{tag}_c"] = np.array([r[1] for r in res], np.int64)
        d[f"stats_{tag}"] = np.array([s.lookups, s.hits, s.misses, len(c2)], np.int64)
        if enabled:                                      # roll_stats, clear, then one more get
            c2.roll_stats()
            s1, cu = c2.stats(), c2.cumulative_stats()
            c2.clear()
            k = keys[0]
            v = c2.get(k)
            s2 = c2.stats()
            d["after_ops"] = np.array([s1.lookups, s1.hits, s1.misses, cu.lookups, cu.hits, cu.misses,
                                       len(c2), int(v is None), s2.lookups, s2.misses], np.int64)
    d["produced_by"] = np.array("otflm.context_table.IndexTable.encode; otflm.cache.rnnlm_prob; RescoreCache.get/put")
    np.savez_compressed(G.OUT / "tables.npz", **d)
    print("tables.npz", (G.OUT / "tables.npz").stat().st_size, "len", tl1, len(table), d["stats_on"], d["stats_off"])


if __name__ == "__main__":
    main()
