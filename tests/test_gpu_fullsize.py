"""Parity at the bench's full sizes.

The headline workload itself -- config b, 64 utterances x 300 frames,
V = 20,000, H = 256, MaxEnt 2^21, beam 8, the bench's seed, TF32X3 stream
schedule -- decoded on the B200 and by the exact CPU oracle (utterance-
parallel over the host's cores, a few seconds), plus config c geometry
(V = 65,536, H = 512) at full utterance length.

Bar (BASELINE.json north star): outputs match the CPU reference, the 1-best
identical except where competing path costs tie within the tolerance.  The
exact FP64 mode is held to identity at the full bench size (arcs, expansions,
context ids, cache counters; scores within 1e-9).  The TF32X3 tensor-core
mode is held to the stated looser bound in its test.  Size-independent
property in both: the GPU's combined score equals the oracle's rescoring of
the GPU's own arcs (`oracle_path_score`, reference tests/conftest.py:65-78).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


# identical TF32X3 1-bests measured for the seeds below (regression pins)
TF32X3_SAME = {"b": 53, "c": 8}


def _gpu_decode(s, beam, precision):
    from paper_2007_11794_b200.rescore import BatchDecoder
    need = BatchDecoder.contexts_needed(s.lattices, beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision=precision)
    dec.prepare(s.lattices, beam)
    dec.run(1.0)
    hyps, out = dec.fetch()
    return dec, hyps, out, dec.streams.stats()


def _compare(s, beam, precision):
    """Per utterance: (arcs identical, expansions identical, |GPU - oracle
    best| score, oracle rescoring of the GPU path - oracle best)."""
    dec, hyps, out, st = _gpu_decode(s, beam, precision)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=beam)
    om, og = O.OracleModel(s.model, s.tree), O.OracleNgram(s.small_lm)
    rows = []
    for u, (r, counts) in enumerate(ref):
        h = hyps[u]
        gpu_path = O.path_score(om, None, og, s.lattices[u], h.arcs)
        rows.append(dict(arcs=h.arcs == r.arcs, exp=int(out["expansions"][u]) == r.expansions,
                         counts=tuple(int(x) for x in st[u, :3]) == counts,
                         end_ctx=h.end_context == r.end_context,
                         d_score=abs(h.combined_score - r.combined_score),
                         self_consistency=abs(h.combined_score - gpu_path),
                         gap=gpu_path - r.combined_score))
    return dec, rows


def test_bench_config_b_full_workload_fp64_exact():
    """The bench's N=1 workload (bench.py: build_setup(CONFIG, 64, 300,
    seed=7)) in the exact FP64 mode: 1-best arcs, expansions, end context,
    cache lookups / hits / misses identical for all 64 utterances, combined
    scores within 1e-9."""
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("b", n_utt=64, T=300, seed=7)
    dec, rows = _compare(s, 8, "fp64")
    for u, r in enumerate(rows):
        assert r["arcs"] and r["exp"] and r["end_ctx"] and r["counts"], (u, r)
        assert r["d_score"] <= 1e-9 and r["self_consistency"] <= 1e-9, (u, r)


def _assert_exact(rows, table_len_ok=True):
    for u, r in enumerate(rows):
        assert r["arcs"] and r["exp"] and r["end_ctx"] and r["counts"], (u, r)
        assert r["d_score"] <= 1e-9 and r["self_consistency"] <= 1e-9, (u, r)


def test_bench_config_b_full_workload_exact_stream():
    """The EXACT precision of the persistent stream kernel (integer
    digit-plane tcgen05 update and HS with certified rounding) on the bench's
    config-b workload: identical to the oracle for all 64 utterances x 300
    frames (arcs, expansions, end context, cache counters; scores 1e-9)."""
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("b", n_utt=64, T=300, seed=7)
    dec, rows = _compare(s, 8, "exact")
    assert dec.schedule == "stream"
    _assert_exact(rows)


def test_bench_config_e_batch_exact_stream():
    """One full batch of the bench's default workload (config e: V=65,536,
    H=512, MaxEnt 2^22; utterance ids 0..73 of the 4,096, 300 frames; the
    bench's per-id lattices): EXACT stream decode identical to the oracle."""
    from paper_2007_11794_b200 import synth
    base = synth.build_setup("e", n_utt=1, T=300, seed=31)
    base.lattices = synth.lattices_for_ids(base, range(74), 300)
    dec, rows = _compare(base, 8, "exact")
    assert dec.schedule == "stream"
    _assert_exact(rows)


def test_bench_config_e_full_batch_exact_solo():
    """Exactly one batch of the benched path: utterance ids 0..147 of the
    bench's config-e workload (its per-id lattices, 300 frames), decoded by
    k_decode_solo (the automatic choice for a 148-stream EXACT batch, as in
    bench.py) -- every observable identical to the oracle for all 148."""
    from paper_2007_11794_b200 import synth
    base = synth.build_setup("e", n_utt=1, T=300, seed=31)
    base.lattices = synth.lattices_for_ids(base, range(148), 300)
    dec, rows = _compare(base, 8, "exact")
    assert dec.schedule == "stream1"
    _assert_exact(rows)


@pytest.mark.parametrize("config,n_utt,seed", [("b", 64, 7), ("c", 8, 17)])
def test_full_size_tf32x3_stream_vs_oracle(config, n_utt, seed):
    """TF32X3 (fp32-faithful tcgen05 recurrent update, stream schedule) at
    full utterance length: an APPROXIMATE precision (per-query scores within
    ~1e-6 of the reference's float64-accumulated values), not the benched
    one -- EXACT is (bit-identical, tests above).  Held here: for every
    utterance the GPU's combined score equals the oracle's rescoring of the
    GPU's own arcs within 1e-4 per frame (every per-query score on the path is
    right, reference tests/conftest.py:65-78), identical 1-bests score within
    1e-4 per frame of the oracle's, and the number of identical 1-bests is
    pinned to the measured value for these seeds (a regression guard).  The
    other utterances diverge where the fp32-level differences reorder tokens
    at a beam cut; that they are ties is not proven (profiles/r01q_*), which
    is why the bench does not run this mode."""
    from paper_2007_11794_b200 import synth
    T = 300
    s = synth.build_setup(config, n_utt=n_utt, T=T, seed=seed)
    dec, rows = _compare(s, 8, "tf32x3")
    assert dec.schedule == "stream"
    same = sum(r["arcs"] for r in rows)
    gaps = [r["gap"] for r in rows if not r["arcs"]]
    print(f"config {config} full length tf32x3: identical 1-best {same}/{len(rows)}, "
          f"divergent gaps {sorted(round(g, 4) for g in gaps)}")
    for u, r in enumerate(rows):
        assert r["self_consistency"] <= 1e-4 * T, (u, r)
        if r["arcs"]:
            assert r["d_score"] <= 1e-4 * T, (u, r)
    assert same >= TF32X3_SAME[config], same


@pytest.mark.parametrize("precision", ["fp64", "tf32x3", "exact"])
def test_fat_variant_vs_oracle(precision):
    """SURVEY.md §8d config (b) fat variant: breadth 16, beam 64 (about 15k
    requests per frame per utterance, 256 tokens x 16 arcs per node set)."""
    from paper_2007_11794_b200 import synth
    T = 10
    s = synth.build_setup("b_fat", n_utt=4, T=T, seed=3)
    dec, rows = _compare(s, 64, precision)
    for u, r in enumerate(rows):
        if precision in ("fp64", "exact"):
            assert r["arcs"] and r["exp"] and r["end_ctx"] and r["counts"], (u, r)
            assert r["d_score"] <= 1e-9 and r["self_consistency"] <= 1e-9, (u, r)
        else:
            assert r["self_consistency"] <= 1e-4 * T, (u, r)
            assert r["arcs"] or -2e-3 * T <= r["gap"] <= 1e-4 * T, (u, r)
    print(f"fat {precision}: schedule {dec.schedule}, identical 1-best {sum(r['arcs'] for r in rows)}/{len(rows)}")


def test_fat_variant_full_length_exact_modes_agree():
    """The fat variant at full length (4 x 300, breadth 16, beam 64: 19.5M
    requests, 19.2M IndexTable rows) -- the shape where round 1's FP64 level
    schedule stopped with a digest error.  FP64 (level schedule, CUDA-core
    float64), EXACT level (k_advance_exact) and EXACT stream (digit-plane
    tensor-core kernels) are three different code paths computing the
    reference's arithmetic: every observable must agree between them, and
    the table lengths are pinned to the measured FP64 result."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("b_fat", n_utt=4, T=300, seed=3)
    need = BatchDecoder.contexts_needed(s.lattices, 64)
    runs = {}
    for prec, sched in (("fp64", "level"), ("exact", "level"), ("exact", "stream")):
        dec = BatchDecoder(s.model, s.tree, s.small_lm, 4, need, precision=prec, schedule=sched)
        dec.prepare(s.lattices, 64)
        dec.run(1.0)
        hyps, out = dec.fetch()
        st = dec.streams.stats()
        runs[(prec, sched)] = (hyps, out["expansions"].copy(), st[:, :4].copy())
        del dec
    h0, e0, s0 = runs[("fp64", "level")]
    assert [int(x) for x in s0[:, 3]] == [4800217, 4792179, 4794547, 4787347]
    assert int(e0.sum()) == 19481664
    for key, (h, e, st) in runs.items():
        assert np.array_equal(e, e0), key
        assert np.array_equal(st, s0), key
        for a, b in zip(h, h0):
            assert a.arcs == b.arcs and a.end_context == b.end_context, key
            assert abs(a.combined_score - b.combined_score) <= 1e-9, key
