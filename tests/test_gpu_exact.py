"""The EXACT precision of the persistent stream kernel (exact_update.cuh) on
the B200: integer digit-plane recurrent update on tcgen05 (kind::i8) with
certified f32 rounding + the reference's sequential float64 loop for the
uncertified elements, float64 HS.  Every hidden state is the reference's
float32 value, so against the CPU oracle the decode is identical in every
observable: 1-best arcs, expansions, end context, cache lookups / hits /
misses and IndexTable length; scores differ only by float64 summation order
(|d| <= 1e-9).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _decode(s, precision, schedule, beam, enabled=True):
    from paper_2007_11794_b200.rescore import BatchDecoder
    need = BatchDecoder.contexts_needed(s.lattices, beam)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, enabled=enabled,
                       precision=precision, schedule=schedule)
    assert dec.schedule == schedule
    dec.prepare(s.lattices, beam)
    dec.run(1.0)
    hyps, out = dec.fetch()
    return hyps, out, dec.streams.stats()


def _assert_identical(hyps, out, st, ref):
    for u, (r, (lk, hi, mi)) in enumerate(ref):
        assert hyps[u].arcs == r.arcs, f"utterance {u}: 1-best differs"
        assert abs(hyps[u].combined_score - r.combined_score) <= 1e-9
        assert abs(hyps[u].lm_score - r.lm_score) <= 1e-9
        assert int(out["expansions"][u]) == r.expansions
        assert hyps[u].end_context == r.end_context
        assert (int(st[u, 0]), int(st[u, 1]), int(st[u, 2])) == (lk, hi, mi), f"utterance {u}: cache counters"
        assert int(st[u, 3]) == r.table_len, f"utterance {u}: IndexTable length"


# (config, n_utt, frames, beam, cache): H = 64 / 256 / 512; cache off and a
# wide beam push a level past one 96-row chunk and one 512-request assign chunk
CASES = [("a", 12, 60, 8, True), ("a", 6, 30, 32, False), ("b", 6, 60, 8, True), ("c", 3, 30, 8, True)]


@pytest.mark.parametrize("schedule", ["stream", "stream1"])
@pytest.mark.parametrize("case", CASES)
def test_exact_stream_identical_to_oracle(case, schedule):
    """Both persistent schedules: the 2-CTA cluster per stream and the
    one-CTA-per-stream kernel (exact_solo.cuh)."""
    from paper_2007_11794_b200 import synth
    name, n_utt, T, beam, enabled = case
    s = synth.build_setup(name, n_utt=n_utt, T=T, seed=5)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=beam, enabled=enabled, n_threads=4)
    hyps, out, st = _decode(s, "exact", schedule, beam, enabled)
    _assert_identical(hyps, out, st, ref)


def test_exact_is_the_auto_stream_choice_and_matches_fp64_level():
    """BatchDecoder(schedule="auto") runs EXACT on the stream kernel; the FP64
    level schedule and the EXACT stream kernel give the same decode."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("b", n_utt=8, T=50, seed=17)
    need = BatchDecoder.contexts_needed(s.lattices, 8)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision="exact")
    assert dec.schedule == "stream"
    hs, os_, ss = _decode(s, "exact", "stream", 8)
    hl, ol, sl = _decode(s, "fp64", "level", 8)
    assert np.array_equal(ss[:, :4], sl[:, :4])
    assert np.array_equal(os_["expansions"], ol["expansions"])
    for a, b in zip(hs, hl):
        assert a.arcs == b.arcs and a.end_context == b.end_context
        assert abs(a.combined_score - b.combined_score) <= 1e-9


@pytest.mark.parametrize("case", [("b", 6, 60, 8, True), ("c", 3, 30, 8, True)])
def test_exact_level_schedule_identical_to_oracle(case):
    """EXACT in the level-synchronous schedule (k_advance_exact + the float64
    HS kernels): the same identity with the oracle."""
    from paper_2007_11794_b200 import synth
    name, n_utt, T, beam, enabled = case
    s = synth.build_setup(name, n_utt=n_utt, T=T, seed=5)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=beam, enabled=enabled, n_threads=4)
    hyps, out, st = _decode(s, "exact", "level", beam, enabled)
    _assert_identical(hyps, out, st, ref)


@pytest.mark.parametrize("schedule", ["stream", "stream1"])
@pytest.mark.parametrize("capacity", [0, 32 * 4000])
def test_exact_stream_retained_streams_vs_oracle(capacity, schedule):
    """Retained streams (BatchDecoder.run(retain=True), reset_utterance(retain=True),
    cache.py:185-191): each stream decodes a sequence of utterances with
    repeats, so whole levels hit the cache (nothing computed) -- their
    requests still need the small-LM term.  Per round: 1-best, score, end
    context and cache counters equal an oracle stack with the same history;
    unbounded and capacity-bounded (LFU) caches."""
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("a", n_utt=3, T=30, seed=13)
    seqs = [[0, 1, 0, 0], [2, 2, 1, 2]]          # stream -> lattice per round
    need = BatchDecoder.contexts_needed(s.lattices, 8) * 4
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(seqs), need, precision="exact", capacity_bytes=capacity,
                       schedule=schedule)
    om, og = O.OracleModel(s.model, s.tree), O.OracleNgram(s.small_lm)
    stacks = [O.OracleStack(om, None, capacity_bytes=capacity) for _ in seqs]
    for k in range(4):
        dec.prepare([s.lattices[q[k]] for q in seqs], 8)
        dec.run(1.0, retain=k > 0)
        hyps, out = dec.fetch()
        st = dec.streams.stats()
        for u, q in enumerate(seqs):
            if k > 0:
                stacks[u].reset(True)
            r = stacks[u].rescore_onthefly(s.lattices[q[k]], og, beam=8)
            o = stacks[u].stats()
            assert hyps[u].arcs == r.arcs, (k, u)
            assert abs(hyps[u].combined_score - r.combined_score) <= 1e-9, (k, u)
            assert hyps[u].end_context == r.end_context, (k, u)
            assert (int(st[u, 0]), int(st[u, 1]), int(st[u, 2])) == (o.lookups, o.hits, o.misses), (k, u)
    assert int(st[:, 1].sum()) > 0          # the repeats really hit
