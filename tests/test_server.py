"""The paper's search <-> rescorer boundary (decoder.py:83-104, codec.py:23-92)
against a RescoreServer session recorded from the reference
(tests/golden/server.npz, made by tests/golden/make_golden_server.py)."""
import struct

import numpy as np
import pytest

from paper_2007_11794_b200 import (PackOverflowError, RescoreRequest, RescoreResponse, edit_distance,
                                   first_pass_weight, pack, quantize_delta, small_context, unpack)
from paper_2007_11794_b200.model import NgramModel


def test_wire_layouts_roundtrip_reference_bytes(golden):
    d = golden("server")
    for raw in d["requests"][:50]:
        r = RescoreRequest.from_bytes(raw.tobytes())
        assert r.to_bytes() == raw.tobytes()
        assert len(r.to_bytes()) == 16
    for raw in d["responses"][:50]:
        r = RescoreResponse.from_bytes(raw.tobytes())
        assert r.to_bytes() == raw.tobytes()
        assert r.delta == quantize_delta(r.delta)


def test_quantize_and_pack():
    assert quantize_delta(0.1) == struct.unpack("<f", struct.pack("<f", 0.1))[0]   # codec.py:57-60
    assert pack(1, 2, 32) == 4294967298                                             # tests/test_codec.py:20-24
    assert unpack(pack(123, 45, 40), 40) == (123, 45)
    with pytest.raises(PackOverflowError):
        pack(1 << 32, 0)
    with pytest.raises(ValueError):
        pack(1, 1, 64)


def test_small_context_and_helpers():
    lm = NgramModel(order=3, vocab_size=10, bos_id=1, eos_id=2)
    assert small_context([], lm) == [1, 1]
    assert small_context([7], lm) == [1, 7]
    assert small_context([5, 6, 7], lm) == [5, 6, 7]
    assert edit_distance([1, 2, 3], [1, 3]) == 1
    assert edit_distance([], [4, 5]) == 2
    assert edit_distance("kitten", "sitting") == 3

    class A:
        acoustic, smalllm = -2.0, -0.5
    assert first_pass_weight(A, 0.7) == -2.0 + 0.7 * -0.5


def _stack(gm):
    from paper_2007_11794_b200 import IndexTable, RescoreCache, RescoreStack, TransferLedger
    return RescoreStack(model=gm.model, tree=gm.tree, table=IndexTable(16, 3), cache=RescoreCache(),
                        ledger=TransferLedger())


@pytest.mark.gpu
def test_serve_session_matches_reference_bytes(golden, small):
    """1500 serve() calls: every response byte-identical to the reference's
    (f32 delta, packed successor index); ledger and cache counters equal."""
    from paper_2007_11794_b200 import RescoreServer
    d = golden("server")
    _, gm, _ = small
    st = _stack(gm)
    srv = RescoreServer(st, gm.lm)
    got = [srv.serve(raw.tobytes()) for raw in d["requests"]]
    ref = [r.tobytes() for r in d["responses"]]
    bad = [i for i in range(len(ref)) if got[i] != ref[i]]
    assert not bad, f"{len(bad)} responses differ, first {bad[:5]}"
    assert [st.ledger.requests, st.ledger.bytes_indexed, st.ledger.bytes_full_baseline] == list(d["ledger"])
    s = st.cache.stats()
    assert [s.lookups, s.hits, s.misses, len(st.table)] == list(d["stats"])


@pytest.mark.gpu
def test_serve_batch_matches_one_by_one(golden, small):
    """The same session answered in device batches (a batch closes before a
    request whose context index was first returned inside it)."""
    from paper_2007_11794_b200 import RescoreServer
    d = golden("server")
    _, gm, _ = small
    srv = RescoreServer(_stack(gm), gm.lm)
    reqs = [r.tobytes() for r in d["requests"]]
    ref = [r.tobytes() for r in d["responses"]]
    born = {0: -1}
    for i, r in enumerate(ref):
        born.setdefault(int.from_bytes(r[4:12], "little") >> 32, i)
    out, i, n_batches = [], 0, 0
    while i < len(reqs):
        j = i
        while j < len(reqs) and born[RescoreRequest.from_bytes(reqs[j]).packed >> 32] < i:
            j += 1
        resp = srv.serve_batch(b"".join(reqs[i:j]))
        out += [resp[k:k + 16] for k in range(0, len(resp), 16)]
        i, n_batches = j, n_batches + 1
    assert out == ref
    assert n_batches < len(reqs) // 2


@pytest.mark.gpu
def test_server_errors(small):
    from paper_2007_11794_b200 import RescoreServer, UnknownIndexError
    _, gm, _ = small
    lm3 = NgramModel(order=5, vocab_size=gm.model.vocab_size, bos_id=1, eos_id=2)
    with pytest.raises(ValueError, match="small LM order"):
        RescoreServer(_stack(gm), lm3)
    srv = RescoreServer(_stack(gm), gm.lm)
    with pytest.raises(ValueError):
        srv.serve(b"\0" * 15)
    with pytest.raises(ValueError):
        srv.serve(RescoreRequest(pack(0, 0), gm.model.vocab_size, 0).to_bytes())
    with pytest.raises(UnknownIndexError):
        srv.serve(RescoreRequest(pack(999, 0), 5, 0).to_bytes())


@pytest.mark.gpu
def test_rescored_path_score_matches_reference(golden, small):
    from paper_2007_11794_b200 import rescored_path_score
    d = golden("server")
    _, gm, lats = small
    off = 0
    for li in range(len(d["path_scores"])):
        n = int(d["path_lens"][li])
        arcs = [int(a) for a in d["path_arcs"][off:off + n]]
        off += n
        got = rescored_path_score(lats[li], arcs, gm.model, gm.tree, gm.lm, 1.0 if li % 2 else 0.7)
        assert abs(got - float(d["path_scores"][li])) <= 1e-9


@pytest.mark.gpu
def test_index_table_serialized_matches_reference(golden, small):
    """IndexTable.serialized after the serve session: history slots, order and
    index bytes identical; hidden f32 within 1 ulp (exact-mode bound)."""
    from paper_2007_11794_b200 import RescoreServer, UnknownIndexError
    d = golden("server")
    _, gm, _ = small
    st = _stack(gm)
    srv = RescoreServer(st, gm.lm)
    for raw in d["requests"]:
        srv.serve(raw.tobytes())
    H = gm.model.hidden_size
    for idx, ref in zip(d["ser_idx"], d["serialized"]):
        got = np.frombuffer(st.table.serialized(int(idx)), np.uint8)
        assert got.shape == ref.shape == (st.table.element_bytes,)
        assert np.array_equal(got[4 * H:], ref[4 * H:])
        gh, rh = got[:4 * H].view(np.int32), ref[:4 * H].view(np.int32)
        assert np.all(np.abs(gh.astype(np.int64) - rh) <= 1)
    with pytest.raises(UnknownIndexError):
        st.table.serialized(len(st.table) + 1)
