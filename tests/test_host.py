"""Host-side logic (no GPU): input builders, lattice container and text
format, n-gram lookup, packing, the C-ABI boundary of the built library."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.lattice import Lattice, generate_lattice
from paper_2007_11794_b200.model import RnnlmModel, ngram_logprob


ROOT = Path(__file__).resolve().parent.parent


def test_generator_structure_and_scores():
    lm = synth.synth_bigram(500, seed=2)
    lat = generate_lattice([7, 9, 11, 13], 500, lm, 3, noise_seed=5)
    # one start node, b nodes per later position, b arcs per node except start
    assert lat.n_arcs == 3 + 3 * 3 * 3
    assert len(lat.finals) == 3
    ref_path_ac = [a.acoustic for a in lat.arcs if a.word in (7, 9, 11, 13)]
    assert all(a == 0.0 for a in ref_path_ac)
    for a in lat.arcs[:20]:
        pred = {b.word for b in lat.arcs if b.dst == a.src} or {1}
        (h,) = pred
        assert a.smalllm == ngram_logprob(lm, [h], a.word)
    # topological order = ascending id for generator lattices
    assert lat.topo_order == sorted(lat.topo_order)


def test_lattice_text_round_trip(tmp_path):
    lm = synth.synth_bigram(200, seed=1)
    lat = generate_lattice([5, 6, 7], 200, lm, 2, noise_seed=1)
    p = tmp_path / "x.lat"
    lat.save(p)
    back = Lattice.load(p)
    assert back.n_arcs == lat.n_arcs and back.finals == lat.finals and back.start == lat.start
    assert np.array_equal(back.arc_acoustic, lat.arc_acoustic)
    assert np.array_equal(back.arc_smalllm, lat.arc_smalllm)


def test_oracle_ngram_matches_host_lookup():
    lm = synth.synth_bigram(300, seed=3)
    og = O.OracleNgram(lm)
    rng = np.random.RandomState(0)
    for _ in range(300):
        h, w = int(rng.randint(0, 300)), int(rng.randint(0, 300))
        assert og.logprob([h], w) == ngram_logprob(lm, [h], w)
        assert og.logprob([], w) == ngram_logprob(lm, [], w)


def test_rnlm_file_round_trip(tmp_path):
    m = synth.synth_model(50, 8, 6)
    m.save(tmp_path / "m.bin")
    m2 = RnnlmModel.load(tmp_path / "m.bin")
    for name in ("input_weights", "recurrent_weights", "node_vectors", "maxent_table"):
        assert np.array_equal(getattr(m, name), getattr(m2, name))


def test_pack_unpack_reference_vectors():
    from paper_2007_11794_b200 import PackOverflowError, pack, unpack
    assert pack(1, 2, 32) == 4294967298          # test_codec.py:20-24
    assert unpack(4294967298, 32) == (1, 2)
    with pytest.raises(PackOverflowError, match="rnnlm_index"):
        pack(1 << 32, 0, 32)


def test_synthetic_setup_deterministic():
    a = synth.build_setup("a", n_utt=2, T=20, seed=4)
    b = synth.build_setup("a", n_utt=2, T=20, seed=4)
    assert np.array_equal(a.lattices[1].arc_smalllm, b.lattices[1].arc_smalllm)
    assert np.array_equal(a.model.maxent_table, b.model.maxent_table)


def _declared_symbols():
    hdr = (ROOT / "include" / "otflm_b200.h").read_text()
    return sorted(set(re.findall(r"\b(otflm_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    from paper_2007_11794_b200 import _lib
    assert _lib.LIB_PATH.exists(), "run __graft_entry__.build() first"
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = _declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_product_has_no_oracle_dependency():
    pkg = ROOT / "paper_2007_11794_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu*")):
        text = p.read_text()
        assert "oracle" not in text.lower().replace("no cpu fallback", ""), p


def test_lattice_generator_matches_reference_generator(golden):
    """The vectorised synthetic-lattice generator (the bench's input builder)
    is the reference's generate_lattice (lattice.py:130-183) draw for draw:
    same arcs (src, dst, word, acoustic, small-LM score), start and finals for
    bigram and trigram small LMs and breadths 1-8 (tests/golden/lattices.npz,
    made by tests/golden/make_golden_lattices.py from the reference)."""
    from paper_2007_11794_b200.lattice import generate_lattice
    from paper_2007_11794_b200.model import ngram_from_arrays
    d = golden("lattices")
    V = int(d["V"])
    for p in d["cases"]:
        p = str(p)
        o = p[:3]
        lm = ngram_from_arrays(*(d[f"{o}ng_{k}"] for k in ("order", "V", "bos", "eos", "pk", "pl", "pv",
                                                            "bk", "bl", "bv")))
        lat = generate_lattice([int(w) for w in d[p + "ref"]], V, lm, int(d[p + "breadth"]),
                               int(d[p + "seed"]))
        arcs = sorted(lat.arcs, key=lambda a: a.id)
        assert lat.start == int(d[p + "start"]), p
        assert sorted(lat.finals) == [int(x) for x in d[p + "finals"]], p
        assert [a.src for a in arcs] == [int(x) for x in d[p + "src"]], p
        assert [a.dst for a in arcs] == [int(x) for x in d[p + "dst"]], p
        assert [a.word for a in arcs] == [int(x) for x in d[p + "word"]], p
        assert np.array_equal(np.array([a.acoustic for a in arcs]), d[p + "ac"]), p
        assert np.allclose(np.array([a.smalllm for a in arcs]), d[p + "slm"], rtol=0, atol=1e-12), p
