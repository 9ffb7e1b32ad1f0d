"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu`` and call the
product path through the C-ABI; CPU tests cover the oracle (pinned against
the reference's golden vectors), host logic and the library boundary."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libotflm_b200.so")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))
        return cache[name]

    return load


class GoldenModel:
    """Reference-shaped model/tree/small-LM rebuilt from a golden fixture."""

    def __init__(self, d):
        from paper_2007_11794_b200.model import HuffmanTree, RnnlmModel, ngram_from_arrays
        V = d["U"].shape[0]
        H = d["U"].shape[1]
        self.model = RnnlmModel(hidden_size=H, vocab_size=V, maxent_order=int(d["order"]),
                                maxent_size=d["ME"].shape[0], hash_seed=int(d["seed"]),
                                input_weights=d["U"], recurrent_weights=d["W"],
                                node_vectors=d["NV"], maxent_table=d["ME"])
        self.tree = HuffmanTree(n_words=V, children=np.zeros((V - 1, 2), np.int64),
                                path_nodes=d["pn"], path_signs=d["ps"], path_offsets=d["po"])
        if "ng_order" in d:
            self.lm = ngram_from_arrays(d["ng_order"], d["ng_V"], d["ng_bos"], d["ng_eos"],
                                        d["ng_pk"], d["ng_pl"], d["ng_pv"], d["ng_bk"],
                                        d["ng_bl"], d["ng_bv"])


def golden_lattice(d, prefix):
    from paper_2007_11794_b200.lattice import Lattice
    return Lattice(int(d[f"{prefix}start"]), [int(x) for x in d[f"{prefix}finals"]],
                   src=d[f"{prefix}src"], dst=d[f"{prefix}dst"], word=d[f"{prefix}word"],
                   acoustic=d[f"{prefix}ac"], smalllm=d[f"{prefix}slm"])


@pytest.fixture(scope="session")
def small(golden):
    d = golden("decode_small")
    gm = GoldenModel(d)
    lats = []
    i = 0
    while f"l{i}_src" in d:
        lats.append(golden_lattice(d, f"l{i}_"))
        i += 1
    return d, gm, lats


@pytest.fixture(scope="session")
def config_a(golden):
    """Config (a) geometry: model regenerated from seeds (sha-checked)."""
    import hashlib
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.model import build_huffman_from_counts, ngram_from_arrays
    d = golden("decode_a")
    model = synth.synth_model(int(d["V"]), int(d["H"]), int(d["bits"]))
    tree = build_huffman_from_counts(synth.zipf_counts(int(d["V"])))
    h = hashlib.sha256()
    for a in (model.input_weights, model.recurrent_weights, model.node_vectors,
              model.maxent_table):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(d["model_sha"]), "synthetic model recipe drifted"
    lm = ngram_from_arrays(d["ng_order"], d["ng_V"], d["ng_bos"], d["ng_eos"], d["ng_pk"],
                           d["ng_pl"], d["ng_pv"], d["ng_bk"], d["ng_bl"], d["ng_bv"])
    return d, model, tree, lm, golden_lattice(d, "lat_")


@pytest.fixture(scope="session")
def tp(golden):
    """tests/golden/twopass.npz: reference nbest / rescore_twopass outputs."""
    return golden("twopass")


def small_results(d):
    """rows: (li, bi, enabled, combined, acoustic, lm, end_ctx, expansions,
    lookups, hits, misses, table_len, bytes_indexed, bytes_full)"""
    return d["results"]
