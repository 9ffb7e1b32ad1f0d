"""Kernel-level parity on the B200: sm_100a kernels vs the CPU oracle and the
reference golden vectors.  Tolerances are written per test:

* feature_index, Huffman path indexing: bit-exact.
* word_logprob (float64 accumulation, tree reduction): |d| <= 1e-12.
* advance_hidden FP64 mode (reference summation order): bit-exact except a
  libm-vs-libdevice exp() ulp flip, counted and bounded (< 1e-4 of elements,
  never more than 1 float32 ulp).
* tcgen05 modes: TF32X3 |d| <= 2e-6, TF32 |d| <= 2e-3, BF16 |d| <= 1e-2 on
  h' in (0, 1) (stated looser bounds of the north star).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import GoldenModel
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t
    assert t.cuda.is_available(), "GPU tests need a CUDA device"
    return t


def test_library_loaded_from_tree(torch):
    from paper_2007_11794_b200 import _lib
    L = _lib.load()
    assert str(_lib.LIB_PATH) in L._name


def test_feature_index_bit_exact(golden, torch):
    from paper_2007_11794_b200 import kernels
    fi = golden("kernels")["fi"].astype(np.uint64)
    for row in fi[:50]:
        k = int(row[1])
        got = kernels.feature_index(int(row[0]), k, row[2:2 + k].astype(np.int64), int(row[6]),
                                    int(row[7]))
        assert int(got) == int(row[8])
    rng = np.random.RandomState(3)
    n = 20000
    ks = rng.randint(1, 8, size=n)
    words = rng.randint(0, 2**31 - 1, size=(n, 8)).astype(np.int64)
    nodes = rng.randint(0, 2**31 - 1, size=n).astype(np.int64)
    seed, mask = 0x5DEECE66D, (1 << 22) - 1
    got = kernels.feature_index_batch(seed, mask, ks, words, nodes)
    for i in range(0, n, 97):
        assert int(got[i]) == O.feature_index(seed, int(ks[i]), words[i, :ks[i]], int(nodes[i]), mask)


def test_reference_signature_kernels_vs_golden(golden, torch):
    from paper_2007_11794_b200 import kernels
    d = golden("kernels")
    gm = GoldenModel(d)
    m, t = gm.model, gm.tree
    worst = 0.0
    for i in range(0, len(d["q_w"]), 5):
        L = int(d["q_hl"][i])
        w = int(d["q_w"][i])
        o0, o1 = t.path_offsets[w], t.path_offsets[w + 1]
        lp = kernels.word_logprob(d["q_h"][i], d["q_hist"][i, :L], t.path_nodes[o0:o1],
                                  t.path_signs[o0:o1], m.node_vectors, m.maxent_table,
                                  m.maxent_order, m.hash_seed, m.maxent_size - 1)
        worst = max(worst, abs(lp - d["q_lp"][i]))
        adv = kernels.advance_hidden(m.input_weights[w], m.recurrent_weights, d["q_h"][i])
        assert np.array_equal(adv, d["q_adv"][i])
    assert worst <= 1e-12
    for i in range(3):
        L = int(d["q_hl"][i])
        allw = kernels.all_word_logprobs(d["q_h"][i], d["q_hist"][i, :L], t.path_nodes,
                                         t.path_signs, t.path_offsets, m.node_vectors,
                                         m.maxent_table, m.maxent_order, m.hash_seed,
                                         m.maxent_size - 1)
        assert np.max(np.abs(allw - d["q_all"][i])) <= 1e-12
        assert abs(np.exp(allw).sum() - 1.0) < 1e-9    # test_rnnlm.py:99-106


def _queries(model, n, seed):
    rng = np.random.RandomState(seed)
    H, V, order = model.hidden_size, model.vocab_size, model.maxent_order
    h = rng.uniform(0.001, 0.999, (n, H)).astype(np.float32)
    hl = rng.randint(0, order + 1, size=n).astype(np.int32)
    hist = rng.randint(0, V, size=(n, order)).astype(np.int32)
    w = rng.randint(0, V, size=n).astype(np.int32)
    return h, hist, hl, w


@pytest.mark.parametrize("V,H", [(1000, 64), (20000, 256), (65536, 512), (300, 20)])
def test_word_logprob_batch_vs_oracle(V, H, torch):
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    from paper_2007_11794_b200.model import build_huffman_from_counts
    bits = {1000: 20, 20000: 21, 65536: 22, 300: 12}[V]
    model = synth.synth_model(V, H, bits)
    tree = build_huffman_from_counts(synth.zipf_counts(V))
    dm = DeviceModel(model, tree)
    n = 4096
    h, hist, hl, w = _queries(model, n, seed=V)
    want, _ = O.query_batch(model, tree, h, hist.astype(np.int64), hl, w, want_h=False)
    ctx = torch.arange(n, dtype=torch.int32, device="cuda")
    got = kernels.word_logprob_batch(dm, ctx, torch.from_numpy(h).cuda(),
                                     torch.from_numpy(hist).cuda(), torch.from_numpy(hl).cuda(),
                                     torch.from_numpy(w).cuda()).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-12


@pytest.mark.parametrize("V,H", [(1000, 64), (20000, 256), (65536, 512), (300, 20)])
def test_advance_fp64_matches_oracle(V, H, torch):
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    model = synth.synth_model(V, H, 12)
    dm = DeviceModel(model, None, output=False)
    n = 2048
    h, hist, hl, w = _queries(model, n, seed=H)
    _, want = O.query_batch(model, _NoTree(V), h, hist.astype(np.int64), hl, w, want_p=False)
    ctx = torch.arange(n, dtype=torch.int32, device="cuda")
    got = kernels.advance_hidden_batch(dm, ctx, torch.from_numpy(h).cuda(),
                                       torch.from_numpy(w).cuda(), "fp64").cpu().numpy()
    diff = got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64)
    assert np.max(np.abs(diff)) <= 1           # at most one float32 ulp
    assert np.count_nonzero(diff) <= max(2, 1e-4 * diff.size)


class _NoTree:
    def __init__(self, V):
        self.path_nodes = np.zeros(1, np.int32)
        self.path_signs = np.ones(1, np.float32)
        self.path_offsets = np.zeros(V + 1, np.int64)


@pytest.mark.parametrize("prec,tol", [("tf32x3", 2e-6), ("tf32", 2e-3), ("bf16", 1e-2)])
@pytest.mark.parametrize("H", [64, 256, 512])
def test_advance_tensor_core_modes(prec, tol, H, torch):
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    V = 4000
    model = synth.synth_model(V, H, 12)
    dm = DeviceModel(model, None, output=False)
    n = 3000   # not a multiple of the 128-row tile
    h, hist, hl, w = _queries(model, n, seed=7)
    perm = np.random.RandomState(1).permutation(n).astype(np.int32)   # gathered A rows
    ctx = torch.from_numpy(perm).cuda()
    got = kernels.advance_hidden_batch(dm, ctx, torch.from_numpy(h).cuda(),
                                       torch.from_numpy(w).cuda(), prec).cpu().numpy()
    want = _oracle_perm(model, h, w, perm)
    assert np.max(np.abs(got.astype(np.float64) - want.astype(np.float64))) <= tol


@pytest.mark.parametrize("H", [64, 256, 512])
def test_advance_exact_bit_identical(H, torch):
    """EXACT (k_advance_exact: digit planes on tcgen05 kind::i8, certified
    rounding, the reference loop for the rest): every output float equals
    the reference's bit for bit -- including zero contexts and context rows
    with elements far below the 2^-9 digit resolution."""
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    V = 4000
    model = synth.synth_model(V, H, 12)
    dm = DeviceModel(model, None, output=False)
    n = 3000
    h, hist, hl, w = _queries(model, n, seed=11)
    h[5] = 0.0                                   # the zero context
    h[7, ::3] = 1e-7                             # tiny elements: not representable in 32 fixed-point bits
    h[9, :4] = 3.0e-39                           # subnormals
    perm = np.random.RandomState(2).permutation(n).astype(np.int32)
    got = kernels.advance_hidden_batch(dm, torch.from_numpy(perm).cuda(), torch.from_numpy(h).cuda(),
                                       torch.from_numpy(w).cuda(), "exact").cpu().numpy()
    want = _oracle_perm(model, h, w, perm)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), \
        int(np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)))


def _oracle_perm(model, h, w, perm):
    _, out = O.query_batch(model, _NoTree(model.vocab_size), h[perm],
                           np.zeros((len(perm), model.maxent_order), np.int64),
                           np.zeros(len(perm), np.int32), w, want_p=False)
    return out


@pytest.mark.parametrize("V,H", [(20000, 256), (65536, 512)])
def test_word_logprob_fast_mode_within_spec(V, H, torch):
    """f32 lane-partial HS (used with the tensor-core modes): |d| <= 1e-5,
    inside the north star's 1e-4."""
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    from paper_2007_11794_b200.model import build_huffman_from_counts
    model = synth.synth_model(V, H, 20)
    tree = build_huffman_from_counts(synth.zipf_counts(V))
    dm = DeviceModel(model, tree)
    n = 4096
    h, hist, hl, w = _queries(model, n, seed=V + 1)
    want, _ = O.query_batch(model, tree, h, hist.astype(np.int64), hl, w, want_h=False)
    ctx = torch.arange(n, dtype=torch.int32, device="cuda")
    got = kernels.word_logprob_batch(dm, ctx, torch.from_numpy(h).cuda(), torch.from_numpy(hist).cuda(),
                                     torch.from_numpy(hl).cuda(), torch.from_numpy(w).cuda(),
                                     exact=False).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-5


@pytest.mark.parametrize("precision", ["fp64", "tf32x3", "bf16"])
def test_all_word_logprobs_batch(golden, precision):
    """Batched full-vocabulary scoring vs the reference's all_word_logprobs
    (kernels.npz q_all): fp64 |d| <= 1e-12; tcgen05 TF32X3 |d| <= 1e-5 per
    word; BF16 |d| <= 5e-2 (bf16 operands, the stated looser bound)."""
    import torch
    from conftest import GoldenModel
    from paper_2007_11794_b200 import kernels
    from paper_2007_11794_b200.device import DeviceModel
    d = golden("kernels")
    gm = GoldenModel(d)
    dm = DeviceModel(gm.model, gm.tree)
    k = d["q_all"].shape[0]
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()
    hist = np.where(d["q_hist"][:k] < 0, 0, d["q_hist"][:k]).astype(np.int32)
    ctx = t(np.arange(k)[::-1].copy(), np.int32)     # gathered rows, any order
    out = kernels.all_word_logprobs_batch(dm, ctx, t(d["q_h"][:k], np.float32), t(hist, np.int32),
                                          t(d["q_hl"][:k], np.int32), precision).cpu().numpy()
    want = d["q_all"][::-1]
    tol = {"fp64": 1e-12, "tf32x3": 1e-5, "bf16": 5e-2}[precision]
    assert np.abs(out - want).max() <= tol
    assert np.all(np.abs(np.exp(out).sum(axis=1) - 1.0) <= (1e-9 if precision == "fp64" else 1e-4))


@pytest.mark.parametrize("precision", ["fp64", "tf32x3"])
def test_all_word_logprobs_batch_config_c(precision):
    """V = 65,536, H = 512 (config c): 6 contexts vs the oracle; every
    distribution normalised (acceptance crit 1, tests/test_acceptance.py:74-86).
    TF32X3 bound: fp32 accumulation of 512 products per node activation
    (~5e-6) summed over paths of up to 20 nodes -> |d| <= 3e-4 per word."""
    import torch
    from oracle import oracle as O
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    from paper_2007_11794_b200.model import build_huffman_from_counts
    V, H, bits = 65536, 512, 22
    model = synth.synth_model(V, H, bits)
    tree = build_huffman_from_counts(synth.zipf_counts(V))
    dm = DeviceModel(model, tree)
    words, hidden, hist, hlen, _ = synth.query_set(model, 16, 6)
    hlen = np.array([0, 1, 2, 3, 3, 3], np.int32)
    t = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dt)).cuda()
    out = kernels.all_word_logprobs_batch(dm, t(np.arange(6), np.int32), t(hidden, np.float32),
                                          t(hist, np.int32), t(hlen, np.int32), precision).cpu().numpy()
    for i in range(6):
        want = O.all_word_logprobs(hidden[i], hist[i, :hlen[i]], tree.path_nodes, tree.path_signs,
                                   tree.path_offsets, model.node_vectors, model.maxent_table,
                                   model.maxent_order, model.hash_seed, model.maxent_size - 1)
        tol = 1e-11 if precision == "fp64" else 3e-4
        assert np.abs(out[i] - want).max() <= tol, (i, np.abs(out[i] - want).max())
        assert abs(np.exp(out[i]).sum() - 1.0) <= (1e-9 if precision == "fp64" else 1e-4)
