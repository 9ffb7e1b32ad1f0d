"""Operator table mirror of the reference ``otflm.kernels`` (kernels.py:30-36).

Same names and arguments as the numba kernels; each call runs the sm_100a
kernel through libotflm_b200.so.  ``BACKEND`` is always ``"cuda-sm100a"``:
there is no import-time CPU alternative (kernels.py:13-28 selects numba or
numpy; this table selects nothing).  Batched entry points (``*_batch``) are
the ones the decoder uses; the single-call forms exist for drop-in parity.
Training kernels (sentence_loss/grads, train_sentence) are out of scope.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .device import DeviceModel, cuda, current_stream_ptr

BACKEND = "cuda-sm100a"
NUMBA_DISABLED = True


def _t(x, dtype):
    torch = cuda()
    a = np.ascontiguousarray(x)
    if not a.flags.writeable:            # read-only views (np.frombuffer, np.load): copy, torch needs writable
        a = a.copy()
    return torch.as_tensor(a, dtype=dtype, device="cuda")


class _ArraysModel:
    """Duck-typed model for uploading only the arrays a call needs."""

    def __init__(self, H, V, order, M, seed, U=None, W=None, NV=None, ME=None):
        self.hidden_size, self.vocab_size, self.maxent_order = H, V, order
        self.maxent_size, self.hash_seed = M, seed
        self.input_weights, self.recurrent_weights = U, W
        self.node_vectors, self.maxent_table = NV, ME


_arr_cache: dict = {}


def _model_for(key, build):
    ent = _arr_cache.get(key)
    if ent is None:
        if len(_arr_cache) > 16:
            _arr_cache.clear()
        ent = build()
        _arr_cache[key] = ent
    return ent[-1]


def _akey(*arrays):
    return tuple((a.__array_interface__["data"][0], a.shape, a.dtype.str) for a in arrays)


def feature_index(seed, order_k, words, node_id, mask) -> np.uint64:
    """_kernels_nb.py:27-33 (bit-exact)."""
    words = np.asarray(words, dtype=np.int64)
    out = feature_index_batch(int(seed), int(mask), np.array([int(order_k)]),
                              words.reshape(1, -1), np.array([int(node_id)]))
    return np.uint64(out[0])


def feature_index_batch(seed: int, mask: int, order_k, words, nodes) -> np.ndarray:
    torch = cuda()
    L = _lib.load()
    n = len(order_k)
    w = np.zeros((n, 8), np.int64)
    words = np.asarray(words, np.int64)
    w[:, :words.shape[1]] = words
    ok = _t(np.asarray(order_k, np.int32), torch.int32)
    wd = _t(w, torch.int64)
    nd = _t(np.asarray(nodes, np.int64), torch.int64)
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.check(L.otflm_feature_index_batch(int(seed) & (2**64 - 1), int(mask) & (2**64 - 1), n,
                                           ok.data_ptr(), wd.data_ptr(), nd.data_ptr(),
                                           out.data_ptr(), current_stream_ptr()), "feature_index")
    return out.cpu().numpy().view(np.uint64)


def advance_hidden(input_row, recurrent, hidden, precision: str = "fp64") -> np.ndarray:
    """_kernels_nb.py:51-60: f32(sigmoid(input_row + recurrent @ hidden))."""
    torch = cuda()
    W = np.ascontiguousarray(recurrent, np.float32)
    H = W.shape[0]
    dm = _model_for(("W",) + _akey(W), lambda: (W, DeviceModel(
        _ArraysModel(H, 2, 1, 1, 0, W=W, U=np.zeros((2, H), np.float32)), None, output=False)))
    rows = _t(np.asarray(input_row, np.float32).reshape(1, H), torch.float32)
    h = _t(np.asarray(hidden, np.float32).reshape(1, H), torch.float32)
    ctx = _t(np.zeros(1, np.int32), torch.int32)
    out = torch.empty((1, H), dtype=torch.float32, device="cuda")
    _lib.check(_lib.load().otflm_advance_hidden_rows(dm.handle, 1, rows.data_ptr(), ctx.data_ptr(),
                                                     h.data_ptr(), out.data_ptr(),
                                                     _lib.PREC[precision], current_stream_ptr()),
               "advance_hidden")
    return out.cpu().numpy()[0]


def _output_model(node_vectors, maxent_table, maxent_order, seed):
    NV = np.ascontiguousarray(node_vectors, np.float32)
    ME = np.ascontiguousarray(maxent_table, np.float32)
    key = ("O",) + _akey(NV, ME) + (int(maxent_order), int(seed))
    return _model_for(key, lambda: (NV, ME, DeviceModel(
        _ArraysModel(NV.shape[1], NV.shape[0] + 1, int(maxent_order), ME.shape[0], int(seed),
                     NV=NV, ME=ME), None, recurrent=False)))


def word_logprob(hidden, history, nodes, signs, node_vectors, maxent_table, maxent_order, seed,
                 mask) -> float:
    """_kernels_nb.py:78-86 for one explicit path."""
    torch = cuda()
    ME = np.asarray(maxent_table)
    if int(mask) != ME.shape[0] - 1:
        raise ValueError("mask must equal maxent_size - 1")
    dm = _output_model(node_vectors, maxent_table, maxent_order, seed)
    H = dm.H
    hist = np.asarray(history, np.int64)
    order = dm.order
    hrow = np.zeros((1, order), np.int32)
    n = min(len(hist), order) if len(hist) <= order else order
    # the kernel keeps the last `order` words like the reference slices do
    hh = hist[-order:] if len(hist) > order else hist
    hrow[0, :len(hh)] = hh
    hl = np.array([len(hh)], np.int32)
    codes = (np.asarray(nodes, np.int64) & 0x7FFFFFFF).astype(np.uint32)
    codes |= (np.asarray(signs, np.float32) < 0).astype(np.uint32) << np.uint32(31)
    off = np.array([0, len(codes)], np.int64)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    args = [_t(np.zeros(1, np.int32), torch.int32), _t(np.asarray(hidden, np.float32).reshape(1, H),
                                                       torch.float32),
            _t(hrow, torch.int32), _t(hl, torch.int32), _t(off, torch.int64),
            _t(codes.view(np.int32), torch.int32)]
    _lib.check(_lib.load().otflm_word_logprob_paths(dm.handle, 1, *[a.data_ptr() for a in args],
                                                    out.data_ptr(), current_stream_ptr()),
               "word_logprob")
    return float(out.cpu().numpy()[0])


def all_word_logprobs(hidden, history, path_nodes, path_signs, path_offsets, node_vectors,
                      maxent_table, maxent_order, seed, mask) -> np.ndarray:
    """_kernels_nb.py:89-104."""
    torch = cuda()

    class _Tree:
        pass

    tree = _Tree()
    tree.path_nodes = np.asarray(path_nodes, np.int32)
    tree.path_signs = np.asarray(path_signs, np.float32)
    tree.path_offsets = np.asarray(path_offsets, np.int64)
    NV = np.ascontiguousarray(node_vectors, np.float32)
    ME = np.ascontiguousarray(maxent_table, np.float32)
    key = ("A",) + _akey(NV, ME, tree.path_nodes, tree.path_offsets) + (int(maxent_order), int(seed))
    dm = _model_for(key, lambda: (NV, ME, tree, DeviceModel(
        _ArraysModel(NV.shape[1], NV.shape[0] + 1, int(maxent_order), ME.shape[0], int(seed),
                     NV=NV, ME=ME), tree, recurrent=False)))
    hist = np.asarray(history, np.int32)
    h = _t(np.asarray(hidden, np.float32), torch.float32)
    out = torch.empty(dm.V, dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().otflm_all_word_logprobs(dm.handle, h.data_ptr(), hist.ctypes.data,
                                                   len(hist), out.data_ptr(), current_stream_ptr()),
               "all_word_logprobs")
    return out.cpu().numpy()


# --- batched forms used by the decoder and the query microbenchmark -------

def word_logprob_batch(dmodel: DeviceModel, ctx, h, hist, hist_len, words, exact: bool = True,
                       out=None):
    """Device tensors in, device float64 tensor out (query i: context ctx[i]).
    exact=True: float64 accumulation (|d| <= 1e-12); False: f32 lane partials."""
    torch = cuda()
    n = int(words.shape[0])
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=words.device)
    _lib.check(_lib.load().otflm_word_logprob_batch2(dmodel.handle, n, ctx.data_ptr(), h.data_ptr(),
                                                     hist.data_ptr(), hist_len.data_ptr(),
                                                     words.data_ptr(), out.data_ptr(), int(bool(exact)),
                                                     current_stream_ptr()), "word_logprob_batch")
    return out


def ngram_logprob_batch(dngram, ctx, words, out=None):
    """ngram_logprob (ngram.py:161-179) for n (context, word) pairs on the
    device small-LM hash: ctx int32 [n, order-1] already left-padded with
    <s> (small_context, decoder.py:73-80), words int32 [n]; float64 [n] out.
    KeyError for a word missing from the unigram table, ValueError for a bad
    id (the reference's exceptions)."""
    torch = cuda()
    n = int(words.shape[0])
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=words.device)
    _lib.check(_lib.load().otflm_ngram_logprob_batch(dngram.handle, n, ctx.data_ptr(), words.data_ptr(),
                                                     out.data_ptr(), current_stream_ptr()), "ngram_logprob_batch")
    return out


def advance_hidden_batch(dmodel: DeviceModel, ctx, h, words, precision: str = "fp64", out=None):
    torch = cuda()
    n = int(words.shape[0])
    if out is None:
        out = torch.empty((n, dmodel.H), dtype=torch.float32, device=words.device)
    _lib.check(_lib.load().otflm_advance_hidden_batch(dmodel.handle, n, ctx.data_ptr(), h.data_ptr(),
                                                      words.data_ptr(), out.data_ptr(),
                                                      _lib.PREC[precision], current_stream_ptr()),
               "advance_hidden_batch")
    return out


def all_word_logprobs_batch(dmodel: DeviceModel, ctx, h, hist, hist_len, precision: str = "fp64",
                            out=None):
    """all_word_logprobs (_kernels_nb.py:89-104) for n contexts: device
    tensors in, float64 [n, V] out.  precision "fp64": float64 CUDA-core dot
    products; a tensor-core mode: the [n x (V-1)] node activations are one
    tcgen05 GEMM against the node vectors."""
    torch = cuda()
    n = int(ctx.shape[0])
    if out is None:
        out = torch.empty((n, dmodel.V), dtype=torch.float64, device=ctx.device)
    _lib.check(_lib.load().otflm_all_word_logprobs_batch(dmodel.handle, n, ctx.data_ptr(), h.data_ptr(),
                                                         hist.data_ptr(), hist_len.data_ptr(),
                                                         out.data_ptr(), _lib.PREC[precision],
                                                         current_stream_ptr()),
               "all_word_logprobs_batch")
    return out
