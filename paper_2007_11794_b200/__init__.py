"""B200-native on-the-fly RNNLM rescoring (arXiv 2007.11794 hot path).

Drop-in for the reference package ``otflm``'s decoder/LM API: the same names
(reference ``__init__.py:24-61`` plus the decoder entry points) backed by
hand-written sm_100a kernels in ``libotflm_b200.so`` (C-ABI:
``include/otflm_b200.h``).  Host-side containers (models, trees, n-gram
tables, lattices) are plain numpy; all scoring, the context IndexTable and
the result cache run on the GPU.
"""

__version__ = "0.1.0"

from .model import (  # noqa: F401
    HuffmanTree,
    NgramModel,
    RnnlmContext,
    RnnlmModel,
    build_huffman,
    build_huffman_from_counts,
    ngram_logprob,
)
from .lattice import Arc, Lattice, LatticeFormatError, generate_lattice  # noqa: F401
from .rescore import (  # noqa: F401
    ENTRY_BYTES,
    BatchDecoder,
    CacheStats,
    CacheValue,
    IndexTable,
    PathHypothesis,
    RescoreCache,
    RescoreRequest,
    RescoreResponse,
    RescoreServer,
    RescoreStack,
    TransferLedger,
    TraversalReport,
    edit_distance,
    first_pass_weight,
    quantize_delta,
    rescored_path_score,
    small_context,
    pack,
    reduction_ratio,
    rescore_batch,
    rescore_onthefly,
    reset_utterance,
    rnnlm_prob,
    rnnlm_prob_trace,
    unpack,
)
from .twopass import (  # noqa: F401
    NbestArrays,
    TwopassPlan,
    nbest,
    nbest_arrays,
    nbest_batch,
    rescore_twopass,
    rescore_twopass_batch,
)
from ._lib import PackOverflowError, TableFullError, UnknownIndexError  # noqa: F401


def word_logprob(model, tree, ctx, w: int) -> float:
    """rnnlm.py:195-204 on the device."""
    from . import kernels
    w = int(w)
    if not 0 <= w < model.vocab_size:
        raise ValueError(f"word id {w} out of range 0..{model.vocab_size - 1}")
    o0, o1 = tree.path_offsets[w], tree.path_offsets[w + 1]
    return kernels.word_logprob(ctx.hidden, ctx.history, tree.path_nodes[o0:o1],
                                tree.path_signs[o0:o1], model.node_vectors, model.maxent_table,
                                model.maxent_order, model.hash_seed, model.maxent_size - 1)


def advance_context(model, ctx, w: int, precision: str = "fp64") -> RnnlmContext:
    """rnnlm.py:180-188 on the device."""
    from . import kernels
    w = int(w)
    if not 0 <= w < model.vocab_size:
        raise ValueError(f"word id {w} out of range 0..{model.vocab_size - 1}")
    h = kernels.advance_hidden(model.input_weights[w], model.recurrent_weights, ctx.hidden,
                               precision)
    return RnnlmContext(h, (tuple(ctx.history) + (w,))[-model.maxent_order:])


def compute_rnnlm(model, tree, ctx, w: int):
    """rnnlm.py:217-221: score w against ctx, then advance."""
    return word_logprob(model, tree, ctx, w), advance_context(model, ctx, w)
