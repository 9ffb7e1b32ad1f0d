"""Utterance-sharded data parallelism.

Decoding shards naturally: every utterance is an independent stream with its
own IndexTable and cache, so ranks share nothing on the hot path.  The only
collective is the final gather of fixed-size per-utterance result records
(NCCL over NVLink on the GPU box; gloo in the CPU tests), merged
deterministically by utterance id.
"""

from __future__ import annotations

import numpy as np

REC_FIELDS = ("utt", "path_len", "combined", "acoustic", "lm", "end_ctx", "expansions")


def shard(n_total: int, world: int, rank: int) -> np.ndarray:
    """Contiguous balanced shard of utterance ids for ``rank``."""
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return np.arange(start, start + base + (1 if rank < extra else 0))


def pack_records(utt_ids, out: dict, max_path: int) -> np.ndarray:
    """[n, 7 + max_path] float64 records: fields + padded 1-best arc ids."""
    n = len(utt_ids)
    rec = np.full((n, len(REC_FIELDS) + max_path), -1.0)
    rec[:, 0] = utt_ids
    rec[:, 1] = out["path_len"][:n]
    for j, k in enumerate(("combined", "acoustic", "lm", "end_ctx", "expansions"), start=2):
        rec[:, j] = out[k][:n]
    arcs = out["path_arcs"]
    w = min(max_path, arcs.shape[1])
    rec[:, len(REC_FIELDS):len(REC_FIELDS) + w] = arcs[:n, :w]
    return rec


def gather_records(rec: np.ndarray, n_total: int, device=None) -> np.ndarray | None:
    """All-gather every rank's records (padded to the largest shard) and
    return them ordered by utterance id (on every rank)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    rows = -(-n_total // world)
    buf = np.full((rows, rec.shape[1]), -2.0)
    buf[:len(rec)] = rec
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    allr = torch.cat(parts).cpu().numpy()
    allr = allr[allr[:, 0] >= 0]
    return allr[np.argsort(allr[:, 0], kind="stable")]
