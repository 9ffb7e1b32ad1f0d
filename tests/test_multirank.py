"""World-size-2 gloo test of the N>1 host path: utterance sharding, the
per-rank decode (CPU oracle standing in for the GPU decode, which needs a
device) and the results gather merged by utterance id."""

from __future__ import annotations

import os

import numpy as np
import torch.multiprocessing as mp

from paper_2007_11794_b200.parallel import gather_records, pack_records, shard


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("a", n_utt=5, T=12, seed=9)
    ids = shard(5, world, rank)
    res = O.decode_many(s.model, s.tree, s.small_lm, [s.lattices[i] for i in ids], beam=4,
                        n_threads=1)
    out = dict(path_len=np.array([len(r.arcs) for r, _ in res]),
               combined=np.array([r.combined_score for r, _ in res]),
               acoustic=np.array([r.acoustic_score for r, _ in res]),
               lm=np.array([r.lm_score for r, _ in res]),
               end_ctx=np.array([r.end_context for r, _ in res]),
               expansions=np.array([r.expansions for r, _ in res]),
               path_arcs=np.array([list(r.arcs) for r, _ in res]).reshape(len(res), -1))
    rec = pack_records(ids, out, 12)
    allr = gather_records(rec, 5)
    if rank == 0:
        q.put(allr)
    dist.barrier()
    dist.destroy_process_group()


def test_shards_cover_all_utterances():
    for n in (1, 5, 64, 4096):
        for w in (1, 2, 4, 8):
            ids = np.concatenate([shard(n, w, r) for r in range(w)])
            assert np.array_equal(ids, np.arange(n))


def test_two_rank_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allr = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    from oracle import oracle as O
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("a", n_utt=5, T=12, seed=9)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=4, n_threads=1)
    assert allr.shape[0] == 5
    assert list(allr[:, 0]) == [0, 1, 2, 3, 4]
    for u, (r, _) in enumerate(ref):
        assert allr[u, 2] == r.combined_score
        n = int(allr[u, 1])
        assert tuple(int(a) for a in allr[u, 7:7 + n]) == r.arcs
