"""The N>1 device path with two ranks on one B200 (gloo for the gather, since
NCCL refuses two ranks on one device; the ranks' kernels never wait on each
other -- each decodes its own utterance shard): utterance
sharding (parallel.shard), the per-rank EXACT device decode through the
public BatchDecoder, the fixed-size result records (parallel.pack_records)
and the all-gather merged by utterance id (parallel.gather_records) --
identical to the oracle decode of every utterance (1-best arcs, end
context, expansions; scores within 1e-9)."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_UTT, T, BEAM = 7, 40, 8


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2007_11794_b200 import parallel, synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("b", n_utt=N_UTT, T=T, seed=13)
    ids = parallel.shard(N_UTT, world, rank)
    lats = [s.lattices[i] for i in ids]
    need = BatchDecoder.contexts_needed(lats, BEAM)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(lats), need, precision="exact")
    dec.prepare(lats, BEAM)
    dec.run(1.0)
    hyps, out = dec.fetch()
    torch.cuda.synchronize()
    o = {k: v[:len(ids)] for k, v in out.items()}
    # the records carry each utterance's own arc ids (out["path_arcs"] holds
    # the batch's global ids; the hypotheses are already per lattice)
    arcs = np.full((len(ids), T), -1)
    for i, h in enumerate(hyps[:len(ids)]):
        arcs[i, :len(h.arcs)] = h.arcs
    o["path_arcs"] = arcs
    rec = parallel.pack_records(ids, o, T)
    allr = parallel.gather_records(rec, N_UTT)
    if rank == 0:
        q.put((allr, dec.schedule))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_device_decode_and_gather_match_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    allr, sched = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    from oracle import oracle as O
    from paper_2007_11794_b200 import synth
    s = synth.build_setup("b", n_utt=N_UTT, T=T, seed=13)
    ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=BEAM, n_threads=2)
    assert allr.shape[0] == N_UTT
    assert list(allr[:, 0]) == list(range(N_UTT))
    for u, (r, _) in enumerate(ref):
        n = int(allr[u, 1])
        assert tuple(int(a) for a in allr[u, 7:7 + n]) == r.arcs, (u, sched)
        assert abs(allr[u, 2] - r.combined_score) <= 1e-9
        assert int(allr[u, 5]) == r.end_context and int(allr[u, 6]) == r.expansions
