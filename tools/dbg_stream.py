import sys, time
import numpy as np
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder
name = sys.argv[1] if len(sys.argv) > 1 else "a"
n_utt, T = int(sys.argv[2]) if len(sys.argv) > 2 else 2, int(sys.argv[3]) if len(sys.argv) > 3 else 5
s = synth.build_setup(name, n_utt=n_utt, T=T, seed=5)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
res = {}
for sched in ("level", "stream"):
    dec = BatchDecoder(s.model, s.tree, s.small_lm, len(s.lattices), need, precision="tf32x3", schedule=sched)
    dec.prepare(s.lattices, s.beam)
    t = time.time()
    dec.run(1.0)
    import torch; torch.cuda.synchronize()
    print(sched, "run s", time.time() - t, flush=True)
    hyps, out = dec.fetch()
    res[sched] = (hyps, out, dec.streams.stats())
    print(sched, [h.arcs[:6] for h in hyps][:2], [h.combined_score for h in hyps][:4], flush=True)
    print(sched, res[sched][2][:, :4].tolist()[:4], flush=True)
