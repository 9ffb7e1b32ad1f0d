"""Fat-variant (breadth 16, beam 64) device decode timing probe."""
import json
import sys
import time

import torch

from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

n_utt, T = int(sys.argv[1]), int(sys.argv[2])
s = synth.build_setup("b_fat", n_utt=n_utt, T=T, seed=7)
need = BatchDecoder.contexts_needed(s.lattices, 64)
for prec, sched in (("tf32x3", "level"), ("tf32x3", "stream"), ("fp64", "level")):
    dec = BatchDecoder(s.model, s.tree, s.small_lm, n_utt, need, precision=prec, schedule=sched)
    dec.prepare(s.lattices, 64)
    dec.run(1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        dec.prepare(s.lattices, 64)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dec.run(1.0); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    hyps, out = dec.fetch()
    exp = int(out["expansions"].sum())
    ms = min(ts)
    print(json.dumps({"precision": prec, "schedule": dec.schedule, "n_utt": n_utt, "T": T, "contexts": need,
                      "ms": ms, "frames_per_s": n_utt * T / (ms / 1e3), "requests": exp,
                      "requests_per_s": exp / (ms / 1e3)}), flush=True)
    del dec
    torch.cuda.empty_cache()
