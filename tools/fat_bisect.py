"""Which fat-variant sizes make the level schedule report a digest collision."""
import sys

import torch

from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

for n_utt, T, prec, sched in [(8, 10, "fp64", "level"), (4, 60, "fp64", "level"), (8, 60, "fp64", "level"),
                              (8, 60, "tf32x3", "level"), (16, 10, "fp64", "level"), (8, 300, "tf32x3", "level")]:
    s = synth.build_setup("b_fat", n_utt=n_utt, T=T, seed=7)
    need = BatchDecoder.contexts_needed(s.lattices, 64)
    try:
        dec = BatchDecoder(s.model, s.tree, s.small_lm, n_utt, need, precision=prec, schedule=sched)
        dec.prepare(s.lattices, 64)
        dec.run(1.0)
        hyps, out = dec.fetch()
        R = max(int(x) for x in dec.plan_info()["lvl_req"]) if hasattr(dec, "plan_info") else -1
        print(n_utt, T, prec, sched, "OK", need, int(out["expansions"].sum()), flush=True)
    except Exception as e:  # noqa: BLE001
        print(n_utt, T, prec, sched, "FAIL", need, repr(e)[:200], flush=True)
    del s
    torch.cuda.empty_cache()
