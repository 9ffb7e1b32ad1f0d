"""fp64 level schedule at fat 8 x 300: single run, then re-prepare + run."""
import torch

from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

s = synth.build_setup("b_fat", n_utt=8, T=300, seed=7)
need = BatchDecoder.contexts_needed(s.lattices, 64)
for prec in ("fp64", "tf32x3"):
    dec = BatchDecoder(s.model, s.tree, s.small_lm, 8, need, precision=prec, schedule="level")
    for i in range(3):
        try:
            dec.prepare(s.lattices, 64)
            dec.run(1.0)
            hyps, out = dec.fetch()
            print(prec, "run", i, "OK", int(out["expansions"].sum()), dec.streams.stats()[:, 3].tolist(), flush=True)
        except Exception as e:  # noqa: BLE001
            print(prec, "run", i, "FAIL", repr(e)[:200], flush=True)
            break
    del dec
    torch.cuda.empty_cache()
