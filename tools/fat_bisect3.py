"""fp64 level schedule, fat variant, T=300: which batch sizes overflow."""
import torch

from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

for n_utt, T in [(1, 300), (2, 300), (3, 300), (4, 300), (8, 150)]:
    s = synth.build_setup("b_fat", n_utt=n_utt, T=T, seed=7)
    need = BatchDecoder.contexts_needed(s.lattices, 64)
    try:
        dec = BatchDecoder(s.model, s.tree, s.small_lm, n_utt, need, precision="fp64", schedule="level")
        dec.prepare(s.lattices, 64)
        dec.run(1.0)
        hyps, out = dec.fetch()
        print(n_utt, T, "OK rows", n_utt * need, int(out["expansions"].sum()), flush=True)
        del dec
    except Exception as e:  # noqa: BLE001
        print(n_utt, T, "FAIL rows", n_utt * need, repr(e)[:120], flush=True)
    torch.cuda.empty_cache()
