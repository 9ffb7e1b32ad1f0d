"""One stream-schedule decode (profiling target): python tools/decode_once.py CONFIG N_UTT FRAMES PRECISION [REPS]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

cfg, n, T, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
s = synth.build_setup(cfg, n_utt=n, T=T, seed=7)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision=prec, schedule="stream")
dec.prepare(s.lattices, s.beam)
for _ in range(reps):
    dec.run(1.0)
torch.cuda.synchronize()
hyps, out = dec.fetch()
print("ok", sum(len(h.arcs) for h in hyps), dec.counters())
