"""Per-phase device time of the stream kernel at config c geometry (H=512)."""
import json, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder
cfg = sys.argv[1] if len(sys.argv) > 1 else "c"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
s = synth.build_setup(cfg, n_utt=n, T=300, seed=17)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision="tf32x3")
dec.prepare(s.lattices, s.beam)
dec.run(1.0); torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(); dec.run(1.0); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
dec.profile(1.0)
ph = dec.plan.phase_ns()
print(json.dumps({"config": cfg, "n_utt": n, "ms": ms, "frames_per_s": n * 300 / (ms / 1e3),
                  "us_per_level": {k: round(v / max(ph["ctas"], 1) / 300 / 1e3, 2) for k, v in ph.items() if k != "ctas"}}))
