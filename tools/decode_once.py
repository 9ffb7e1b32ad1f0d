"""One stream-schedule decode (profiling target), then a profiled replay for
the algorithmic-work counters:
    python tools/decode_once.py CONFIG N_UTT FRAMES PRECISION [REPS]
CONFIG e uses the bench's per-utterance-id lattices (bench.py run_config_e)."""
import json
import sys
sys.path.insert(0, ".")
import torch
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

cfg, n, T, prec = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
if cfg == "e":
    s = synth.build_setup("e", n_utt=1, T=T, seed=31)
    s.lattices = synth.lattices_for_ids(s, range(n), T)
else:
    s = synth.build_setup(cfg, n_utt=n, T=T, seed=7)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision=prec, schedule="auto")
dec.prepare(s.lattices, s.beam)
for _ in range(reps):
    dec.run(1.0)
torch.cuda.synchronize()
hyps, out = dec.fetch()
prof = dec.profile(1.0)
cnt = dec.counters()
st = dec.streams.stats()
print(json.dumps({"frames": int(sum(len(h.arcs) for h in hyps)), "requests": int(out["expansions"].sum()),
                  "misses": int(st[:, 2].sum()), "H": s.model.hidden_size, "counters": cnt,
                  "kernel_ms": {k: v[0] for k, v in prof.items()}, "schedule": dec.schedule}))
