import sys; sys.path.insert(0, ".")
import time, json
import numpy as np
import torch
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder
from paper_2007_11794_b200.device import pack_lattices
s = synth.build_setup("b", n_utt=64, T=300, seed=7)
b2 = synth.more_lattices(s, 64, 300, seed=99)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
dec = BatchDecoder(s.model, s.tree, s.small_lm, 64, need, precision="tf32x3", n_buffers=2)
for i in range(3):
    sl = dec.prepare([s.lattices, b2][i % 2], s.beam); dec.run(1.0, slot=sl); dec.fetch(slot=sl)
torch.cuda.synchronize()
T = {}
def tm(k, f):
    t = time.perf_counter(); r = f(); T.setdefault(k, []).append(1e3 * (time.perf_counter() - t)); return r
for i in range(5):
    tm("pack", lambda: pack_lattices(b2))
    sl = tm("prepare_total", lambda: dec.prepare(b2, s.beam))
    tm("run_enqueue", lambda: dec.run(1.0, slot=sl))
    torch.cuda.synchronize()
    tm("fetch", lambda: dec.fetch(slot=sl))
    p = dec.plans[0]
    tm("refresh_only", lambda: p.refresh(b2, stream_ids=dec.spans[0]))
    torch.cuda.synchronize()
print(json.dumps({k: round(float(np.median(v)), 3) for k, v in T.items()}))
