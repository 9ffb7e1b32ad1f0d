"""Config-e batch (148 utterances x 300 frames, EXACT) per schedule: device
time of one decode (events around BatchDecoder.run, after a warm-up run).
    python tools/sched_e.py [N_UTT]"""
import json
import sys
sys.path.insert(0, ".")
import torch
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
s = synth.build_setup("e", n_utt=1, T=300, seed=31)
s.lattices = synth.lattices_for_ids(s, range(n), 300)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
for sched, groups in (("stream1", 1), ("level", 1), ("level", 2), ("level", 4)):
    dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision="exact", schedule=sched, n_groups=groups)
    dec.prepare(s.lattices, s.beam)
    dec.run(1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        dec.run(1.0)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    hyps, out = dec.fetch()
    fr = sum(len(h.arcs) for h in hyps)
    ms = min(ts)
    print(json.dumps({"schedule": sched, "groups": groups, "ms": round(ms, 2), "frames_per_s": round(fr / ms * 1e3)}),
          flush=True)
    del dec
    torch.cuda.empty_cache()
