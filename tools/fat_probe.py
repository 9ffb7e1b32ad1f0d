"""Fat-variant (breadth 16, beam 64) decode at full length in one precision /
schedule: reports success + counters or the decode error (GPU probe):
    python tools/fat_probe.py N_UTT FRAMES PRECISION SCHEDULE"""
import json
import sys
import time
sys.path.insert(0, ".")
import torch
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder

n, T, prec, sched = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
s = synth.build_setup("b_fat", n_utt=n, T=T, seed=3)
need = BatchDecoder.contexts_needed(s.lattices, 64)
res = {"n": n, "T": T, "precision": prec, "schedule": sched, "contexts_needed": int(need)}
try:
    dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision=prec, schedule=sched)
    dec.prepare(s.lattices, 64)
    t0 = time.perf_counter()
    dec.run(1.0)
    hyps, out = dec.fetch()
    torch.cuda.synchronize()
    res["s"] = round(time.perf_counter() - t0, 3)
    st = dec.streams.stats()
    res["ok"] = True
    res["requests"] = int(out["expansions"].sum())
    res["table_len"] = [int(x) for x in st[:, 3]]
    res["scores"] = [h.combined_score for h in hyps]
    res["arcs_hash"] = [hash(tuple(h.arcs)) & 0xFFFFFFFF for h in hyps]
except Exception as e:          # noqa: BLE001 -- the probe reports the failure
    res["ok"] = False
    res["error"] = repr(e)
print(json.dumps(res))
