"""Full-size 1-best agreement: GPU (given precision) vs the exact oracle on
config-b utterances; for every disagreement, the oracle's own path score of
the GPU path vs the oracle's best (a tie within tolerance is allowed)."""
import json, sys
import numpy as np
from paper_2007_11794_b200 import synth
from paper_2007_11794_b200.rescore import BatchDecoder
from oracle import oracle as O

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
sched = sys.argv[3] if len(sys.argv) > 3 else "auto"
s = synth.build_setup("b", n_utt=n, T=300, seed=7)
need = BatchDecoder.contexts_needed(s.lattices, s.beam)
dec = BatchDecoder(s.model, s.tree, s.small_lm, n, need, precision=prec, schedule=sched)
dec.prepare(s.lattices, s.beam)
dec.run(1.0)
hyps, out = dec.fetch()
ref = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=s.beam)
om = O.OracleModel(s.model, s.tree)
og = O.OracleNgram(s.small_lm)
rows = []
for u in range(n):
    r = ref[u][0]
    same = hyps[u].arcs == r.arcs
    d = {"u": u, "same": same, "gpu_score": hyps[u].combined_score, "ref_score": r.combined_score}
    if not same:
        ol = O.OracleLattice(s.lattices[u])
        d["ref_score_of_gpu_path"] = O.path_score(om, s.tree, og, ol, hyps[u].arcs)
        d["gap"] = r.combined_score - d["ref_score_of_gpu_path"]
        # first divergence frame
        k = next((i for i, (a, b) in enumerate(zip(hyps[u].arcs, r.arcs)) if a != b), None)
        d["first_diff_frame"] = k
    d["abs_diff"] = abs(hyps[u].combined_score - r.combined_score)
    rows.append(d)
agree = sum(r["same"] for r in rows)
gaps = [r["gap"] for r in rows if not r["same"]]
print(json.dumps({"precision": prec, "schedule": dec.schedule, "agree": f"{agree}/{n}",
                  "max_gap_of_disagreements": max(gaps) if gaps else 0.0,
                  "max_abs_score_diff": max(r["abs_diff"] for r in rows), "rows": rows}))
