"""Near-tie sensitivity of the config-b bench workload, on the CPU oracle.

Decodes the bench's 64 x 300-frame config-b batch with the exact oracle
twice: with the model as built, and with every recurrent weight moved by one
f32 ulp in a random direction (a perturbation of the contraction of the same
order as the f32-accumulated tensor-core contraction's error).  Counts the
utterances whose 1-best changes and the oracle score gaps, i.e. how many
beam-pruning decisions in this workload tie within fp32 noise.
"""
import dataclasses
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_2007_11794_b200 import synth  # noqa: E402

s = synth.build_setup("b", n_utt=64, T=300, seed=7)
base = O.decode_many(s.model, s.tree, s.small_lm, s.lattices, beam=8)
res = {}
for seed in (1, 2):
    rng = np.random.default_rng(seed)
    W = np.asarray(s.model.recurrent_weights, np.float32)
    Wp = np.where(rng.random(W.shape) < 0.5, np.nextafter(W, np.float32(np.inf)),
                  np.nextafter(W, np.float32(-np.inf))).astype(np.float32)
    mp = dataclasses.replace(s.model, recurrent_weights=Wp)
    t0 = time.time()
    pert = O.decode_many(mp, s.tree, s.small_lm, s.lattices, beam=8)
    om, og = O.OracleModel(s.model, s.tree), O.OracleNgram(s.small_lm)
    gaps = []
    for u, ((r, _), (p, _)) in enumerate(zip(base, pert)):
        if r.arcs != p.arcs:
            gaps.append(round(O.path_score(om, None, og, s.lattices[u], p.arcs) - r.combined_score, 4))
    res[f"seed{seed}"] = {"identical": 64 - len(gaps), "gaps": sorted(gaps), "s": round(time.time() - t0, 1)}
    print(json.dumps(res[f"seed{seed}"]), flush=True)
json.dump(res, open("profiles/r01q_perturb_ties.json", "w"), indent=1)
