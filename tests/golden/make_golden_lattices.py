"""Golden lattices from the REFERENCE generator (otflm.lattice.generate_lattice,
lattice.py:130-183): the repo's vectorised generator (paper_2007_11794_b200.
lattice.generate_lattice, used by the synthetic bench inputs) must produce
the same arcs (src, dst, word, acoustic, small-LM score), start and finals
for the same reference words, small LM, breadth and noise seed.

Run in the build container, where /root/reference is mounted:

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_lattices.py

Output: tests/golden/lattices.npz (committed; nothing at test time reads
/root/reference).  Cases: a bigram and a trigram Kneser-Ney small LM over a
2,000-word Zipf corpus vocabulary, breadths 1 / 2 / 3 / 8, 6-40 positions.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from make_golden import lattice_arrays, ngram_tables  # noqa: E402
from otflm.lattice import generate_lattice  # noqa: E402
from otflm.ngram import train_ngram  # noqa: E402
from otflm.synth import zipfian_corpus  # noqa: E402
from otflm.vocab import build_vocabulary  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    lines = zipfian_corpus(600, 2000, seed=41)
    vocab = build_vocabulary(lines)
    d = {"V": np.int32(vocab.size)}
    cases = []
    for oi, order in enumerate((2, 3)):
        lm = train_ngram(lines, vocab, order, smoothing="kneser-ney")
        d.update({f"o{oi}_{k}": v for k, v in ngram_tables(lm).items()})
        rng = np.random.RandomState(5 + oi)
        for ci, (breadth, T) in enumerate(((1, 6), (2, 12), (3, 40), (8, 9), (3, 25))):
            ref = [int(w) for w in rng.randint(3, vocab.size, size=T)]
            seed = int(rng.randint(0, 1 << 30))
            lat = generate_lattice(ref, vocab, lm, breadth, seed)
            p = f"o{oi}_c{ci}_"
            d.update(lattice_arrays(lat, p))
            d[p + "ref"] = np.array(ref, np.int32)
            d[p + "breadth"] = np.int32(breadth)
            d[p + "seed"] = np.int64(seed)
            cases.append(p)
    d["cases"] = np.array(cases)
    np.savez_compressed(OUT / "lattices.npz", **d)
    print("wrote", OUT / "lattices.npz", len(cases), "lattices")


if __name__ == "__main__":
    main()
