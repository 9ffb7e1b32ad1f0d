"""One all_word_logprobs_batch call per precision (for the ncu launch list)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2007_11794_b200 import kernels, synth
from paper_2007_11794_b200.device import DeviceModel
from paper_2007_11794_b200.model import build_huffman_from_counts
V, H, bits, n = 65536, 512, 22, 256
model = synth.synth_model(V, H, bits)
tree = build_huffman_from_counts(synth.zipf_counts(V))
dm = DeviceModel(model, tree)
_, hidden, hist, hlen, _ = synth.query_set(model, 16, n)
d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
ctx = d(np.arange(n, dtype=np.int32))
for prec in sys.argv[1:] or ["fp64", "tf32x3"]:
    kernels.all_word_logprobs_batch(dm, ctx, d(hidden), d(hist), d(hlen), prec)
torch.cuda.synchronize()
