#!/usr/bin/env python3
"""On-the-fly RNNLM rescoring benchmark (BASELINE.json metric: decode frames/s
& RTF; RNNLM (history, word) queries/s per GPU).

Default workload (the largest single-GPU configuration, BASELINE.json
configs[4] / SURVEY.md §8d config e): synthetic HS+MaxEnt RNNLM with
V=65,536, H=512, MaxEnt 2^22, 4,096 utterances x 300 frames (one lattice
step = one 10 ms frame), breadth 3, beam 8, bigram small LM, fresh streams
per utterance.  The utterances are sharded over the ranks (strong scaling:
the total is fixed); each rank decodes its shard in batches of 148 streams
(one CTA per stream on each of the 148 SMs, k_decode_solo) through the
double-buffered BatchDecoder, in the EXACT precision (integer digit-plane
tcgen05 update with certified rounding + digit-plane HS: every hidden state
and 1-best identical to the reference).  NCCL only all-gathers the per-utterance result records.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--precision P] [--config e|b]
  python bench.py --impl reference      # CPU arm: the reference algorithm on host cores

--gpus N without torchrun re-launches itself under torch.distributed.run.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FRAME_S = 0.01          # one lattice step = one 10 ms frame
CONFIG = "b"
METRIC = "decode frames/sec (RNNLM on-the-fly rescoring, config b: V=20k H=256 HS+MaxEnt 2^21, " \
         "64 utt x 300 frames, beam 8)"
METRIC_E = "decode frames/sec (RNNLM on-the-fly rescoring, config e: V=64k H=512 HS+MaxEnt 2^22, " \
           "4096 utt x 300 frames, beam 8)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--precision", default="exact", choices=["exact", "fp64", "tf32x3", "tf32", "bf16"])
    ap.add_argument("--n-utt", type=int, default=64)
    ap.add_argument("--frames", type=int, default=300)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--groups", type=int, default=4, help="concurrent level chains per GPU (level schedule)")
    ap.add_argument("--schedule", default="auto", choices=["auto", "level", "stream", "stream1"],
                    help="decode schedule: persistent per-stream kernel or level-synchronous graph")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-queries", action="store_true", help="skip the config-d query microbench")
    ap.add_argument("--beam-sweep", action="store_true", help="add the config-c beam sweep extra")
    ap.add_argument("--no-wide", action="store_true",
                    help="config e: skip the config-c beam sweep and fat-variant extras")
    ap.add_argument("--table4", action="store_true", help="add the Table-4 cache-capacity sweep extra")
    ap.add_argument("--config", default="e", choices=["b", "e"],
                    help="b: the headline config (default); e: 4096 utterances at V=64k sharded over ranks")
    ap.add_argument("--e-total", type=int, default=4096, help="config e: total utterances")
    ap.add_argument("--e-batch", type=int, default=148,
                    help="config e: streams decoded at once per GPU (148: one CTA per stream per SM; "
                         "<= 74 selects the 2-CTA cluster kernel)")
    ap.add_argument("--all-word", action="store_true", help="add the all_word_logprobs extra")
    ap.add_argument("--twopass-n", type=int, default=1000, help="n-best size of the two-pass extra (0: skip)")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            "MEASURED_PEAKS.json"
    return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def query_microbench(precision: str, n_queries: int = 1 << 20, n_ctx: int = 1 << 18, reps: int = 5):
    """Config (d): isolated LM queries -- n (history, word) pairs through the
    HS + MaxEnt kernel and the recurrent update, inputs resident in HBM, L2
    flushed before every timed launch.  Algorithmic HS bytes per query:
    P(4H + 4k + 8) + 4H + 16."""
    import torch
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    from paper_2007_11794_b200.model import build_huffman_from_counts
    cfg = synth.CONFIGS["d"]
    V, H, bits = cfg["V"], cfg["H"], cfg["bits"]
    model = synth.synth_model(V, H, bits)
    tree = build_huffman_from_counts(synth.zipf_counts(V))
    dm = DeviceModel(model, tree)
    words, hidden, hist, hlen, ctx = synth.query_set(model, n_queries, n_ctx)
    d = lambda x: torch.from_numpy(x).cuda()
    tw, th, thist, thl, tctx = d(words), d(hidden), d(hist), d(hlen), d(ctx)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    out = torch.empty(n_queries, dtype=torch.float64, device="cuda")
    hout = torch.empty((n_queries, H), dtype=torch.float32, device="cuda")

    def timed(fn):
        fn()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    hs_ms = timed(lambda: kernels.word_logprob_batch(dm, tctx, th, thist, thl, tw, exact=True, out=out))
    hs_fast_ms = timed(lambda: kernels.word_logprob_batch(dm, tctx, th, thist, thl, tw, exact=False, out=out))
    adv_ms = timed(lambda: kernels.advance_hidden_batch(dm, tctx, th, tw, precision, out=hout))
    P = (tree.path_offsets[1:] - tree.path_offsets[:-1])[words]
    k = np.minimum(hlen[ctx], model.maxent_order)
    hs_bytes = float(np.sum(P * (4 * H + 4 * k + 8)) + n_queries * (4 * H + 16))
    hbm, tc_peak, src = peaks()
    gbs = hs_bytes / (hs_ms / 1e3) / 1e9
    gbs_fast = hs_bytes / (hs_fast_ms / 1e3) / 1e9
    flops = 2.0 * H * H * n_queries
    tfs = flops / (adv_ms / 1e3) / 1e12
    return {"workload": f"config d: {n_queries} queries, {n_ctx} contexts, V={V} H={H} MaxEnt 2^{bits}, "
                        "words ~ Zipf(1.05); L2 flushed before each launch",
            "hs_exact_ms": hs_ms, "hs_exact_gbs": gbs, "hs_exact_frac_of_hbm": gbs / hbm,
            "hs_fast_ms": hs_fast_ms, "hs_fast_gbs": gbs_fast, "hs_fast_frac_of_hbm": gbs_fast / hbm,
            "hs_bytes": hs_bytes,
            "mean_path": float(P.mean()),
            "advance_ms": adv_ms, "advance_tflops": tfs, "advance_frac_of_bf16_peak": tfs / tc_peak,
            "advance_precision": precision,
            "queries_per_s": n_queries / ((min(hs_ms, hs_fast_ms) + adv_ms) / 1e3), "peak_source": src}


def twopass_microbench(setup, precision: str, n: int, reps: int = 5):
    """Two-pass rescoring (decoder.py:180-274) on the
    config-(b) batch: n-best lists of every utterance (host search in
    libotflm_b200.so), merged prefix tries, device scoring (rnnlm mode).
    Device time has the tries resident in HBM (L2 flushed before each run);
    e2e = n-best search + trie build + H2D + device scoring + D2H."""
    import torch
    from oracle import oracle as O
    from paper_2007_11794_b200.twopass import TwopassPlan, nbest_arrays
    m = setup.model
    H = m.hidden_size
    t0 = time.perf_counter()
    nb = nbest_arrays(setup.lattices, n, 1.0)
    t_nbest = time.perf_counter() - t0
    t0 = time.perf_counter()
    plan = TwopassPlan(m, setup.tree, None, nb)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    info = plan.info()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    plan.run("rnnlm", 0.5, 1.0, precision)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        plan.run("rnnlm", 0.5, 1.0, precision)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    dev_ms = float(np.median(ts))
    t0 = time.perf_counter()
    lm, comb, best = plan.fetch()
    t_fetch = time.perf_counter() - t0
    e2e_s = t_nbest + t_build + dev_ms / 1e3 + t_fetch
    # algorithmic bytes: every trie node is one HS query (mean path P over its
    # words) + every internal node one update (h, U row in, h' out)
    pl = (setup.tree.path_offsets[1:] - setup.tree.path_offsets[:-1])
    P = float(pl[nb.words].mean())
    byt = info["trie_nodes"] * (P * (4 * H + 20) + 4 * H + 16) + info["updates"] * 12 * H
    hbm, tc_peak, _ = peaks()
    # CPU: the oracle restatement of rescore_twopass on a bounded sample
    om = O.OracleModel(m, setup.tree)
    k = max(1, min(int(nb.n_hyp[0]), 24))
    ws = [nb.words[nb.hyp_off[j]:nb.hyp_off[j + 1]] for j in range(k)]
    t0 = time.perf_counter()
    O.twopass(om, None, ws, nb.scores[:k, 1], "rnnlm")
    cpu_s = time.perf_counter() - t0
    cpu_wps = sum(len(w) for w in ws) / cpu_s
    return {"workload": f"config b: {len(setup.lattices)} utterances x {n}-best lists "
                        f"({info['hypotheses']} hypotheses, {info['words']} words), rnnlm mode, "
                        f"{precision} update; tries resident, L2 flushed before each run",
            "device_ms": dev_ms, "words_per_s": info["words"] / (dev_ms / 1e3),
            "hyps_per_s": info["hypotheses"] / (dev_ms / 1e3),
            "trie_nodes": info["trie_nodes"], "updates": info["updates"], "levels": info["levels"],
            "prefix_sharing": info["words"] / max(info["trie_nodes"], 1),
            "algorithmic_gbs": byt / (dev_ms / 1e3) / 1e9, "frac_of_hbm": byt / (dev_ms / 1e3) / 1e9 / hbm,
            "update_tflops": 2.0 * H * H * info["updates"] / (dev_ms / 1e3) / 1e12,
            "e2e": {"words_per_s": info["words"] / e2e_s, "nbest_s": t_nbest, "trie_build_h2d_s": t_build,
                    "fetch_s": t_fetch, "host_threads": len(os.sched_getaffinity(0))},
            "cpu_baseline": {"words_per_s": cpu_wps, "cores": 1, "kind": "port",
                             "sample": f"oracle rescore_twopass on the first {k} hypotheses of utterance 0 "
                                       "(every word scored and advanced, no prefix sharing)"}}


def all_word_microbench(precision: str, n_ctx: int = 256, reps: int = 5):
    """all_word_logprobs for n contexts at config c/d size (V=65,536, H=512):
    the [n x (V-1)] node activations as one tcgen05 GEMM, then float64
    MaxEnt + log-sigmoids per node and path sums per word."""
    import torch
    from paper_2007_11794_b200 import kernels, synth
    from paper_2007_11794_b200.device import DeviceModel
    from paper_2007_11794_b200.model import build_huffman_from_counts
    cfg = synth.CONFIGS["d"]
    V, H, bits = cfg["V"], cfg["H"], cfg["bits"]
    model = synth.synth_model(V, H, bits)
    tree = build_huffman_from_counts(synth.zipf_counts(V))
    dm = DeviceModel(model, tree)
    _, hidden, hist, hlen, _ = synth.query_set(model, 16, n_ctx)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    ctx = d(np.arange(n_ctx, dtype=np.int32))
    th, thist, thl = d(hidden), d(hist), d(hlen)
    out = torch.empty((n_ctx, V), dtype=torch.float64, device="cuda")
    res = {"workload": f"{n_ctx} contexts x V={V} (H={H}, MaxEnt 2^{bits}); L2 flushed before each run"}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for prec in ("fp64", precision):
        kernels.all_word_logprobs_batch(dm, ctx, th, thist, thl, prec, out=out)
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            kernels.all_word_logprobs_batch(dm, ctx, th, thist, thl, prec, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        res[prec] = {"ms": ms, "contexts_per_s": n_ctx / (ms / 1e3),
                     "word_logprobs_per_s": n_ctx * V / (ms / 1e3),
                     "gemm_tflops_equiv": 2.0 * H * (V - 1) * n_ctx / (ms / 1e3) / 1e12}
    return res


def beam_sweep(precision: str, beams=(1, 2, 4, 8, 16, 32, 64), n_utt: int = 8, frames: int = 300,
               reps: int = 3, schedule: str = "auto"):
    """Config (c): V=65,536 H=512 MaxEnt 2^22, 8 utterances x 300 frames,
    decode throughput and RTF per beam (device time, lattices resident, L2
    flushed before each run)."""
    import torch
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    setup = synth.build_setup("c", n_utt=n_utt, T=frames, seed=17)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rows = []
    for beam in beams:
        need = BatchDecoder.contexts_needed(setup.lattices, beam)
        dec = BatchDecoder(setup.model, setup.tree, setup.small_lm, n_utt, need, precision=precision,
                           schedule=schedule)
        dec.prepare(setup.lattices, beam)
        dec.run(1.0)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            dec.run(1.0)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        hyps, out = dec.fetch()
        fr = sum(len(h.arcs) for h in hyps)
        st = dec.streams.stats()
        rows.append({"beam": beam, "ms": ms, "frames_per_s": fr / (ms / 1e3),
                     "rtf_per_stream": (ms / 1e3) / (frames * FRAME_S),
                     "requests": int(out["expansions"].sum()), "misses": int(st[:, 2].sum()),
                     "queries_per_s": int(st[:, 2].sum()) / (ms / 1e3), "schedule": dec.schedule})
        del dec
        torch.cuda.empty_cache()
    return {"workload": f"config c: V=65536 H=512 MaxEnt 2^22, {n_utt} utterances x {frames} frames, "
                        f"breadth 3, {precision} update; L2 flushed before each run", "sweep": rows}


def fat_variant(precision: str, n_utt: int = 4, frames: int = 300, reps: int = 2):
    """SURVEY.md §8d config (b) fat variant: breadth 16, beam 64 (16 nodes x
    64 tokens x 16 arcs = 16k requests per frame and utterance, ~1k arrival
    slots per node), decoded with the automatic schedule (level: the
    CTA-per-node expand and the multi-CTA assign).  Device time, lattices
    resident, L2 flushed before each run."""
    import torch
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    s = synth.build_setup("b_fat", n_utt=n_utt, T=frames, seed=3)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    need = BatchDecoder.contexts_needed(s.lattices, 64)
    dec = BatchDecoder(s.model, s.tree, s.small_lm, n_utt, need, precision=precision)
    dec.prepare(s.lattices, 64)
    dec.run(1.0)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        dec.run(1.0)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    hyps, out = dec.fetch()
    fr = sum(len(h.arcs) for h in hyps)
    st = dec.streams.stats()
    res = {"workload": f"config b fat variant: V=20000 H=256 MaxEnt 2^21, {n_utt} utterances x {frames} frames, "
                       f"breadth 16, beam 64, {precision}", "schedule": dec.schedule, "ms": ms,
           "frames_per_s": fr / (ms / 1e3), "rtf_per_stream": (ms / 1e3) / (frames * FRAME_S),
           "requests_per_s": int(out["expansions"].sum()) / (ms / 1e3),
           "contexts_created": int(st[:, 3].sum())}
    del dec
    torch.cuda.empty_cache()
    return res


def table4_sweep(precision: str, capacities_kb=(0, 16, 64, 256, 1024, -1), n_streams: int = 74,
                 n_rounds: int = 12, n_templates: int = 40, frames: int = 100, seed: int = 23):
    """The paper's Table-4 experiment (reference cli.py:195-228, :287-298):
    decode throughput and cache behaviour versus RescoreCache capacity.
    Repeated-command traffic (the acceptance crit-8 recipe, scaled up): each
    of n_streams streams decodes n_rounds utterances drawn Zipf-wise from a
    pool of n_templates config-b lattices; capacity 0 = unbounded cache reset
    per utterance, positive capacities retain the bounded LFU cache (and the
    IndexTable) across a stream's utterances; -1 = unbounded and retained.
    Device time per round (lattices resident), summed over rounds.  The
    device memoises every (c, w) value of a retained stream in HBM, so a
    bounded capacity changes the reported cache counters (replayed by the
    exact LFU policy after each decode, lfu.cuh) but not the work; the
    unbounded retained row shows the compute saved by retention itself."""
    import torch
    from paper_2007_11794_b200 import synth
    from paper_2007_11794_b200.rescore import BatchDecoder
    base = synth.build_setup("b", n_utt=n_templates, T=frames, seed=seed)
    rng = np.random.default_rng(seed)
    p = 1.0 / np.arange(1, n_templates + 1) ** 1.0
    p /= p.sum()
    picks = rng.choice(n_templates, size=(n_rounds, n_streams), p=p)
    rows = []
    for cap in capacities_kb:
        retain = cap != 0
        cap = max(cap, 0)
        need = max(BatchDecoder.contexts_needed(base.lattices, base.beam), 1) * (n_rounds if retain else 1)
        dec = BatchDecoder(base.model, base.tree, base.small_lm, n_streams, need, precision=precision,
                           capacity_bytes=cap * 1024)
        ms = 0.0
        fr = 0
        for k in range(n_rounds):
            dec.prepare([base.lattices[int(t)] for t in picks[k]], base.beam)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            dec.run(1.0, retain=retain and k > 0)
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
            hyps, _ = dec.fetch()
            fr += sum(len(h.arcs) for h in hyps)
        st = dec.streams.stats()                 # cumulative columns 4..6 after the last round
        look, hit, miss = (int(st[:, 4].sum() + st[:, 0].sum()), int(st[:, 5].sum() + st[:, 1].sum()),
                           int(st[:, 6].sum() + st[:, 2].sum()))
        cs = dec.streams.cache_stats()
        rows.append({"capacity_kb": cap, "retain": retain, "frames_per_s": fr / (ms / 1e3),
                     "rtf_per_stream": (ms / 1e3) / n_rounds / (frames * FRAME_S),
                     "lookups": look, "hits": hit, "computes": miss,
                     "hit_ratio": hit / look if look else 0.0,
                     "evictions_cumulative": int(cs[:, 1].sum()), "evictions_last_round": int(cs[:, 0].sum()),
                     "resident_entries": int(cs[:, 2].sum())})
        del dec
        torch.cuda.empty_cache()
    return {"workload": f"Table 4 (cli.py:195-228): {n_streams} streams x {n_rounds} utterances each, drawn "
                        f"Zipf(1) from {n_templates} config-b lattices x {frames} frames; {precision}; "
                        "capacity 0 = unbounded cache reset per utterance, else retained LFU cache",
            "sweep": rows}


def cpu_baseline(setup, n_sample: int, threads: int):
    """The reference algorithm on host cores: the C oracle port
    (oracle/otflm_oracle.c), fresh stream per utterance, utterance-parallel."""
    from oracle import oracle as O
    lats = setup.lattices[:n_sample]
    om = O.OracleModel(setup.model, setup.tree)
    og = O.OracleNgram(setup.small_lm)
    ols = [O.OracleLattice(l) for l in lats]
    O.decode_many(om, None, og, ols[:1], beam=setup.beam, n_threads=1)   # warm-up
    t0 = time.perf_counter()
    res = O.decode_many(om, None, og, ols, beam=setup.beam, n_threads=threads)
    dt = time.perf_counter() - t0
    frames = sum(len(r[0].arcs) for r in res)
    reqs = sum(r[1][0] for r in res)
    return frames, reqs, dt, res


def _ref_lattices(args, threads):
    """The reference arm's bounded sample of the benchmarked workload."""
    from paper_2007_11794_b200 import synth
    if args.config == "e":
        base = synth.build_setup("e", n_utt=1, T=args.frames, seed=31)
        n_sample = max(threads, 16)
        lats = synth.lattices_for_ids(base, range(n_sample), args.frames)
        base.lattices = lats
        return base, n_sample, (f"config e: V=65536 H=512 MaxEnt 2^22, utterances 0..{n_sample - 1} of the "
                                f"{args.e_total}-utterance workload x {args.frames} frames, breadth 3, beam 8")
    n_sample = min(args.n_utt, max(threads, 16))
    setup = synth.build_setup(CONFIG, n_utt=n_sample, T=args.frames, seed=7)
    return setup, n_sample, (f"config {CONFIG}: V=20000 H=256 MaxEnt 2^21, {n_sample} utt x "
                             f"{args.frames} frames sample of the 64-utt batch, breadth 3, beam 8")


def numba_reference_sample(setup, n_frames_cap: int = 300):
    """The unmodified reference (otflm, numba kernels) from baseline/_ref on
    one utterance of the workload: rescore_onthefly (decoder.py:114-173) with
    a fresh RescoreStack, built from the same synthetic arrays.  Returns None
    when baseline/_ref is absent."""
    ref_root = ROOT / "baseline" / "_ref"
    if not (ref_root / "otflm").exists():
        return None
    sys.path.insert(0, str(ref_root))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_otflm")
    try:
        from otflm import cache as rc, codec as rcod, context_table as rct, decoder as rdec
        from otflm import huffman as rh, lattice as rl, ngram as rng_, rnnlm as rr
        from paper_2007_11794_b200 import synth
    except Exception as e:                                   # pragma: no cover
        return {"unavailable": f"import failed: {e}"}
    m = setup.model
    model = rr.RnnlmModel(m.hidden_size, m.vocab_size, m.maxent_order, m.maxent_size, m.hash_seed,
                          m.input_weights, m.recurrent_weights, m.node_vectors, m.maxent_table)
    tree = rh.build_huffman_from_counts([int(c) for c in synth.zipf_counts(m.vocab_size)])
    lm = rng_.NgramModel(setup.small_lm.order, setup.small_lm.vocab_size, setup.small_lm.bos_id,
                         setup.small_lm.eos_id, setup.small_lm.probs, setup.small_lm.backoffs)
    lat = setup.lattices[0]
    arcs = [rl.Arc(i, int(lat.arc_src[i]), int(lat.arc_dst[i]), int(lat.arc_word[i]),
                   float(lat.arc_acoustic[i]), float(lat.arc_smalllm[i])) for i in range(len(lat.arc_word))]
    rlat = rl.Lattice(lat.start, set(lat.finals), arcs)

    def stack():
        return rdec.RescoreStack(model=model, tree=tree, table=rct.IndexTable(m.hidden_size, m.maxent_order),
                                 cache=rc.RescoreCache(), ledger=rcod.TransferLedger())
    # JIT warm-up (numba compiles or loads its cache) on a short prefix
    short = [a for a in arcs if rlat.times.get(a.dst, 0) <= 3]
    ends = {a.dst for a in short if rlat.times.get(a.dst, 0) == 3}
    if short and ends:
        rdec.rescore_onthefly(rl.Lattice(lat.start, ends, short), lm, stack(), beam=setup.beam)
    t0 = time.perf_counter()
    hyp, rep = rdec.rescore_onthefly(rlat, lm, stack(), beam=setup.beam)
    dt = time.perf_counter() - t0
    frames = len(hyp.arcs)
    return {"value": frames / dt, "unit": "frames/s", "cores": 1, "kind": "reference",
            "sample": f"utterance 0 ({frames} frames, {rep.expansions} requests) through the unmodified "
                      "reference otflm.decoder.rescore_onthefly (numba kernels, one thread), baseline/_ref",
            "seconds": dt, "requests_per_s": rep.expansions / dt,
            "one_best": list(hyp.arcs)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    setup, n_sample, workload = _ref_lattices(args, threads)
    times = []
    frames = reqs = 0
    res = None
    for i in range(args.warmup + args.steps):
        f, r, dt, res = cpu_baseline(setup, n_sample, threads)
        if i >= args.warmup:
            times.append(dt)
            frames, reqs = f, r
    t = float(np.mean(times))
    v = frames / t
    numba = numba_reference_sample(setup)
    if numba and "one_best" in numba:
        numba["one_best_equals_port"] = numba.pop("one_best") == list(res[0][0].arcs)
    line = {
        "impl": "reference", "metric": METRIC_E if args.config == "e" else METRIC, "value": v, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong" if args.config == "e" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "n_utt": n_sample, "frames": args.frames},
        "rtf": (t / (frames * FRAME_S)),
        "queries_per_s": reqs / t,
        "cpu_baseline": {"value": v, "unit": "frames/s", "cores": threads, "kind": "port",
                         "sample": f"{n_sample} utterances x {args.frames} frames per step through "
                                   "oracle/otflm_oracle.c (the reference decoder restated in C, bit-exact with "
                                   "the reference's golden vectors), fresh stream per utterance, "
                                   f"{threads} threads"},
        "numba_reference": numba,
        "e2e": {"value": v, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line) + "\n")


_E_BASE = None


def _e_lattices(ids):
    from paper_2007_11794_b200 import synth
    base, frames = _E_BASE
    return synth.lattices_for_ids(base, ids, frames)


def _alg_bytes(H: int, cnt: dict, misses: int, requests: int) -> float:
    """SURVEY.md §8d algorithmic bytes of one decode: HS per query
    P(4H + 4k + 8) + 4H + 16, the recurrent update 3 x 4H per computed
    context (h_c and U[w] read, h' written), ~96 B of request / arrival /
    cache state per request."""
    hs = cnt["sum_path"] * (4 * H + 8) + 4 * cnt["sum_path_k"] + cnt["hs_queries"] * (4 * H + 16)
    return float(hs + 12.0 * H * misses + 96.0 * requests)


def run_config_e(args):
    """Config (e): 4,096 utterances (V=65,536, H=512, MaxEnt 2^22, 300
    frames, breadth 3, beam 8) sharded over the ranks (parallel.shard); each
    rank decodes its shard in batches of --e-batch streams through the
    double-buffered BatchDecoder (host compile + H2D of batch i+1 overlap the
    decode of batch i), then NCCL all-gathers the per-utterance result
    records.  One step = the whole shard; strong scaling (total work fixed)."""
    import torch
    import torch.distributed as dist
    from paper_2007_11794_b200 import parallel, synth
    from paper_2007_11794_b200.device import last_launch_count
    from paper_2007_11794_b200.rescore import BatchDecoder
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_total = args.e_total
    ids = parallel.shard(n_total, world, rank)
    B = args.e_batch
    base = synth.build_setup("e", n_utt=1, T=args.frames, seed=31)
    H = base.model.hidden_size
    # lattices of this rank's shard, generated on host worker processes
    # (forked before CUDA is initialised; each lattice is a function of its id)
    t0 = time.perf_counter()
    global _E_BASE
    _E_BASE = (base, args.frames)
    import multiprocessing as mp
    n_proc = max(1, min(len(os.sched_getaffinity(0)) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1"))), 32))
    parts = [ids[i:i + 16] for i in range(0, len(ids), 16)]
    with mp.get_context("fork").Pool(n_proc) as pool:
        lat_parts = pool.map(_e_lattices, parts)
    lat_all = [l for part in lat_parts for l in part]
    batches = [(ids[b0:b0 + B], lat_all[b0:b0 + B]) for b0 in range(0, len(ids), B)]
    t_gen = time.perf_counter() - t0
    torch.cuda.set_device(local)
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    # a short last batch: with at most half an SM per stream short of a full
    # wave it gets its own decoder (the automatic schedule then gives each of
    # its streams a 2-CTA cluster, ~1.5x faster per stream than one CTA);
    # otherwise it is padded with repeats of its own utterances (decoded, not
    # counted) so every batch has the same compiled structure and the plans
    # are refreshed in place instead of rebuilt
    sel, lats = batches[-1]
    tail_dec = None
    if len(lats) < B and len(batches) > 1:
        if args.schedule == "auto" and 2 * len(lats) <= n_sm:
            tail_dec = BatchDecoder(base.model, base.tree, base.small_lm, len(lats),
                                    BatchDecoder.contexts_needed(lats, base.beam), precision=args.precision)
        else:
            pad = [lats[i % len(lats)] for i in range(B - len(lats))]
            batches[-1] = (sel, lats + pad)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    need = max(BatchDecoder.contexts_needed(l, base.beam) for _, l in (batches[:-1] if tail_dec else batches))
    dec = BatchDecoder(base.model, base.tree, base.small_lm, B, need, precision=args.precision,
                       schedule=args.schedule, n_buffers=2, n_groups=args.groups)
    stream = torch.cuda.current_stream()
    launches = [0]

    def one_pass(record: bool):
        """decode the shard: device time (sum of the batch decodes) and e2e."""
        recs = []
        frames = requests = misses = 0
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s_prev, prev_sel = None, None
        evs = []
        h2d = d2h = 0

        def take(d_, slot, sel_):
            nonlocal frames, requests, misses, d2h
            hyps, out = d_.fetch(slot=slot)
            n = len(sel_)
            frames += int(sum(len(h.arcs) for h in hyps[:n]))
            requests += int(out["expansions"][:n].sum())
            d2h += int(sum(v.nbytes for v in out.values()))
            if record:
                o = {k: v[:n] for k, v in out.items()}
                arcs = np.full((n, args.frames), -1)       # per-utterance arc ids (out holds batch-global ids)
                for i, h in enumerate(hyps[:n]):
                    arcs[i, :min(len(h.arcs), args.frames)] = h.arcs[:args.frames]
                o["path_arcs"] = arcs
                recs.append(parallel.pack_records(sel_, o, args.frames))
        d_prev = None
        for bi, (sel_, lats_) in enumerate(batches):
            d_cur = tail_dec if (tail_dec is not None and bi == len(batches) - 1) else dec
            s_cur = d_cur.prepare(lats_, base.beam)       # host compile + pinned H2D (overlaps the previous decode)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            d_cur.run(1.0, slot=s_cur)
            e1.record(stream)
            launches[0] += last_launch_count()
            evs.append((e0, e1))
            if s_prev is not None:
                take(d_prev, s_prev, prev_sel)
            s_prev, prev_sel, d_prev = s_cur, sel_, d_cur
        take(d_prev, s_prev, prev_sel)
        b.record(stream)
        torch.cuda.synchronize()
        dev_ms = sum(x.elapsed_time(y) for x, y in evs)
        return dev_ms, a.elapsed_time(b), frames, requests, d2h, recs

    for _ in range(args.warmup):
        one_pass(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    dev, e2e = [], []
    with Clocks(local) as clk:
        for i in range(args.steps):
            d_ms, e_ms, fr, rq, d2h, recs = one_pass(i == args.steps - 1)
            dev.append(d_ms)
            e2e.append(e_ms)
    dev_ms, e2e_ms = float(np.mean(dev)), float(np.mean(e2e))
    if world > 1:
        t = torch.tensor([dev_ms, e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, e2e_ms = (float(x) for x in t.cpu())
        allr = parallel.gather_records(np.concatenate(recs), n_total, device="cuda")
    else:
        allr = np.concatenate(recs)
    total_frames = int(allr[:, 1].sum())
    total_requests = int(allr[:, 6].sum())
    # ---- roofline of the persistent decode kernel: one profiled batch
    # (event-record nodes around every kernel) gives the algorithmic-work
    # counters and the kernel's share of a decode run ----
    s_last = dec.prepare(batches[0][1], base.beam)
    prof = dec.profile(1.0)
    cnt = dec.counters()
    phases = dec.plan.phase_ns()
    hyps0, out0 = dec.fetch(slot=s_last)
    st0 = dec.streams.stats()
    req0, miss0 = int(out0["expansions"].sum()), int(st0[:, 2].sum())
    byt0 = _alg_bytes(H, cnt, miss0, req0)
    run_ms = sum(v[0] for v in prof.values())
    share = prof["stream"][0] / run_ms if "stream" in prof and run_ms > 0 else 1.0
    n_batches = len(batches)
    kern_ms = dev_ms / n_batches * share                  # avg persistent-kernel launch, timed region
    byt = byt0 * (total_requests / world / n_batches) / max(req0, 1)   # per launch, scaled to the timed batches
    hbm, tc_peak, peak_src = peaks()
    kname = "k_decode_solo" if dec.schedule == "stream1" else "k_decode_streams"
    roof = {"kernel": kname + " (persistent: expand + tcgen05 digit-plane update + digit-plane HS + assign)",
            "bound": "hbm", "achieved": byt / (kern_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "traffic": None, "peak_source": peak_src, "avg_launch_us": kern_ms * 1e3,
            "algorithmic_bytes_per_launch": byt, "launches_per_step": n_batches,
            "kernel_share_of_decode_run": share,
            "tensor_int8_tops": 17 * 2.0 * H * H * miss0 / (prof.get("stream", (run_ms, 1))[0] / 1e3) / 1e12}
    roof["frac"] = roof["achieved"] / roof["peak"]
    tfile = ROOT / "profiles" / "traffic.json"
    key = f"{kname}_e_{args.precision}"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text()).get(key)
            if tj:
                roof["traffic"] = tj["dram_bytes_per_launch"] * (byt / tj["algorithmic_bytes_per_launch"])
                roof["traffic_source"] = tj["source"]
        except (KeyError, ValueError, ZeroDivisionError):
            pass
    nl = max(1, args.frames)
    ph = {k: round(v / max(phases["ctas"], 1) / nl / 1e3, 3) for k, v in phases.items() if k != "ctas"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from types import SimpleNamespace
        threads = len(os.sched_getaffinity(0))
        n_sample = max(threads, 16)
        sample = SimpleNamespace(model=base.model, tree=base.tree, small_lm=base.small_lm,
                                 beam=base.beam, lattices=batches[0][1][:n_sample])
        f, r, dt, ref = cpu_baseline(sample, n_sample, threads)
        agree = sum(1 for u in range(n_sample) if tuple(hyps0[u].arcs) == tuple(ref[u][0].arcs))
        cpu = {"value": f / dt, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"the first {n_sample} utterances of the shard x {args.frames} frames "
                         "(oracle/otflm_oracle.c, all host threads)",
               "one_best_agreement": f"{agree}/{n_sample}"}
    extras = {}
    if rank == 0 and not args.no_queries:
        extras["config_d_queries"] = query_microbench("exact" if args.precision == "exact" else args.precision)
    if rank == 0 and not args.no_wide:
        # big beams / wide lattices (the level schedule's CTA-per-node expand and multi-CTA assign)
        extras["config_c_beam_sweep"] = beam_sweep(args.precision, beams=(8, 16, 32, 64), reps=2)
        extras["fat_variant"] = fat_variant(args.precision)
    if rank == 0 and args.table4:
        extras["table4_capacity_sweep"] = table4_sweep(args.precision)
    if rank == 0:
        line = {
            "metric": METRIC_E,
            "value": total_frames / (dev_ms / 1e3), "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8 digit planes / s32 accumulation / f64 scores (exact)" if args.precision == "exact"
                     else "f64 scores / f32 weights / " + args.precision + " recurrent update",
            "data": "synthetic (seeded per utterance id; RnnlmModel.new recipe + Zipf Huffman + synthetic bigram)",
            "config": {"workload": f"config e: V=65536 H=512 MaxEnt 2^22, {n_total} utterances x {args.frames} "
                                   f"frames sharded over {world} GPU(s), batches of {B} streams, breadth 3, beam 8",
                       "n_utt_total": n_total, "batch_streams": B, "precision": args.precision,
                       "schedule": dec.schedule, "lattice_generation_s": round(t_gen, 2),
                       "tail_batch": (f"{len(batches[-1][0])} streams, own decoder, schedule {tail_dec.schedule}"
                                      if tail_dec is not None else "padded to the batch size"),
                       "l2": "inputs (4096 lattices, arenas, 280 MB of weights) far larger than L2; not flushed"},
            "rtf": (dev_ms / 1e3) / (total_frames * FRAME_S),
            "rtf_per_stream": (dev_ms / 1e3) / n_batches / (args.frames * FRAME_S),
            "requests_per_s": total_requests / (dev_ms / 1e3),
            "utterances_gathered": int(len(allr)),
            "roofline": roof,
            "stream_phase_us_per_level": ph,
            "exact_uncertified_elements_per_batch": cnt.get("exact_fallbacks"),
            "e2e": {"value": total_frames / (e2e_ms / 1e3), "unit": "frames/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(cnt["h2d_bytes"] * n_batches),
                    "d2h_bytes_per_step": int(d2h),
                    "pipeline": "double-buffered batches through the public BatchDecoder API: host compile + "
                                "pinned H2D of batch i+1 overlap the decode of batch i; 1-best D2H per batch"},
            "gpu_launches": int(launches[0]),
            "clocks": clk.summary(),
            "extras": extras,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
        if args.out:
            Path(args.out).write_text(json.dumps(line) + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _self_launch(args) -> bool:
    """--gpus N outside torchrun: re-run this command under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous)."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return False
    if args.gpus <= 1:
        return False
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    args = parse()
    _self_launch(args)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.config == "e":
        run_config_e(args)
        return
    run_config_b(args)


def run_config_b(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2007_11794_b200 import _lib, synth
    from paper_2007_11794_b200.device import last_launch_count
    from paper_2007_11794_b200.rescore import BatchDecoder

    setup = synth.build_setup(CONFIG, n_utt=args.n_utt, T=args.frames, seed=7 + 1000 * rank)
    H = setup.model.hidden_size
    need = BatchDecoder.contexts_needed(setup.lattices, setup.beam)
    dec = BatchDecoder(setup.model, setup.tree, setup.small_lm, len(setup.lattices), need,
                       precision=args.precision, n_groups=args.groups, schedule=args.schedule,
                       n_buffers=2)
    dec.prepare(setup.lattices, setup.beam)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MB > L2
    use_graph = not args.no_graph

    for _ in range(args.warmup):
        dec.run(1.0, use_graph=use_graph)
    torch.cuda.synchronize()
    launches_per_step = last_launch_count() + 1          # graph kernels + stream reset kernel

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()                                  # L2 flush between iterations
            ev[i][0].record(stream)
            dec.run(1.0, use_graph=use_graph)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    hyps, out = dec.fetch()
    frames_per_step = int(sum(len(h.arcs) for h in hyps))
    requests = int(out["expansions"].sum())
    stats = dec.streams.stats()
    misses = int(stats[:, 2].sum())
    ms = total_ms / args.steps
    value = frames_per_step * world / (ms / 1e3)

    # ---- per-kernel CUDA-event timing: one run replayed from a graph with
    # event-record nodes around every kernel (device-side spans) ----
    prof = dec.profile(1.0)
    cnt = dec.counters()
    hbm, tc_peak, peak_src = peaks()
    # algorithmic bytes: HS per query P(4H + 4k + 8) + 4H + 16;
    # recurrent update per miss 3 x 4H (h_c read, U row read, h' write) and
    # 2H^2 flops; W (H^2 x 4 B x passes) is re-read per 128-row tile.
    hs_bytes = cnt["sum_path"] * (4 * H + 8) + 4 * cnt["sum_path_k"] + cnt["hs_queries"] * (4 * H + 16)
    adv_flops = 2.0 * H * H * misses
    kinds = {k: v for k, v in prof.items() if v[1] > 0}
    dominant = max(kinds, key=lambda k: kinds[k][0])
    dom_ms, dom_n = kinds[dominant]
    if dominant == "stream":
        # persistent kernel: all algorithmic bytes of the path (HS rows +
        # update rows 3 x 4H per miss + ~96 B of request / arrival state)
        byt = hs_bytes + 12.0 * H * misses + 96.0 * requests
        roof = {"kernel": "k_decode_streams (persistent: expand + tcgen05 update + HS + assign)",
                "bound": "hbm", "achieved": byt / (dom_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                "tensor_tflops": adv_flops * (3 if args.precision == "tf32x3" else 1) / (dom_ms / 1e3) / 1e12}
    elif dominant == "hs":
        roof = {"kernel": "k_hs_prim (HS + MaxEnt gather)", "bound": "hbm",
                "achieved": hs_bytes / (dom_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s"}
    elif dominant == "advance":
        roof = {"kernel": f"recurrent update ({args.precision})", "bound": "tensor",
                "achieved": adv_flops / (dom_ms / 1e3) / 1e12, "peak": tc_peak, "unit": "TFLOP/s"}
    else:
        # control kernels: bytes ~ requests x ~96 B of request/arrival state
        roof = {"kernel": f"k_{dominant}", "bound": "hbm",
                "achieved": requests * 96 / (dom_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    # DRAM bytes per launch of the dominant kernel from the committed ncu
    # capture of this same command (profiles/traffic.json), else null
    roof["traffic"] = None
    tfile = Path(__file__).resolve().parent / "profiles" / "traffic.json"
    if dominant == "stream" and tfile.exists():
        try:
            t = json.loads(tfile.read_text())["k_decode_streams"]
            roof["traffic"] = t["dram_bytes_per_launch"]
            roof["traffic_source"] = t["source"]
            roof["algorithmic_bytes"] = roof["achieved"] * 1e9 * (dom_ms / 1e3)
        except (KeyError, ValueError):
            pass
    roof["peak_source"] = peak_src
    roof["launches"] = dom_n
    roof["avg_launch_us"] = dom_ms * 1e3 / max(dom_n, 1)
    kernel_ms = {k: round(v[0], 4) for k, v in prof.items() if v[1]}
    phases = None
    if dec.schedule != "level":
        ph = dec.plan.phase_ns()
        n_lv = max(1, args.frames)
        phases = {k: round(ph[k] / max(ph["ctas"], 1) / n_lv / 1e3, 3)
                  for k in ph if k != "ctas"}

    # ---- end to end through the public API: host lattices in, 1-best out;
    # two different batches alternate (same compiled structure -> the plans
    # are refreshed in place and the captured graph is replayed) ----
    batches = [setup.lattices, synth.more_lattices(setup, args.n_utt, args.frames, seed=99 + 1000 * rank)]
    # double-buffered through the public API: each step compiles + uploads
    # (pinned H2D) batch i+1 on the host while the GPU decodes batch i, then
    # reads batch i's 1-best back (D2H).  The pipeline is filled untimed.
    n_e2e = max(3, args.steps)
    s_prev = dec.prepare(batches[0], setup.beam)
    dec.run(1.0, use_graph=True, slot=s_prev)
    for i in range(1, 3):                                 # both buffers built and warm
        s_cur = dec.prepare(batches[i % 2], setup.beam)
        dec.run(1.0, use_graph=True, slot=s_cur)
        dec.fetch(slot=s_prev)
        s_prev = s_cur
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t_host = time.perf_counter()
    a.record(stream)
    for i in range(1, n_e2e + 1):
        s_cur = dec.prepare(batches[i % 2], setup.beam)   # host compile + H2D, overlaps the decode of s_prev
        dec.run(1.0, use_graph=True, slot=s_cur)          # queued behind s_prev on the GPU
        h2, o2 = dec.fetch(slot=s_prev)                   # D2H of s_prev's 1-best (copy stream) while s_cur decodes
        if world > 1:
            rec = torch.from_numpy(np.concatenate([o2["combined"], o2["path_len"].astype(np.float64)])).cuda()
            gathered = [torch.empty_like(rec) for _ in range(world)]
            dist.all_gather(gathered, rec)                # NCCL: results only
        s_prev = s_cur
    h2, o2 = dec.fetch(slot=s_prev)
    b.record(stream)
    torch.cuda.synchronize()
    e2e = a.elapsed_time(b) / n_e2e
    e2e_host = (time.perf_counter() - t_host) * 1e3 / n_e2e
    if world > 1:
        t = torch.tensor([e2e], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    d2h = int(sum(v.nbytes for v in o2.values()))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        n_sample = min(args.n_utt, max(threads, 16))
        f, r, dt, ref = cpu_baseline(setup, n_sample, threads)
        agree = sum(1 for u in range(n_sample) if hyps[u].arcs == ref[u][0].arcs)
        cpu = {"value": f / dt, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"{n_sample} of the {args.n_utt} utterances x {args.frames} frames "
                         "(oracle/otflm_oracle.c, all host threads)",
               "one_best_agreement": f"{agree}/{n_sample}"}

    clocks = clk.summary()
    extras = {}
    if rank == 0 and not args.no_queries:
        extras["config_d_queries"] = query_microbench(args.precision)
    if rank == 0 and args.all_word:
        extras["all_word_logprobs"] = all_word_microbench(args.precision)
    if rank == 0 and args.beam_sweep:
        extras["config_c_beam_sweep"] = beam_sweep(args.precision)
    if rank == 0 and args.table4:
        extras["table4_capacity_sweep"] = table4_sweep(args.precision)
    if rank == 0 and args.twopass_n > 0:
        extras["twopass"] = twopass_microbench(setup, args.precision, args.twopass_n)
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 scores / f32 weights / " + args.precision + " recurrent update",
        "data": "synthetic (seeded: RnnlmModel.new recipe + Zipf Huffman + synthetic bigram)",
        "config": {"workload": f"config {CONFIG}: V=20000 H=256 MaxEnt 2^21 HS+MaxEnt RNNLM, "
                               f"{args.n_utt} utterances x {args.frames} frames per GPU, breadth 3, "
                               "beam 8, per-utterance streams (retain=False)",
                   "n_utt_per_gpu": args.n_utt, "frames": args.frames, "beam": setup.beam,
                   "precision": args.precision, "schedule": dec.schedule,
                   "cuda_graph": use_graph and dec.schedule == "level",
                   "concurrent_groups": dec.n_groups,
                   "l2": "flushed (256 MB write) between timed iterations"},
        "rtf": (ms / 1e3) / (frames_per_step * FRAME_S) * (1 if world == 1 else 1),
        "rtf_per_stream": (ms / 1e3) / (args.frames * FRAME_S),
        "queries_per_s": misses * world / (ms / 1e3),
        "requests_per_s": requests * world / (ms / 1e3),
        "kernel_ms_per_step": kernel_ms,
        "exact_uncertified_elements_per_step": cnt.get("exact_fallbacks"),
        "stream_phase_us_per_level": phases,
        "roofline": roof,
        "e2e": {"value": frames_per_step * world / (e2e / 1e3), "unit": "frames/s",
                "h2d_bytes_per_step": cnt["h2d_bytes"], "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e, "host_wall_ms_per_step": e2e_host,
                "pipeline": "double-buffered plans: host compile + pinned H2D of batch i+1 overlap the decode of batch i"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "extras": extras,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.out:
            Path(args.out).write_text(json.dumps(line) + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
