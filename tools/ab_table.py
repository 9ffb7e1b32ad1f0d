"""Print a compact A/B table of variant bench + config-c phase files."""
import json, sys, glob
tag = sys.argv[1]
keys = ["expand", "update_kloop", "update_epilogue", "mma_wait_operands", "hs_setup", "hs_pairs", "hs_group_total", "assign", "control_waits_for_update"]
for f in sorted(glob.glob(f"gpurun_out/{tag}_*_bench.jsonl")):
    v = f[len(f"gpurun_out/{tag}_"):-len("_bench.jsonl")]
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ph = d["stream_phase_us_per_level"]
        print(f"{v:10s} b: {d['value']/1e3:8.1f}k e2e {d['e2e']['value']/1e3:8.1f}k ", " ".join(f"{k[:10]}={ph[k]:.1f}" for k in keys))
    except Exception as e:
        print(v, "bench?", e)
    try:
        c = json.loads(open(f"gpurun_out/{tag}_{v}_phc.json").read().strip().splitlines()[-1])
        ph = c["us_per_level"]
        print(f"{v:10s} c: {c['frames_per_s']/1e3:8.1f}k              ", " ".join(f"{k[:10]}={ph[k]:.1f}" for k in keys))
    except Exception as e:
        print(v, "phc?", e)
