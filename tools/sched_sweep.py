"""Config-c beam sweep (8 utterances x 300 frames, EXACT) per schedule, to
place the automatic schedule choice (GPU):  python tools/sched_sweep.py"""
import json
import sys
sys.path.insert(0, ".")
import bench

for sched in ("level", "stream1", "stream"):
    rows = bench.beam_sweep("exact", beams=(8, 16, 32, 64), reps=2, schedule=sched)["sweep"]
    for r in rows:
        print(json.dumps({"schedule": sched, "beam": r["beam"], "ms": round(r["ms"], 2),
                          "frames_per_s": round(r["frames_per_s"]), "rtf_per_stream": r["rtf_per_stream"]}),
              flush=True)
