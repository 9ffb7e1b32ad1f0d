"""Standalone config-(d) query microbench (for ncu captures)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

if __name__ == "__main__":
    prec = sys.argv[1] if len(sys.argv) > 1 else "tf32x3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    print(json.dumps(bench.query_microbench(prec, reps=reps)))
