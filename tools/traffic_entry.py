"""profiles/traffic.json entry from one `ncu --set full` capture of the decode
kernel and the tools/decode_once.py counters of the same decode:
    python tools/traffic_entry.py REP.ncu-rep DECODE_ONCE.json KEY "source text"
(algorithmic bytes by bench._alg_bytes; DRAM bytes = dram__bytes_read.sum +
dram__bytes_write.sum of the captured launch)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import _alg_bytes  # noqa: E402

rep, once, key, src = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
col = {name: i for i, name in enumerate(h)}


def val(name):
    x = float(v[col[name]].replace(",", ""))
    unit = u[col[name]]
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "us": 1e-3, "ns": 1e-6}.get(unit, 1)


dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
ms = val("gpu__time_duration.sum")
d = json.loads(Path(once).read_text().strip().splitlines()[-1])
alg = _alg_bytes(d["H"], d["counters"], d["misses"], d["requests"])
tf = Path("profiles/traffic.json")
t = json.loads(tf.read_text())
t[key] = {"dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": alg, "kernel_ms_ncu": ms, "source": src}
tf.write_text(json.dumps(t, indent=1) + "\n")
print(key, t[key], "dram/alg", dram / alg)
