"""DRAM traffic of the dominant kernel of a bench case from an `ncu --set full` report.

usage: ncu_traffic.py <report.ncu-rep | raw-page.csv> <config:case> [kernel-regex]
Reads `ncu -i <report> --page raw --csv` (or that page already exported to a file), takes the launches whose name matches the regex
(default: translate), averages dram__bytes_read.sum + dram__bytes_write.sum over them and
records the result in profiles/ncu_traffic_r02.json, which bench.py quotes as
`roofline.traffic` (never a literal in the source)."""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep, key = sys.argv[1], sys.argv[2]
pattern = re.compile(sys.argv[3] if len(sys.argv) > 3 else "translate")
if rep.endswith(".csv"):
    raw = Path(rep).read_text()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], stdout=subprocess.PIPE, text=True,
                         check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(v.replace(",", "")) * scale


sel = [r for r in data if pattern.search(r[ix["Kernel Name"]])]
if not sel:
    raise SystemExit("no launch matches")
tot = []
for r in sel:
    rd = to_bytes(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
    wr = to_bytes(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
    tot.append((rd, wr))
rd = sum(t[0] for t in tot) / len(tot)
wr = sum(t[1] for t in tot) / len(tot)
path = ROOT / "profiles" / "ncu_traffic_r02.json"
rec = json.loads(path.read_text()) if path.exists() else {}
name = sel[0][ix["Kernel Name"]]
rec[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "launches": len(sel),
            "kernel": name.split("(")[0][-60:], "source": Path(rep).name,
            "duration_us": float(sel[0][ix["gpu__time_duration.sum"]].replace(",", "")) if "gpu__time_duration.sum" in ix else None}
path.write_text(json.dumps(rec, indent=1, sort_keys=True) + "\n")
print(key, rec[key])
