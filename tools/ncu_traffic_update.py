"""Rewrite profiles/ncu_traffic.json's C2 fp32 entries from a committed ncu --set full raw page
of one C2 forward (13 launches in forward order): DRAM read + write bytes per launch.
usage: python tools/ncu_traffic_update.py profiles/r2_ncu_fwd_v2_raw.csv"""
import csv
import json
import sys
from pathlib import Path

NAMES = ["stem", "enc0.s1", "enc0.s2", "enc0.gate", "enc1.s1", "enc1.s2", "enc1.gate",
         "dec0.s1", "dec0.s2", "dec0.gate", "dec1.s1", "dec1.s2", "head"]
raw = sys.argv[1]
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def mbytes(r, k):
    v = float(r[col[k]])
    u = units[col[k]]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


assert len(data) == len(NAMES), (len(data), "launches in the capture")
p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
entries = [e for e in json.loads(p.read_text())
           if not (e["batch"] == 64 and e["map"] == [128, 128] and e["precision"] == "fp32")]
for name, r in zip(NAMES, data):
    entries.append({"launch": name, "batch": 64, "map": [128, 128], "precision": "fp32",
                    "dram_bytes": int(mbytes(r, "dram__bytes_read.sum") + mbytes(r, "dram__bytes_write.sum")),
                    "source": f"{raw}: {r[col['Kernel Name']][:70]}"})
p.write_text(json.dumps(entries, indent=1) + "\n")
print(f"{len(NAMES)} entries from {raw}; forward sum "
      f"{sum(e['dram_bytes'] for e in entries if e['batch'] == 64 and e['map'] == [128, 128] and e['precision'] == 'fp32') / 1e6:.0f} MB")
