"""DRAM traffic of the decode kernel from an ncu --set full capture, for bench.py's
roofline.traffic (profiles/r02_decode_traffic.json).

    python tools/decode_traffic.py gpurun_out/<tag>/decode_full.ncu-rep <tag>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, tag = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units, data = rows[0], rows[1], rows[2]


def val(name):
    i = head.index(name)
    v = float(data[i].replace(",", ""))
    u = units[i].strip().lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
    return int(round(v * scale))


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
kernel = data[head.index("Kernel Name")]
out = {"kernel": kernel.split("(")[0].replace("void ", "").replace("<unnamed>::", ""),
       "source": f"profiles/{tag}_ncu.md (ncu --set full --clock-control none, run {tag}, this commit's build)",
       "dram_bytes_read": rd, "dram_bytes_write": wr, "bytes_per_launch": rd + wr,
       "algorithmic_bytes_per_launch": 302056032}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02_decode_traffic.json")
with open(path, "w") as f:
    json.dump(out, f)
print(json.dumps(out))
