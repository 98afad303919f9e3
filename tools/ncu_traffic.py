"""Summarise an ncu --set full capture of the persistent solve kernel into
profiles/ncu_traffic.json: DRAM bytes (read + write) per launch, with the
iteration count of the profiled launch, keyed by kernel and tree.

    python tools/ncu_traffic.py gpurun_out/x.ncu-rep --tree SMPC3 --iters 50
"""
import argparse
import csv
import io
import json
import pathlib
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--tree", required=True)
ap.add_argument("--iters", type=int, required=True)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out_p = pathlib.Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
d = json.loads(out_p.read_text()) if out_p.exists() else {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    kern = name.split("(")[0].strip()
    if kern.startswith("void "):
        kern = kern[5:]
    kern = kern.split("<")[0]  # template arguments (apg_wide_kernel<2>)
    kern = kern if kern.startswith("tsmpc::") else "tsmpc::" + kern
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    t = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
    tu = units[hdr.index("gpu__time_duration.sum")]
    d.setdefault(kern, {})[a.tree] = {"dram_bytes": tot, "iters": a.iters,
                                      "time": f"{t} {tu}", "source": pathlib.Path(a.rep).name}
    print(kern, a.tree, f"{tot / 1e6:.2f} MB per launch of {a.iters} iterations", t, tu)
out_p.write_text(json.dumps(d, indent=1) + "\n")
