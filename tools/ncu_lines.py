"""Map ncu per-instruction stall samples / instruction counts onto CUDA source lines.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [paper_1604_01074_b200/libtsmpc.so] [--top 40]

ncu's source page only carries metrics at SASS level for this build, so this
script disassembles the profiled library with line info (nvdisasm -g) and
attributes every SASS row (matched by function-relative address) to file:line.
"""

import argparse
import csv
import io
import pathlib
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("lib", nargs="?", default="paper_1604_01074_b200/libtsmpc.so")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--cubin", default="tsmpc_apg.sm_100a.cubin")
ap.add_argument("--by-instr", action="store_true", help="rank lines by instructions executed")
a = ap.parse_args()

src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ii = hdr.index("Instructions Executed")
si = hdr.index("Source")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[0], 16), r))
    except (ValueError, IndexError):
        pass

with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(pathlib.Path(a.lib).resolve())], cwd=td,
                   capture_output=True)
    sass = subprocess.run(["nvdisasm", "-g", "-c", str(pathlib.Path(td) / a.cubin)],
                          capture_output=True, text=True).stdout
# instruction sequence with line info, in program order (the kernel and the
# device functions it calls are laid out contiguously in the .text section)
seq = []
cur = None
for ln in sass.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", ln)
    if m:
        seq.append((int(m.group(1), 16), m.group(2).strip(), cur))
# ncu rows are the same instruction stream; align by position (first kernel in file)
base = min(d[0] for d in data)
by_off = {}
for off, ins, loc in seq:
    by_off.setdefault(off, (ins, loc))
agg = defaultdict(lambda: defaultdict(float))
miss = 0
for addr, r in data:
    hit = by_off.get(addr - base)
    loc = hit[1] if hit else ("?", 0)
    if hit is None:
        miss += 1
    agg[loc]["instr"] += float(r[ii] or 0)
    for c in stall_cols:
        agg[loc][hdr[c]] += float(r[c] or 0)
tot_s = sum(sum(v for k, v in d.items() if k != "instr") for d in agg.values()) or 1.0
tot_i = sum(d["instr"] for d in agg.values()) or 1.0
files = {}
print(f"unmatched rows: {miss}/{len(data)}   total stall samples {tot_s:.0f}")
items = sorted(agg.items(), key=(lambda kv: -kv[1]["instr"]) if a.by_instr else
               (lambda kv: -sum(v for k, v in kv[1].items() if k != "instr")))
for loc, d in items[: a.top]:
    s = sum(v for k, v in d.items() if k != "instr")
    top = sorted(((k.replace("stall_", ""), v) for k, v in d.items() if k != "instr" and v > 0),
                 key=lambda x: -x[1])[:3]
    text = ""
    if loc[0] != "?":
        p = next(pathlib.Path("paper_1604_01074_b200/csrc").glob(loc[0]), None)
        if p:
            files.setdefault(loc[0], p.read_text().splitlines())
            text = files[loc[0]][loc[1] - 1].strip()[:70]
    print(f"{100 * s / tot_s:5.1f}% smp {100 * d['instr'] / tot_i:5.1f}% ins {loc[0]}:{loc[1]:<4} "
          f"{','.join(f'{k}:{int(v)}' for k, v in top):38s} {text}")

# optional: per-region instruction totals (--region a-b, inclusive line numbers)
