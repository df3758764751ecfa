"""Per-source-line hot spots of one kernel in an ncu report (instructions executed and warp
stall samples).  usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res = []
fname = None
hdr = None
seen = set()
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < 8:
        continue
    key = (fname, r[0])
    if key in seen:       # one report per launch: keep the first kernel instance
        continue
    seen.add(key)
    try:
        samp = int(r[4]); inst = int(r[7])
    except ValueError:
        continue
    res.append((samp, inst, fname, r[0], r[1].strip()[:90]))
tot_s = sum(x[0] for x in res) or 1
tot_i = sum(x[1] for x in res) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln}  {src}")
