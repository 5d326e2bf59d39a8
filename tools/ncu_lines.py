"""Per-source-line instruction / thread / stall totals from an ncu report
(`--page source --print-source cuda,sass`).  usage: ncu_lines.py rep [topN]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr = None, None
inst, thr, stall, src = collections.Counter(), collections.Counter(), collections.Counter(), {}
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = {}
        for i, h in enumerate(r):
            hdr.setdefault(h, i)
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    key = (fname, line)
    src[key] = r[1].strip()[:70]
    ie = r[hdr["Instructions Executed"]]
    if ie and ie != "-":
        try:
            int(ie), int(r[hdr["Thread Instructions Executed"]] or 0)
            int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except ValueError:
            continue   # a source line whose text broke the CSV quoting
        inst[key] += int(ie)
        tv = r[hdr["Thread Instructions Executed"]]
        thr[key] += int(tv) if tv not in ("", "-") else 0
        sv = r[hdr["Warp Stall Sampling (All Samples)"]]
        stall[key] += int(sv) if sv not in ("", "-") else 0
T = sum(inst.values())
S = max(1, sum(stall.values()))
print(f"total warp instructions {T:.3e}")
for key, v in inst.most_common(top):
    print(f"{key[0][:14]:14s}:{key[1]:<4d} {100 * v / T:5.1f}% thr={thr[key] / v:5.1f} stall={100 * stall[key] / S:5.1f}%  {src.get(key, '')}")
