"""Summarise ptxas -v logs (build/*.ptxas.log): kernel, registers, spills."""
import glob
import re
import sys

for path in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "build/*.ptxas.log")):
    cur = None
    rows = []
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            k = re.search(r"(fsm_init_kernel|fsm_run_kernel|lockstep_kernel|target_eval_kernel|"
                          r"prng_fill_kernel|diag_\w+_kernel)", name)
            fam = re.search(r"4(Drmh|Nuts)|3(Ess)", name)
            ge = re.findall(r"Li(\d+)E", name)
            cur = [k.group(1) if k else name[:40],
                   (fam.group(1) or fam.group(2) or fam.group(3)) if fam else "", "x".join(ge)]
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur is not None:
            cur += [m.group(1), m.group(2)]
        m = re.search(r"Used (\d+) registers", line)
        if m and cur is not None:
            rows.append(cur + [m.group(1)])
            cur = None
    for r in rows:
        print(f"{path.split('/')[-1][:14]:14s} {r[0]:18s} {r[1]:5s} {r[2]:6s} regs={r[-1]:4s} spill_st={r[3] if len(r) > 4 else '?'}")
