"""Markdown table of bench.py lines: python tools/bench_table.py DIR [PREFIX] [configs...]
(reads DIR/<PREFIX><config>.json, PREFIX default "bench_", the last JSON line of each)."""
import json
import os
import sys


def line(path):
    with open(path) as f:
        rows = [r for r in f.read().strip().splitlines() if r.startswith("{")]
    return json.loads(rows[-1]) if rows else None


def main():
    d = sys.argv[1]
    rest = sys.argv[2:]
    prefix = "bench_"
    if rest and not rest[0].startswith("c"):
        prefix, rest = rest[0], rest[1:]
    cfgs = rest or ["c2", "c1", "c3", "c4", "c5", "c2f", "c3f"]
    print("| config | samples/s | e2e samples/s (host output) | ESS/s | lock-step speed-up (R(m)) | "
          "roofline frac (8(d)) | issue frac | CPU port | clocks |")
    print("|---|---:|---:|---:|---:|---:|---:|---:|---|")
    for c in cfgs:
        p = os.path.join(d, f"{prefix}{c}.json")
        if not os.path.exists(p):
            continue
        b = line(p)
        if b is None:
            continue
        lock = b.get("lockstep") or {}
        lk = "-"
        if lock:
            lk = f"{lock['speedup']:.2f}x"
            if lock.get("R_of_m"):
                lk += f" ({lock['R_of_m']:.2f})"
        roof = b["roofline"]
        issue = roof.get("issue", {}).get("frac")
        cpu = b.get("cpu_baseline") or {}
        clk = b.get("clocks", {})
        ess = b.get("ess_per_sec")
        print(f"| {c} | {b['value']:.3e} | {b['e2e']['value']:.3e} | "
              f"{'-' if ess is None else f'{ess:.3e}'} | {lk} | {roof['frac']:.3f} ({roof['bound']}) | "
              f"{'-' if issue is None else f'{issue:.2f}'} | "
              f"{'-' if not cpu else f'{cpu['value']:.3e} ({cpu['cores']} thr)'} | "
              f"{clk.get('sm_mhz')} MHz {','.join(clk.get('reasons', [])) or 'no throttle'} |")


if __name__ == "__main__":
    main()
