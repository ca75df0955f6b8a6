"""Summarise an ncu SASS source CSV (tools/perf/ncu_src.sh): the hot loop's instructions with
their stall samples, and totals by phase marker.  Usage: python tools/perf/src_hot.py X_src.csv [min]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 300
h = next(r for r in rows if "Address" in r)
ix = {k: i for i, k in enumerate(h)}
data = rows[rows.index(h) + 1:]


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (ValueError, KeyError, IndexError):
        return 0.0


ex = [f(r, "Instructions Executed") for r in data]
mx = max(ex)
hot = [i for i, e in enumerate(ex) if e > mx * 0.5]
lo, hi = hot[0], hot[-1]
tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
cum = 0
for i in range(lo, hi + 1):
    r = data[i]
    src = r[ix["Source"]].strip()
    smp = f(r, "Warp Stall Sampling (All Samples)")
    cum += smp
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    key = any(op.startswith(k) for k in ["LDS", "STS", "SHFL", "MUFU", "LDG", "BRA", "BAR"])
    if key or smp > mn:
        print(f"{i:5d} cum{cum:7.0f} {smp:6.0f} ss{f(r, 'stall_short_sb'):5.0f} w{f(r, 'stall_wait'):5.0f} | {src[:80]}")
print(f"hot loop {lo}-{hi}: {hi - lo + 1} instrs, {cum:.0f} of {tot:.0f} samples")
