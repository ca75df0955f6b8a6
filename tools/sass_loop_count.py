"""Count SASS instructions in the hottest loop of a kernel (the basic-block region between the
back-branch and its target that contains the most MUFU.EX2).  Usage:
  python tools/sass_loop_count.py <.so or .cubin> <kernel-substring>"""
import re
import subprocess
import sys
from collections import Counter


MIN_EX2 = 16
REQ_RCP = 1


def main(path, kname):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    body = next(f for f in funcs if kname in f.split("\n")[0])
    lines = [ln for ln in body.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln)]
    ins = []
    for ln in lines:
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for k, (addr, txt) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
        if not m or not m.group(1):
            continue
        tgt = int(m.group(1), 16)
        if tgt < addr:
            region = [t for a, t in ins if tgt <= a <= addr]
            ex2 = sum("MUFU.EX2" in t for t in region)
            # innermost loop holding the event steps: smallest region with >= min_ex2 exps
            rcp = sum("MUFU.RCP" in t for t in region)
            if ex2 >= MIN_EX2 and rcp >= REQ_RCP and (best is None or len(region) < len(best[1])):
                best = (ex2, region)
    if best is None:
        print("no loop found")
        return
    ex2, region = best
    ops = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in region)
    print(f"hot loop: {len(region)} instrs, {ex2} MUFU.EX2 -> {len(region) / (ex2 / 2):.1f} instrs per event-step")
    print(", ".join(f"{k} {v}" for k, v in ops.most_common()))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
