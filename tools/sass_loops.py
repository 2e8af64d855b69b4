"""List the backward-branch loops of one kernel's SASS with their op mix.
    python tools/sass_loops.py file.o mangled_name [min_len]"""
import collections, re, subprocess, sys
obj, fn = sys.argv[1], sys.argv[2]
minlen = int(sys.argv[3]) if len(sys.argv) > 3 else 100
txt = subprocess.run(["cuobjdump", "-sass", "-fun", fn, obj], capture_output=True, text=True).stdout
ins = []
for line in txt.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = [a for a, _ in ins]
for k, (a, t) in enumerate(ins):
    m = re.search(r"\bBRA(?:\.\w+)*\s+(?:`?\(?\.?L?_?x?_?\d*\)?)?\s*0x([0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a:
        continue
    body = [x for aa, x in ins if tgt <= aa <= a]
    if len(body) < minlen:
        continue
    c = collections.Counter()
    for x in body:
        op = x.split()[0]
        if op.startswith("@"):
            op = x.split()[1]
        c[op.split(".")[0]] += 1
    print(f"loop {tgt:#x}-{a:#x} len={len(body)}: " + ", ".join(f"{o}={n}" for o, n in c.most_common(12)))
