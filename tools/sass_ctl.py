"""Static view of a kernel's SASS schedule (cuobjdump -sass output): decodes each instruction's
control word (stall count, yield, write/read barrier, wait mask) and prints, per straight-line
region between labels/branches, the instruction mix, the sum of the static stall cycles (the
least time ONE warp needs to issue the region alone) and the fp64 pipe time (2 cycles per
DFMA/DADD/DMUL warp instruction on sm_100's 16-lane fp64 unit).

cuobjdump -sass -fun NAME obj.o | python tools/sass_ctl.py [--dump]
"""
import re
import sys
import collections

dump = "--dump" in sys.argv
ins = []
cur = None
for line in sys.stdin:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* 0x([0-9a-f]{16}) \*/", line)
    if m:
        cur = [int(m.group(1), 16), m.group(2).strip(), int(m.group(3), 16), None]
        continue
    m = re.match(r"\s*/\* 0x([0-9a-f]{16}) \*/", line)
    if m and cur:
        cur[3] = int(m.group(1), 16)
        ins.append(cur)
        cur = None

def ctl(hi):
    return dict(stall=(hi >> 41) & 15, yld=(hi >> 45) & 1, wr=(hi >> 46) & 7, rd=(hi >> 49) & 7, wait=(hi >> 52) & 63)

def klass(s):
    op = s.split()[0]
    if op.startswith("@"):
        op = s.split()[1]
    if op[:4] in ("DFMA", "DADD", "DMUL"):
        return "fp64"
    for k in ("LDS", "STS", "LDG", "STG", "LDGSTS", "BAR", "SHFL", "BRA", "WARPSYNC", "UBLKPF", "LDL", "STL"):
        if op.startswith(k):
            return k
    return "other"

targets = set()
for a, s, lo, hi in ins:
    m = re.search(r"BRA\S*\s+(?:\S+,\s*)?(0x[0-9a-f]+)", s)
    if m:
        targets.add(int(m.group(1), 16))

regions = []
start = 0
for i, (a, s, lo, hi) in enumerate(ins):
    k = klass(s)
    if a in targets and i > start:
        regions.append((start, i))
        start = i
    if k in ("BRA",) or s.startswith("EXIT") or "BAR.SYNC" in s:
        regions.append((start, i + 1))
        start = i + 1
if start < len(ins):
    regions.append((start, len(ins)))

print(f"{len(ins)} instructions, {len(regions)} regions")
for b, e in regions:
    if e - b < 40 and not dump:
        continue
    mix = collections.Counter()
    stall = 0
    waits = 0
    for a, s, lo, hi in ins[b:e]:
        c = ctl(hi)
        mix[klass(s)] += 1
        stall += max(c["stall"], 1)
        if c["wait"]:
            waits += 1
    f = mix["fp64"]
    print(f"[{ins[b][0]:05x}..{ins[e-1][0]:05x}] n={e-b:5d} static_stall={stall:6d} fp64={f:5d} (pipe {2*f:5d}) waits={waits:4d} "
          + " ".join(f"{k}:{v}" for k, v in mix.most_common() if k != "fp64"))
    if dump:
        for a, s, lo, hi in ins[b:e]:
            c = ctl(hi)
            print(f"   {a:05x} st={c['stall']:2d} y={c['yld']} wr={c['wr']} rd={c['rd']} wt={c['wait']:02x}  {s}")
