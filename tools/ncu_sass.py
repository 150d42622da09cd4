"""Per-kernel SASS view of an ncu source page (ncu -i X.ncu-rep --page source --csv --print-source cuda,sass):
stall samples by opcode class and reason, and the hottest instructions with their CUDA line.

python tools/ncu_sass.py src.csv [KERNEL_SUBSTRING] [TOP]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30

hdr = None
func = None
fname = None
line = None
per = collections.defaultdict(list)  # func -> [(addr, sass, samples, stalls{}, file, line, executed)]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        line = (fname, int(r[0]))
        continue
    try:
        samples = int(r[4])
        execd = int(r[7])
    except (ValueError, IndexError):
        continue
    st = {}
    for i, h in enumerate(hdr):
        if not h.startswith("stall_") or "Not" in h or i >= len(r):
            continue
        try:
            v = int(r[i])
        except ValueError:
            v = 0
        if v:
            st[h.replace("stall_", "")] = v
    per[func].append((r[2], r[3].strip(), samples, st, line, execd))


def klass(s):
    op = s.split()[0] if s else "?"
    if op.startswith("@"):
        op = s.split()[1]
    for k in ("DFMA", "DADD", "DMUL"):
        if op.startswith(k):
            return "fp64"
    for k in ("LDS", "STS", "LDG", "STG", "LDGSTS", "BAR", "SHFL", "LDC", "WARPSYNC", "LDGDEPBAR", "DEPBAR", "UBLKPF"):
        if op.startswith(k):
            return k
    return "other"


for f, ins in per.items():
    if want not in f:
        continue
    tot = sum(i[2] for i in ins)
    print(f"== {f}: {len(ins)} SASS instructions, {tot} samples")
    byk = collections.Counter()
    byk_n = collections.Counter()
    byk_exec = collections.Counter()
    byr = collections.Counter()
    bykr = collections.defaultdict(collections.Counter)
    for a, s, n, st, ln, ex in ins:
        k = klass(s)
        byk[k] += n
        byk_n[k] += 1
        byk_exec[k] += ex
        for r, v in st.items():
            byr[r] += v
            bykr[k][r] += v
    print("  by reason: " + ", ".join(f"{r} {100*v/tot:.1f}%" for r, v in byr.most_common(10)))
    for k, v in byk.most_common():
        print(f"  {k:8s} {100*v/tot:5.1f}% of samples, {byk_n[k]:5d} static, {byk_exec[k]:9d} executed | "
              + ", ".join(f"{r} {100*x/tot:.1f}" for r, x in bykr[k].most_common(5)))
    print("  hottest instructions:")
    for a, s, n, st, ln, ex in sorted(ins, key=lambda i: -i[2])[:top]:
        print(f"   {100*n/tot:5.2f}% {s[:60]:60s} {ln[0]}:{ln[1]} " + ",".join(f"{r}:{v}" for r, v in sorted(st.items(), key=lambda x: -x[1])[:3]))
