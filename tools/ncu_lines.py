"""Aggregate an ncu source page (--print-source cuda,sass --csv) into per-CUDA-line stall samples."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = collections.Counter(); src = {}
fname = None; cur = None; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0]:  # a CUDA line row
        cur = (fname, int(r[0])); src[cur] = r[1].strip()[:100]
        continue
    try: v = int(r[4])
    except (ValueError, IndexError): continue
    if cur: agg[cur] += v
tot = sum(agg.values())
print("total samples", tot)
for k, v in agg.most_common(top):
    print(f"{100*v/tot:5.1f}% {k[0]}:{k[1]}  {src.get(k,'')}")
