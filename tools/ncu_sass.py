"""SASS of an ncu source page (--page source --csv --print-source cuda,sass) in address order, with
samples / executed / top stall reasons, for the CUDA lines [lo, hi] of one file.
usage: python tools/ncu_sass.py page.csv file.cu lo hi [min_samples]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
fname, lo, hi = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
mins = int(sys.argv[5]) if len(sys.argv) > 5 else 0
hdr = next(r for r in rows if r and r[0] == "Line No")
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stalls = [(i, n[6:]) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
cur, infile, out = None, False, []
for r in rows:
    if r and r[0] == "File Path":
        infile = r[1].endswith(fname)
        continue
    if not infile or not r or r[0] == "Line No":
        continue
    if r[0].isdigit():
        cur = int(r[0])
        continue
    if cur is None or not (lo <= cur <= hi) or len(r) < len(hdr) or not r[2].startswith("0x"):
        continue
    num = lambda v: int(v) if v not in ("", "-") else 0
    c = collections.Counter({n: num(r[i]) for i, n in stalls if num(r[i])})
    out.append((int(r[2], 16), cur, r[3].strip(), num(r[iS]), num(r[iE]), c))
tot = sum(o[3] for o in out)
print(f"samples in range: {tot}")
for addr, ln, sass, s, e, c in sorted(out):
    if s >= mins:
        print(f"{addr & 0xfffff:6x} L{ln:<5d} {s:5d} {e:9d}  {sass[:60]:60s} {c.most_common(2)}")
