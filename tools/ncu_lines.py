"""Per-CUDA-source-line samples / instructions of an ncu report (needs -lineinfo):
python tools/ncu_lines.py rep.ncu-rep file.cu [ranges "name:lo-hi,..."]"""
import csv, io, subprocess, sys, collections
rep, fname = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
stall_cols = [(i, n) for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]
per_line = collections.defaultdict(lambda: [0, 0, collections.Counter()])
infile = False
num = lambda v: int(v) if v not in ("", "-") else 0
for r in rows:
    if r and r[0] == "File Path":
        infile = r[1].endswith(fname)
        continue
    if not infile or len(r) < len(hdr) or not r[0] or r[0] == "Line No":
        continue
    try:
        cur = int(r[0])     # CUDA line rows carry the per-line aggregates
    except ValueError:
        continue
    r = r[:4] + r[len(r) - (len(hdr) - 4):]     # source text may hold unescaped quotes: align from the end
    per_line[cur][0] += num(r[iS])
    per_line[cur][1] += num(r[iE])
    for i, n in stall_cols:
        v = num(r[i])
        if v:
            per_line[cur][2][n[6:]] += v
ranges = []
if len(sys.argv) > 3:
    for part in sys.argv[3].split(","):
        name, lr = part.split(":")
        lo, hi = map(int, lr.split("-"))
        ranges.append((name, lo, hi))
tot_s = sum(v[0] for v in per_line.values()); tot_e = sum(v[1] for v in per_line.values())
print(f"total samples {tot_s}, warp instructions {tot_e}")
for name, lo, hi in ranges:
    s = sum(v[0] for l, v in per_line.items() if lo <= l <= hi)
    e = sum(v[1] for l, v in per_line.items() if lo <= l <= hi)
    c = collections.Counter()
    for l, v in per_line.items():
        if lo <= l <= hi: c.update(v[2])
    print(f"{name:10s} lines {lo}-{hi}: samples {s:6d} ({100*s/max(tot_s,1):4.1f}%)  instr {e:10d} ({100*e/max(tot_e,1):4.1f}%)  top stalls {c.most_common(4)}")
top = sorted(per_line.items(), key=lambda kv: -kv[1][0])[:25]
for l, v in sorted(top):
    print(f"line {l:5d}: samples {v[0]:6d} instr {v[1]:9d}  {v[2].most_common(3)}")
