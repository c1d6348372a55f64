"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: python tools/launches.py file.csv [last_n]."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if 'Kernel Name' in r)
out = []
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d['Metric Name'] == 'gpu__time_duration.sum':
        name = d['Kernel Name'].split('(')[0].replace('tn::<unnamed>::', '')
        out.append((name, float(d['Metric Value'].replace(',', '')) / 1e3, d.get('Grid Size', ''), d.get('Block Size', '')))
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(out)
sel = out[-last:]
tot = sum(o[1] for o in sel)
for o in sel:
    print(f"{o[0][:60]:60s} {o[1]:9.1f} us {100*o[1]/tot:5.1f}%  grid {o[2]} blk {o[3]}")
print(f"total {tot:.1f} us over {len(sel)} launches")
