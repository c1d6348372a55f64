"""Key metrics + SASS hot spots of an ncu report: python tools/ncu_summary.py rep.ncu-rep [nsass]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]
nsass = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
pat = (r'^dram__bytes_(read|write)\.sum$|^gpu__time_duration.sum$|imma_cycles_active.avg.pct_of_peak_sustained_active|'
       r'^sm__throughput.avg.pct_of_peak_sustained_elapsed|pipe_shared_cycles_active.avg.pct_of_peak_sustained_active|'
       r'^sm__inst_executed_pipe_(alu|lsu|fma|adu|xu|uniform|cbu).avg.pct_of_peak_sustained_active|'
       r'^smsp__inst_executed.sum$|^smsp__issue_active.avg.pct_of_peak_sustained_active|launch__registers_per_thread$|'
       r'sm__cycles_elapsed.avg.per_second|launch__grid_size|l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum$|'
       r'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum$')
for k, un, x in zip(h, u, v):
    if re.search(pat, k):
        print(f"{k:70s} {x} {un}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = [x for x in rows[2:] if len(x) == len(hh)]
iS, iE, iSrc = hh.index('Warp Stall Sampling (All Samples)'), hh.index('Instructions Executed'), hh.index('Source')
tot_s = sum(int(x[iS] or 0) for x in data)
tot_e = sum(int(x[iE] or 0) for x in data)
print(f"stall samples {tot_s}, warp instructions {tot_e}")
top = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:nsass]
for i in sorted(top):
    x = data[i]
    print(f"{i:5d} {x[iSrc].strip()[:64]:64s} samples {x[iS]:>6s} exec {x[iE]:>9s}")
