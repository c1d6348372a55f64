"""Registers and spills of every conv_tz_kernel instantiation (nvcc -Xptxas -v on conv_tz.cu).
usage: python tools/ptxas_report.py [source.cu] [extra nvcc flags, e.g. -DTN_EXP64=8]"""
import re, subprocess, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "paper_1801_09449_b200", "csrc", sys.argv[1] if len(sys.argv) > 1 else "conv_tz.cu")
r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
                    "-Xptxas", "-v", "-c", src, "-o", "/tmp/ptxas_report.o"] + sys.argv[2:], capture_output=True, text=True)
cur = None
info = {}
for line in r.stderr.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        info.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        info.setdefault(cur, {})["regs"] = int(m.group(1))
for k, v in sorted(info.items()):
    m = re.search(r"conv_tz_kernelILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)ELb(\d)ELb(\d)E", k)
    if m:
        K, CT, NS, S, P, F, F4 = m.groups()
        print(f"K={K:2s} CT={CT} NSEG={NS} S={S} PRED={P} FIRST={F} F4={F4}  regs {v.get('regs')}  spill {v.get('spill')}")
