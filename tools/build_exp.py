"""Build experiment variants of libtn.so into exp/ (e.g. python tools/build_exp.py prof:-DTN_EXP_PROF=1 noepi:-DTN_EXP_PROF=1,-DTZ_EXP_NOEPI=1)."""
import concurrent.futures as cf, subprocess, sys
def b(spec):
    name, flags = spec.split(":", 1)
    extra = [f for f in flags.split(",") if f]
    code = ("import sys; sys.path.insert(0,'paper_1801_09449_b200'); import build; "
            f"build.build_library(extra={extra!r}, lib_path='exp/libtn_{name}.so', obj_dir='exp/obj_{name}')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    return name, r.returncode, r.stderr[-400:]
with cf.ThreadPoolExecutor(4) as ex:
    for name, rc, err in ex.map(b, sys.argv[1:]):
        print(name, "ok" if rc == 0 else "FAILED\n" + err)
