"""Build an A/B variant library fast: recompile only the given sources (default
inst_f32.cu) with extra -D defines, link with the in-tree objects of everything else.

    python tools/quick_variant.py lib_x.so MM_LW_SLEEP=0 [--src inst_f32.cu,inst_u8.cu]
"""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_cs_0610046_b200 import _build  # noqa: E402

args = sys.argv[1:]
srcs = ["inst_f32.cu"]
if "--src" in args:
    i = args.index("--src")
    srcs = args[i + 1].split(",")
    del args[i:i + 2]
out, defines = args[0], args[1:]
tag = "_".join(d.replace("=", "") for d in defines) or "plain"
bdir = f"/tmp/qv_{tag}"
os.makedirs(bdir, exist_ok=True)
nv = _build._nvcc()
procs = []
for s in srcs:
    o = os.path.join(bdir, s[:-3] + ".o")
    cmd = [nv, *_build.ARCH, *_build.NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(_build.CSRC, s), "-o", o]
    procs.append(subprocess.Popen(cmd))
assert all(p.wait() == 0 for p in procs)
objs = [os.path.join(bdir, s[:-3] + ".o") if os.path.basename(o)[:-2] + ".cu" in srcs else o
        for o in sorted(glob.glob(os.path.join(_build.BUILD, "*.o")))]
lib = os.path.join(_build.HERE, out)
subprocess.run([nv, *_build.ARCH, "-shared", "-o", lib, *objs], check=True)
print(lib)
