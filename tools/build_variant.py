"""Build a development variant of libsptrsv.so with extra -D flags:
python tools/build_variant.py NAME -DSPTRSV_BLOCK_FW=4 ...  ->  paper_1710_04985_b200/lib/var_NAME.so
(select it with SPTRSV_DEV_LIB=<path>)."""
import os
import subprocess
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1710_04985_b200 import build as B

name, flags = sys.argv[1], sys.argv[2:]
odir = os.path.join(B.LIBDIR, f"obj_{name}")
os.makedirs(odir, exist_ok=True)
objs = []
for cu in [s for s in B.sources() if s.endswith(".cu")]:
    o = os.path.join(odir, os.path.basename(cu)[:-3] + ".o")
    subprocess.check_call([B.nvcc(), *B.NVCC_FLAGS, *flags, "-I" + B.INCLUDE, "-I" + B.CSRC, "-c", "-o", o, cu])
    objs.append(o)
out = os.path.join(B.LIBDIR, f"var_{name}.so")
subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out, *objs])
print(out)
