"""Build a variant of libvlmp.so with extra -D flags into scripts/vlibs/ (dev aid, CPU; travels with gpurun).

    python scripts/build_variant.py NAME -DVLMP_ROWPAIR=1 [...]   -> scripts/vlibs/libvlmp_NAME.so
Prints the ptxas register / spill lines of k_tile32. Select it with VLMP_LIB=<path>.
"""
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_13447_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(b.ROOT, "scripts", "vlibs")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, f"libvlmp_{name}.so")
cmd = [b.nvcc(), *b.NVCC_FLAGS, "-Xptxas=-v", *defs, "-o", out, *b.SRCS]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    print("\n".join(l for l in r.stderr.splitlines() if "error" in l or "^" in l)[-3000:])
    sys.exit(r.returncode)
lines = r.stderr.splitlines()
for k, line in enumerate(lines):
    if "k_tile32" in line and "Compiling entry" in line:
        for l2 in lines[k + 1:k + 4]:
            if re.search(r"registers|spill", l2):
                print(name, l2.strip())
print(out)
