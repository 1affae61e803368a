"""Build an experimental variant of the library: lib/libdsssp_<name>.so with
extra -D flags (select it at run time with DS_LIB=...)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_06895_b200 import build as b
name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(b.LIB_DIR, f"libdsssp_{name}.so")
cmd = [b._nvcc(), *b.NVCC_FLAGS, *flags, "-o", out, *[os.path.join(b.CSRC, s) for s in b.SOURCES]]
subprocess.run(cmd, check=True)
print(out)
