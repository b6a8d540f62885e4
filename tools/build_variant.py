"""Build libvtgs with extra -D defines into paper_2506_02741_b200/ab/<name>.so (compile-time A/B
variants for tools/gpu_lib_ab.sh; not used by the tests or the product path)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_02741_b200 import build as b
name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(b.HERE, "ab")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, name + ".so")
cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *[f"-D{d}" for d in defs], *[os.path.join(b.CSRC, s) for s in b.SOURCES], "-o", out]
subprocess.check_call(cmd, cwd=b.CSRC)
print(out)
