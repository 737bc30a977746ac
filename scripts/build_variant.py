"""Development aid: build libtc_b200.so variants with -D overrides into variants/<name>/."""
import os, subprocess, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1804_06926_b200 import _build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(B.HERE, "..", "variants", name)
os.makedirs(out, exist_ok=True)
objs = []
for src in B.SOURCES:
    obj = os.path.join(out, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.FLAGS, *["-D" + d for d in defs], "-c", os.path.join(B.CSRC, src), "-o", obj],
                   check=True, capture_output=True)
    objs.append(obj)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", os.path.join(out, "libtc_b200.so"), *objs], check=True)
print("built", name, defs)
