"""Build an experiment variant of libcc.so with extra nvcc defines (e.g. -DDF_STAGES=5) into
variants/<name>.so; select it with CC_LIB=variants/<name>.so.  Usage: build_variant.py name -DX=1 ...
VARIANT_SRC (comma list, default "dataflow") selects the sources compiled with the defines."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02257_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.ROOT, "variants")
os.makedirs(out_dir, exist_ok=True)
B.build()
objs = []
for src in B._sources():
    rel = os.path.relpath(src, B.CSRC).replace(os.sep, "_")
    obj = os.path.join(B.OBJ, rel + ".o")
    if src.endswith(".cu") and any(k in src for k in os.environ.get("VARIANT_SRC", "dataflow").split(",")):
        obj = os.path.join(out_dir, name + "_" + rel + ".o")
        subprocess.run([B.NVCC] + B.ARCH + B.FLAGS + defs + ["-c", src, "-o", obj], check=True)
    objs.append(obj)
lib = os.path.join(out_dir, name + ".so")
subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs, check=True)
print(lib)
