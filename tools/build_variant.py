"""Build a libskx.so variant with extra -D flags on one source file, for A/B
timing on the GPU box: tools/build_variant.py NAME SRC.cu -DFOO=1 ...
Output: tools/variants/libskx_NAME.so (git-ignored)."""
import glob
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build_libskx()
out_dir = os.path.join(B.ROOT, "tools", "variants")
os.makedirs(out_dir, exist_ok=True)
obj = os.path.join(out_dir, f"{name}_{os.path.basename(src)[:-3]}.o")
B._run([B._nvcc(), *B.NVCC_FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj])
objs = [o for o in sorted(glob.glob(os.path.join(B.OBJ, "*.o")))
        if os.path.basename(o) != os.path.basename(src)[:-3] + ".o"] + [obj]
so = os.path.join(out_dir, f"libskx_{name}.so")
B._run([B._nvcc(), *B.ARCH, "-shared", "-o", so, *objs, "-lcudart_static", "-lnccl", "-lrt",
        "-lpthread", "-ldl"])
os.remove(obj)
print(so)
