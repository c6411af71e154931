"""Experiment helper: build libmdcuda.so variants that differ in -D flags of the fused-kernel
translation units only (the other objects come from the regular build cache).

usage: python scripts/build_variant.py TAG [-DNAME=V ...]  -> variants/libmdcuda_TAG.so
Select at run time with MD_LIB=variants/libmdcuda_TAG.so.
"""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_2245_b200 import build as B

VARIED = tuple(os.environ.get("MD_VARIED", "md_fused_box_a.cu md_fused_box_b.cu md_fused.cu").split())
tag, defs = sys.argv[1], sys.argv[2:]
# run the regular build first: its object cache supplies the unchanged translation units
out_dir = os.path.join(B.ROOT, "build", "variants")
os.makedirs(out_dir, exist_ok=True)
objs = []
for f in sorted(os.listdir(B.OBJ)):
    if f.endswith(".o") and not any(f.startswith(v[:-3] + "-") for v in VARIED):
        objs.append(os.path.join(B.OBJ, f))


def cc(src):
    o = os.path.join(out_dir, f"{tag}-{src[:-3]}.o")
    r = subprocess.run([B._nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", o],
                       capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    return o


with ThreadPoolExecutor(3) as ex:
    objs += list(ex.map(cc, VARIED))
so_dir = os.path.join(B.ROOT, "variants")              # git-ignored, travels with gpurun
os.makedirs(so_dir, exist_ok=True)
so = os.path.join(so_dir, f"libmdcuda_{tag}.so")
subprocess.run([B._nvcc(), *B.ARCH, "-shared", "-o", so, *objs, "-lcudart"], check=True)
print(so)
