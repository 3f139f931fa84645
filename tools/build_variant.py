"""Build an EXPERIMENT copy of libvlcache.so with extra nvcc flags (timing studies only; never the
product library): python tools/build_variant.py out.so -DFOO=1 ..."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2512_12977_b200 import _build as B  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
objdir = os.path.join("/tmp", "vlc_variant_" + os.path.basename(out))
os.makedirs(objdir, exist_ok=True)


def one(src):
    obj = os.path.join(objdir, src.replace(".cu", ".o"))
    subprocess.run([B.NVCC, *B.FLAGS, *extra, "-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
    return obj


with ThreadPoolExecutor(len(B.SOURCES)) as ex:
    objs = list(ex.map(one, B.SOURCES))
subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs], check=True)
print(out)
