"""Build an A/B variant of libsparseprop with extra -D defines into
paper_2302_04852_b200/build/variants/<name>.so (git-ignored; travels with
gpurun snapshots).  Load it with SPARSEPROP_LIB=<path>.  Measurement tool only:
the product is the default build."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_04852_b200 import _build as B  # noqa: E402


def build(name, defines):
    out = os.path.join(B.BUILD, "variants", name)
    os.makedirs(out, exist_ok=True)

    def one(src):
        obj = os.path.join(out, src.replace(".cu", ".o"))
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *[f"-D{d}" for d in defines], "-c", os.path.join(B.CSRC, src), "-o", obj]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode:
            raise RuntimeError(p.stderr)
        return obj
    with cf.ThreadPoolExecutor(len(B.SOURCES)) as ex:
        objs = list(ex.map(one, B.SOURCES))
    lib = os.path.join(B.BUILD, "variants", name + ".so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"])
    return lib


if __name__ == "__main__":
    print(build(sys.argv[1], sys.argv[2:]))
