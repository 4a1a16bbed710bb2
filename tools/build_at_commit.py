"""Build libsparseprop from the sources of an earlier commit into
paper_2302_04852_b200/build/variants/at_<commit>.so (A/B and bisection; load
with SPARSEPROP_LIB).  Measurement tool only."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2302_04852_b200 import _build as B  # noqa: E402


def build(commit):
    src = os.path.join(B.BUILD, "at_" + commit)
    csrc = os.path.join(src, "pkg", "csrc")
    os.makedirs(csrc, exist_ok=True)
    os.makedirs(os.path.join(src, "include"), exist_ok=True)
    files = subprocess.check_output(["git", "-C", ROOT, "ls-tree", "--name-only", commit,
                                     "paper_2302_04852_b200/csrc/"], text=True).split()
    for f in files + ["include/sparseprop.h"]:
        data = subprocess.check_output(["git", "-C", ROOT, "show", f"{commit}:{f}"])
        dst = os.path.join(src, "include" if f.startswith("include") else os.path.join("pkg", "csrc"),
                           os.path.basename(f))
        open(dst, "wb").write(data)
    bsrc = subprocess.check_output(["git", "-C", ROOT, "show", f"{commit}:paper_2302_04852_b200/_build.py"], text=True)
    ns = {}
    line = [l for l in bsrc.splitlines() if l.startswith("SOURCES")][0]
    exec(line, ns)
    objs = []
    for s in ns["SOURCES"]:
        o = os.path.join(src, s.replace(".cu", ".o"))
        subprocess.check_call([B.NVCC, *B.ARCH, *B.FLAGS, "-c", os.path.join(csrc, s), "-o", o],
                              stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        objs.append(o)
    os.makedirs(os.path.join(B.BUILD, "variants"), exist_ok=True)
    lib = os.path.join(B.BUILD, "variants", f"at_{commit}.so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"])
    return lib


if __name__ == "__main__":
    for c in sys.argv[1:]:
        print(build(c))
