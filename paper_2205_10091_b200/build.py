"""Build libtcx.so in-tree for sm_100a (nvcc; no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtcx.so")
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
              "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


# (source, output, extra defines): pass_inst.cu is compiled once per precision x mode
UNITS = [("tcx.cu", "tcx.o", []), ("plan.cpp", "plan.o", [])] + [
    ("pass_inst.cu", f"pass_{tag}_{km}.o", [f"-DTCX_REAL={real}", f"-DTCX_TAG={tag}", f"-DTCX_KM={km}"])
    for real, tag in (("float", "f32"), ("double", "f64")) for km in (0, 1, 2)]


def _deps():
    return [os.path.join(CSRC, f) for f in ("tcx.cu", "plan.cpp", "pass_inst.cu", "kernels.cuh",
                                             "plan.h")] + [os.path.join(ROOT, "include", "tcx.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for name, oname, defs in UNITS:
        src = os.path.join(CSRC, name)
        obj = os.path.join(bdir, oname)
        if src.endswith(".cu"):
            cmd = [nvcc, "-c", src, "-o", obj] + ARCH + NVCC_FLAGS + defs
        else:
            cmd = ["g++", "-c", src, "-o", obj, "-O2", "-std=c++17", "-fPIC",
                   "-I" + os.path.join(ROOT, "include")]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("build failed: " + " ".join(cmd))
        if verbose:
            sys.stderr.write(out.decode())
        if cmd[0] == nvcc:
            with open(os.path.join(bdir, os.path.basename(cmd[4]) + ".ptxas.log"), "w") as f:
                f.write(out.decode())
    tmp = LIB + ".tmp"
    link = [nvcc, "-shared", "-o", tmp] + objs + ARCH + ["-cudart", "static", "-Xcompiler", "-fPIC"]
    subprocess.check_call(link)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
