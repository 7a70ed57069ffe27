"""Build libzorse_b200.so (sm_100a) in-tree with nvcc.

The shared library is the drop-in C-ABI boundary declared in include/zorse_b200.h.
It is built into the package directory so it travels with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libzorse_b200.so")
OBJDIR = os.path.join(HERE, "..", "build", "obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_paths():
    """Torch-bundled NCCL (2.28.x) headers and library, used at runtime by torch too."""
    site = sysconfig.get_paths()["purelib"]
    root = os.path.join(site, "nvidia", "nccl")
    inc = os.path.join(root, "include")
    lib = os.path.join(root, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(verbose: bool = False, jobs: int = 8, defines=(), out: str = OUT) -> str:
    """Compile every csrc/ source for sm_100a and link the C-ABI library.
    ``defines`` / ``out``: experiment builds (separate object dir, other .so name)."""
    objdir = OBJDIR if not defines else OBJDIR + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(objdir, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_paths()
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    headers.append(os.path.join(HERE, "..", "include", "zorse_b200.h"))
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    cmds = []
    objs = []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        if _newer(obj, [src] + headers):
            continue
        cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", CSRC, "-I", os.path.join(HERE, "..", "include"), "-I", nccl_inc,
               *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        else:  # host planner code: no FMA contraction (bit parity with the Python planner)
            cmd[1:1] = ["-Xcompiler", "-ffp-contract=off"]
        cmds.append(cmd)
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        if len(procs) >= jobs:
            _drain(procs, verbose)
    _drain(procs, verbose)
    if cmds or not os.path.exists(out):
        link = ["nvcc", *ARCH, "-shared", "-o", out, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
                "-Xlinker", "-rpath", "-Xlinker", nccl_lib, "-lcudart", "-ldl"]
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.run(link, check=True)
    return out


def _drain(procs, verbose):
    while procs:
        cmd, p = procs.pop(0)
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            sys.stderr.write(text)
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
        if verbose and text.strip():
            print(text)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
