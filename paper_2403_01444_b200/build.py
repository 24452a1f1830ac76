"""Build the sm_100a C-ABI library `libss_b200.so` in-tree with nvcc.

python -m paper_2403_01444_b200.build   (also called by __graft_entry__.build())
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libss_b200.so")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC]


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _compile(src: str, obj: str = OBJ, defs: tuple = ()) -> tuple[str, str]:
    out = os.path.join(obj, src[:-3] + ".o")
    inp = os.path.join(CSRC, src)
    deps = [inp] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    deps.append(os.path.join(INCLUDE, "ss_b200.h"))
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out, ""
    cmd = [NVCC, *ARCH, *FLAGS, *defs, "-c", inp, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(out + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return out, r.stderr


def build(verbose: bool = False, defs: tuple = (), lib: str = LIB, obj: str = OBJ) -> str:
    """defs / lib / obj: a tuning variant (-D flags) built beside the product
    library, e.g. for tools/ A/B runs with SS_LIB pointing at it."""
    os.makedirs(obj, exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda f: _compile(f, obj, tuple(defs)), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for o, log in results:
            if log:
                print(log, file=sys.stderr)
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(lib) or os.path.getmtime(lib) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    # python -m paper_2403_01444_b200.build [-v] [--variant NAME -DX=1 ...]
    args = sys.argv[1:]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        defs = tuple(a for a in args if a.startswith("-D"))
        print(build("-v" in args, defs, os.path.join(ROOT, "build", f"libss_b200_{name}.so"),
                    os.path.join(ROOT, "build", f"obj_{name}")))
    else:
        print(build(verbose="-v" in args))
