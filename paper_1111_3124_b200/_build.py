"""Build libmps_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

The library is split into translation units compiled in parallel and linked into
one shared object; cudart is linked statically.  Called by __graft_entry__.build().
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libmps_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
UNITS = ["capi.cu", "state.cu", "tier280.cu", "tier512.cu"]
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-diag-suppress", "177,550"]


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "mps_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """out / defines: development A/B builds (e.g. out=libmps_b200_x.so, defines=["JACOBI_GAUSS_D=0"])
    loaded with MPS_B200_SO=<path>; the default build is the product library."""
    if out is None and not force and up_to_date():
        return OUT
    target = out or OUT
    objdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out).split(".")[0])
    os.makedirs(objdir, exist_ok=True)

    def compile_unit(u):
        src = os.path.join(CSRC, u)
        obj = os.path.join(objdir, u.replace(".cu", ".o"))
        cmd = [NVCC] + FLAGS + ["-D" + d for d in defines] + ["-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {u}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    units = [u for u in UNITS if os.path.exists(os.path.join(CSRC, u))]
    with cf.ThreadPoolExecutor(max_workers=len(units)) as ex:
        res = list(ex.map(compile_unit, units))
    if verbose:
        for _, err in res:
            sys.stderr.write(err)
    objs = [o for o, _ in res]
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", target] + objs + ["-cudart", "static"]
    subprocess.check_call(cmd)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
