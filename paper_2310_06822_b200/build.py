"""Build libnb.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2310_06822_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libnb.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE,
          "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES = {
    "nb_api.cu": [],
    "nb_simt.cu": [],
    "nb_fwd_tc.cu": [],
    "nb_fwd_tc_w64l4_d3.cu": [],
    "nb_fwd_tc_w128l4_d6.cu": [],
    "nb_fwd_tc_w128l6h24_d4.cu": [],
    "nb_fwd_tc_gen32.cu": [],
    "nb_fwd_tc_gen64.cu": [],
    "nb_fwd_tc_gen128.cu": [],
    "nb_fwd_tc2.cu": [],
    "nb_train_tc.cu": [],
    "nb_train_tc2.cu": [],
    "nb_train_fused.cu": [],
    "nb_fwd_exit.cu": [],
    "nb_hier.cu": [],
    "nb_fwd_tc_ext32.cu": [],
    "nb_fwd_tc_ext64.cu": [],
    "nb_fwd_tc_ext128.cu": [],
    "nb_label.cu": ["-fmad=false"],   # exact fp64 DDA rounding (no FMA contraction)
    "nb_comm.cpp": [],
}
HEADERS = ["nb_internal.cuh", "nb_device.cuh", "nb_fwd_tc.cuh", "nb_adam.cuh"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, extra: list[str], objdir: str = OBJ) -> tuple[str, str]:
    obj = os.path.join(objdir, src + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(INCLUDE, "nb.h"), __file__]
    if not _stale(obj, deps):
        return obj, ""
    lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
    cmd = [NVCC] + lang + ARCH + COMMON + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, defines: tuple = (), name: str = "",
          only: tuple = ()) -> str:
    """Build libnb.so; `defines` (e.g. ("NB_W64_NSLOT=5",)) + `name` build a
    measurement variant libnb_<name>.so from its own object directory; with
    `only`, just those sources get the defines (the rest link the main objects)."""
    objdir = os.path.join(OBJ, name) if name else OBJ
    lib = os.path.join(HERE, f"libnb_{name}.so") if name else LIB
    os.makedirs(objdir, exist_ok=True)
    if force:
        for f in os.listdir(objdir):
            if os.path.isfile(os.path.join(objdir, f)):
                os.remove(os.path.join(objdir, f))
    dflags = [f"-D{d}" for d in defines]
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        futs = {s: ex.submit(_compile, s, e + (dflags if not only or s in only else []),
                             objdir if not only or s in only else OBJ)
                for s, e in SOURCES.items()}
        objs = []
        for s, f in futs.items():
            obj, log = f.result()
            objs.append(obj)
            if verbose and log:
                print(f"[{s}]\n{log}")
    if force or _stale(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    nm = next((a[7:] for a in sys.argv[1:] if a.startswith("--name=")), "")
    on = tuple(x for a in sys.argv[1:] if a.startswith("--only=") for x in a[7:].split(","))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs, name=nm, only=on))
