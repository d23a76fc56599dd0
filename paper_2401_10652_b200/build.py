"""Build libautochunk.so in-tree with nvcc (sm_100a) and g++.

    python -m paper_2401_10652_b200.build      (or __graft_entry__.build())

CUDA sources: -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
Host planner sources: -O2 -ffp-contract=off (plans must be bit-identical to the
Python oracle's IEEE-double arithmetic).
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libautochunk.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    try:
        import nvidia.nccl  # noqa: F401
        base = os.path.dirname(sys.modules["nvidia.nccl"].__file__ or "")
        if not base:
            base = list(sys.modules["nvidia.nccl"].__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    return None


def sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    return cu, cpp


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def _digest(path, flags):
    h = hashlib.sha256()
    h.update(" ".join(flags).encode())
    with open(path, "rb") as f:
        h.update(f.read())
    for hdr in sorted(os.listdir(CSRC)):
        if hdr.endswith((".h", ".cuh")):
            with open(os.path.join(CSRC, hdr), "rb") as f:
                h.update(f.read())
    for hdr in sorted(os.listdir(os.path.join(ROOT, "include"))):
        with open(os.path.join(ROOT, "include", hdr), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cu, cpp = sources()
    inc = ["-I" + CSRC, "-I" + os.path.join(ROOT, "include")]
    ninc = _nccl_include()
    defs = []
    if os.environ.get("AC_DEBUG_HANG"):
        defs.append("-DAC_DEBUG_HANG=1")
    for d in os.environ.get("AC_EXTRA_DEFS", "").split():  # experiments: variants at build time
        defs.append("-D" + d)
    if ninc:
        inc.append("-I" + ninc)
        defs.append("-DAC_HAVE_NCCL_H=1")
    cu_flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                       "-Xptxas", "-v"] + inc + defs
    cpp_flags = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-I/usr/local/cuda/include"] + inc + defs
    objs = []
    jobsq = []
    for f in cu:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + "." + _digest(src, cu_flags) + ".o")
        objs.append(obj)
        if not os.path.exists(obj):
            jobsq.append([NVCC, "-c", src, "-o", obj] + cu_flags)
    for f in cpp:
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + "." + _digest(src, cpp_flags) + ".o")
        objs.append(obj)
        if not os.path.exists(obj):
            jobsq.append(["g++", "-c", src, "-o", obj] + cpp_flags)
    procs = []
    logs = []
    for cmd in jobsq:
        while len(procs) >= jobs:
            p, c = procs.pop(0)
            out, err = p.communicate()
            if p.returncode != 0:
                raise RuntimeError("build failed:\n" + " ".join(c) + "\n" + out + err)
            logs.append(err)
        procs.append((subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True), cmd))
    for p, c in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("build failed:\n" + " ".join(c) + "\n" + out + err)
        logs.append(err)
    if verbose:
        for l in logs:
            sys.stdout.write(l)
    out = os.environ.get("AC_LIB_OUT", LIB)  # experiments: a variant library beside the default
    tmp = out + ".tmp"
    _run([NVCC, "-shared", "-o", tmp] + ARCH + objs + ["-lcudart", "-ldl", "-lpthread"])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
