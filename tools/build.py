#!/usr/bin/env python3
"""Build every native artefact in-tree (the .so files travel to the GPU box).

Targets:
  oracle       oracle/liboracle.so            gcc, -O2 -ffp-contract=off -fno-fast-math (CPU oracle)
  inputs       inputs/libmoa_inputs.so         gcc (host input generator)
  inputs_cuda  inputs/libmoa_inputs_cuda.so    nvcc sm_100a (device input generator)
  moa          paper_2306_11148_b200/libmoa.so nvcc sm_100a (the product: C-ABI + kernels, links NCCL)
  shim         tests/nccl_shim/libmoa_nccl_shim.so  test-only NCCL stand-in (several ranks on one GPU)
  all          everything (default)

Incremental: a target is rebuilt only when a source/header is newer than its output
(or with --force). The oracle and the product share no sources, headers or flags.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_root() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl")
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found (torch-bundled nvidia/nccl expected)")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]):
    print("  $", " ".join(cmd), flush=True)
    subprocess.check_call(cmd, cwd=ROOT)


def build_oracle(force=False):
    src = os.path.join(ROOT, "oracle", "moa_oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared", "-pthread",
              src, "-o", out, "-lm"])
    return out


def build_inputs(force=False):
    src = os.path.join(ROOT, "inputs", "moa_inputs.c")
    hdr = os.path.join(ROOT, "inputs", "moa_inputs.h")
    out = os.path.join(ROOT, "inputs", "libmoa_inputs.so")
    if force or _stale(out, [src, hdr]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", src, "-o", out])
    return out


def build_inputs_cuda(force=False):
    src = os.path.join(ROOT, "inputs", "moa_inputs_cuda.cu")
    hdr = os.path.join(ROOT, "inputs", "moa_inputs.h")
    out = os.path.join(ROOT, "inputs", "libmoa_inputs_cuda.so")
    if force or _stale(out, [src, hdr]):
        _run([NVCC, *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", src, "-o", out])
    return out


def build_moa(force=False, verbose_ptxas=False):
    pkg = os.path.join(ROOT, "paper_2306_11148_b200")
    csrc = os.path.join(pkg, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cu")) + glob.glob(os.path.join(csrc, "*.cpp")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))
    out = os.path.join(pkg, "libmoa.so")
    nccl = _nccl_root()
    objdir = os.path.join(ROOT, "build", "moa")
    os.makedirs(objdir, exist_ok=True)
    if not (force or _stale(out, srcs + hdrs)):
        return out
    common = [*ARCH, "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
              "-I", csrc, "-I", os.path.join(nccl, "include")]
    if verbose_ptxas:
        common += ["-Xptxas", "-v"]
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC, *common, "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    _run([NVCC, *ARCH, "-shared", *objs, "-o", out, "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
          "-Xlinker", "-rpath=" + os.path.join(nccl, "lib"), "-lcudart"])
    return out


def build_shim(force=False):
    """tests/nccl_shim/libmoa_nccl_shim.so: TEST INFRASTRUCTURE (an LD_PRELOAD stand-in for
    the NCCL subset libmoa.so calls, so several processes can share one GPU in the
    multi-rank tests). Never linked into the product."""
    src = os.path.join(ROOT, "tests", "nccl_shim", "moa_nccl_shim.cu")
    out = os.path.join(ROOT, "tests", "nccl_shim", "libmoa_nccl_shim.so")
    nccl = _nccl_root()
    if force or _stale(out, [src]):
        _run([NVCC, *ARCH, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(nccl, "include"),
              src, "-o", out, "-L/usr/local/cuda/lib64/stubs", "-lcuda", "-lcudart"])
    return out


def build_asan(force=False):
    """Sanitizer builds of the HOST code (tests/test_sanitizers.py): the oracle, and
    libmoa.so with moa_host.cpp / moa_tma.cpp compiled by g++ -fsanitize=address,undefined
    (the device translation units are the product's own objects, build/moa/*.cu.o)."""
    build_moa(force)
    nccl = _nccl_root()
    san = ["-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer", "-g", "-O1"]
    src = os.path.join(ROOT, "oracle", "moa_oracle.c")
    out_o = os.path.join(ROOT, "oracle", "liboracle_asan.so")
    if force or _stale(out_o, [src]):
        _run(["gcc", *san, "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared", "-pthread", src, "-o",
              out_o, "-lm"])
    csrc = os.path.join(ROOT, "paper_2306_11148_b200", "csrc")
    objdir = os.path.join(ROOT, "build", "asan")
    os.makedirs(objdir, exist_ok=True)
    host = [os.path.join(csrc, "moa_host.cpp"), os.path.join(csrc, "moa_tma.cpp")]
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))
    out = os.path.join(objdir, "libmoa_asan.so")
    dev_objs = sorted(glob.glob(os.path.join(ROOT, "build", "moa", "*.cu.o")))
    if force or _stale(out, host + hdrs + dev_objs):
        objs = []
        for s in host:
            o = os.path.join(objdir, os.path.basename(s) + ".o")
            _run(["g++", *san, "-std=c++17", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", csrc, "-I",
                  os.path.join(nccl, "include"), "-I", "/usr/local/cuda/include", "-c", s, "-o", o])
            objs.append(o)
        _run(["g++", *san, "-shared", *objs, *dev_objs, "-o", out, "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
              "-Wl,-rpath=" + os.path.join(nccl, "lib"), "-L/usr/local/cuda/lib64", "-lcudart",
              "-Wl,-rpath=/usr/local/cuda/lib64"])
    return out


TARGETS = {"oracle": build_oracle, "inputs": build_inputs, "inputs_cuda": build_inputs_cuda, "moa": build_moa,
           "shim": build_shim, "asan": build_asan}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("targets", nargs="*", default=["all"])
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    a = ap.parse_args(argv)
    names = [t for t in TARGETS if t != "asan"] if "all" in a.targets else a.targets
    for n in names:
        print(f"[build] {n}", flush=True)
        if n == "moa":
            build_moa(a.force, a.ptxas_v)
        else:
            TARGETS[n](a.force)


if __name__ == "__main__":
    sys.exit(main())
