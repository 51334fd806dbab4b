"""Build libfgs.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo).

    python -m paper_2409_04751_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libfgs.so")
OBJ = os.path.join(HERE, "_obj")
ROOT = os.path.dirname(HERE)
EXAMPLE_SRC = os.path.join(ROOT, "tools", "fgs_render_example.cpp")
EXAMPLE_BIN = os.path.join(ROOT, "tools", "fgs_render_example")
CLI_SRC = os.path.join(ROOT, "tools", "fgs_cli.cpp")
CLI_BIN = os.path.join(ROOT, "tools", "fgs_cli")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]
# Per-file flags: preprocess.cu keeps the reference's fp32 op order exactly (no FMA contraction).
SOURCES = {
    "preprocess.cu": ["--fmad=false"],
    "binning.cu": [],
    "raster.cu": [],
    "train.cu": [],
    "bruteforce.cu": [],
    "fgs_api.cu": [],
    "comm.cu": [],
}


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def _programs_stale() -> bool:
    inputs = [CLI_SRC, EXAMPLE_SRC, OUT] + [os.path.join(ROOT, "include", h) for h in
                                            ("fgs.h", "fgs.hpp", "fgs_io.hpp", "fgs_omnisplat.hpp")]
    newest = max(os.path.getmtime(p) for p in inputs if os.path.exists(p))
    outs = [CLI_BIN, EXAMPLE_BIN]
    if os.path.exists(os.path.join(REF_INC, "omnisplat", "splatting.hpp")):
        outs += [o for _, o, _ in OMNI_PROGRAMS]
        newest = max([newest] + [os.path.getmtime(s) for s, _, _ in OMNI_PROGRAMS])
    return any(not os.path.exists(o) or os.path.getmtime(o) < newest for o in outs)


def build(verbose=False, force=False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "fgs.h")]
    if not force and os.path.exists(OUT) and _programs_stale():
        build_example(verbose)
    newest = max(os.path.getmtime(p) for p in deps)
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    nvcc = _nvcc()
    objs = []
    for src, extra in SOURCES.items():
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(obj)
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", OUT, *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    build_example(verbose)
    return OUT


REF_INC = "/root/reference/proj/include"
SHIM = os.path.join(ROOT, "oracle", "eigen_shim")
# Programs written against the reference's own types (omnisplat::Scene / Camera / RenderResult)
# through include/fgs_omnisplat.hpp: compiled only where the reference headers are mounted (this
# container), against the repo's Eigen-subset shim; the binaries travel to the GPU box.
OMNI_PROGRAMS = [(os.path.join(ROOT, "tools", "omnisplat_bench.cpp"), os.path.join(ROOT, "tools", "omnisplat_bench"),
                  "$ORIGIN/../paper_2409_04751_b200"),
                 (os.path.join(ROOT, "tests", "cpp", "omni_dropin_check.cpp"),
                  os.path.join(ROOT, "tests", "cpp", "omni_dropin_check"), "$ORIGIN/../../paper_2409_04751_b200")]


def build_example(verbose=False):
    """C++ host programs over include/fgs.hpp / fgs_io.hpp (the render example and the
    reference-compatible CLI), linked against libfgs.so (rpath $ORIGIN/..); and, with the
    reference headers mounted, the omnisplat-typed drop-in programs."""
    for src, out in ((EXAMPLE_SRC, EXAMPLE_BIN), (CLI_SRC, CLI_BIN)):
        if not os.path.exists(src):
            continue
        cmd = ["g++", "-O2", "-std=c++17", "-o", out, src, "-L" + HERE, "-lfgs",
               "-Wl,-rpath,$ORIGIN/../paper_2409_04751_b200"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    if os.path.exists(os.path.join(REF_INC, "omnisplat", "splatting.hpp")):
        for src, out, rpath in OMNI_PROGRAMS:
            cmd = ["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-isystem", SHIM, "-I" + REF_INC, "-o", out, src,
                   "-L" + HERE, "-lfgs", "-Wl,-rpath," + rpath, "-lpthread"]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
