"""Build libfgs.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo).

    python -m paper_2409_04751_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

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


CHECKED_OUT = os.path.join(HERE, "libfgs_checked.so")


def _build_lib(out, objdir, defines, deps, verbose, force):
    """nvcc every source (in parallel) and link one shared library; skipped when up to date."""
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in deps):
        return False
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    cmds, objs = [], []
    for src, extra in SOURCES.items():
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmds.append([nvcc, *ARCH, *COMMON, *defines, *extra, "-c", os.path.join(CSRC, src), "-o", obj])
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for cmd in cmds:
            if verbose:
                print(" ".join(cmd))
        for r in ex.map(lambda c: subprocess.run(c, check=True), cmds):
            pass
    cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return True


def build(verbose=False, force=False, checked=True) -> str:
    """libfgs.so (the product) and libfgs_checked.so (the same sources with -DFGS_CHECKED: device
    bounds / invariant checks that trap, for tests/test_checked_gpu.py)."""
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "fgs.h")]
    if not force and os.path.exists(OUT) and _programs_stale():
        build_example(verbose)
    built = _build_lib(OUT, OBJ, [], deps, verbose, force)
    if checked:
        _build_lib(CHECKED_OUT, OBJ + "_checked", ["-DFGS_CHECKED"], deps, verbose, force)
    if built:
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


def build_variant(name: str, defines, verbose=False) -> str:
    """Experiment builds: libfgs_<name>.so from the same sources with extra -D defines, loaded with
    FGS_LIB=<name> (A/B timing of a code path on one GPU run; profiles/variants.sh)."""
    out = os.path.join(HERE, f"libfgs_{name}.so")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    _build_lib(out, OBJ + "_" + name, [d if d.startswith("-") else "-D" + d for d in defines], deps, verbose, False)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        print(build_variant(sys.argv[2], sys.argv[3:], verbose=True))
    else:
        print(build(verbose=True, force="--force" in sys.argv))
