"""Build libmgk.so (all CUDA sources, sm_100a) in-tree with nvcc.

    python -m paper_1910_06310_b200.build

The shared object lands next to this file so it travels with the repo
snapshot to the GPU box; nothing is installed into site-packages.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libmgk.so"
SOURCES = ["capi.cu", "tiles.cu", "pcg_warp.cu", "pcg_panel.cu", "pcg_block.cu", "pbr.cu", "bench_support.cu",
           "gram_post.cu", "ingest.cu", "order.cu"]
# sources compiled more than once: (source, object stem, extra flags)
VARIANTS = {"pcg_panel.cu": [("pcg_panel_256", ["-DMGK_PANEL_THREADS=256", "-DMGK_PANEL_NS=p256"]),
                             ("pcg_panel_512", ["-DMGK_PANEL_THREADS=512", "-DMGK_PANEL_NS=p512"])]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or "/usr/local/cuda/bin/nvcc"
    return cand if Path(cand).exists() else "nvcc"


def build(verbose: bool = False, force: bool = False) -> Path:
    srcs = [CSRC / s for s in SOURCES]
    deps = srcs + list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "mgk.h"]
    if LIB.exists() and not force and all(LIB.stat().st_mtime >= d.stat().st_mtime for d in deps):
        return LIB
    objdir = HERE / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-I", str(CSRC), "-I", str(HERE.parent / "include")]
    if verbose:
        common += ["-Xptxas", "-v"]
    procs = []
    for s in srcs:
        for stem, extra in VARIANTS.get(s.name, [(s.stem, [])]):
            o = objdir / (stem + ".o")
            objs.append(o)
            procs.append((s, subprocess.Popen(common + extra + ["-c", str(s), "-o", str(o)], stdout=subprocess.PIPE,
                                              stderr=subprocess.STDOUT, text=True)))
    for s, p in procs:
        out, _ = p.communicate()
        if verbose or p.returncode:
            sys.stderr.write(out)
        if p.returncode:
            raise RuntimeError(f"nvcc failed on {s.name}")
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
