"""Build the in-tree sm_100a extension (libdses_b200.so).

    python -m paper_2502_00115_b200.build

nvcc cross-compiles for sm_100a without a GPU.  The .so lands in
paper_2502_00115_b200/_lib/ (git-ignored, shipped to the GPU box by gpurun).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libdses_b200.so")
SOURCES = ["dses_vote.cu", "dses_score.cu", "dses_sparse.cu", "dses_capi.cu", "dses_probe.cu",
           "dses_sweep.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def nvcc_version(exe: str) -> str:
    out = subprocess.run([exe, "--version"], capture_output=True, text=True).stdout
    for tok in out.replace(",", " ").split():
        if tok.startswith("V") and tok[1:2].isdigit():
            return tok[1:]
    return "unknown"


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "dses_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), out: str = OUT) -> str:
    """defines: extra -D flags (kernel variants for A/B timing, tools/gpu_ab.sh)."""
    if not force and not needs_build():
        return OUT
    exe = nvcc()
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [exe, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-Wall,-Wextra,-Winfinite-recursion", "-shared",
           f'-DDSES_NVCC_VERSION="{nvcc_version(exe)}"', *[f"-D{d}" for d in defines],
           "-o", out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    # python -m paper_2502_00115_b200.build [--force] [-v] [-DNAME=V ... -o OUT.so]
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    dest = args[args.index("-o") + 1] if "-o" in args else OUT
    print(build(force="--force" in args or bool(defs) or dest != OUT, verbose="-v" in args,
                defines=defs, out=dest))
