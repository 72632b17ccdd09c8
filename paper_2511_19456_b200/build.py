"""Build libqed.so in-tree for sm_100a: run the generator, nvcc every translation unit, link.

    python -m paper_2511_19456_b200.build [--force] [--jobs N]

Output: paper_2511_19456_b200/lib/libqed.so (+ lib/ptxas_*.log with register/spill
reports).  Only nvcc and a host compiler are needed; no GPU.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
GEN_DIR = os.path.join(CSRC, "generated")
LIB_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(LIB_DIR, "libqed.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                     "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _headers() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
        [os.path.join(ROOT, "include", "qed.h")]


def _compile(src: str, force: bool) -> str:
    obj = os.path.join(OBJ_DIR, os.path.basename(src).replace(".cu", ".o"))
    deps = [src] + _headers()
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    log = os.path.join(LIB_DIR, "ptxas_" + os.path.basename(src).replace(".cu", ".log"))
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:   # (compile-time lines dropped: the tracked logs change only with the code)
        text = r.stdout + r.stderr
        f.write(" ".join(cmd) + "\n" + "".join(ln for ln in text.splitlines(True) if "Compile time" not in ln))
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, jobs: int | None = None) -> str:
    sys.path.insert(0, ROOT) if ROOT not in sys.path else None
    from paper_2511_19456_b200.gen.emit import generate_all
    from paper_2511_19456_b200.gen.emit_bg import generate_bg
    from paper_2511_19456_b200.gen.emit_regs import generate_regs

    os.makedirs(OBJ_DIR, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    sources = generate_all(GEN_DIR) + generate_regs(GEN_DIR) + generate_bg(GEN_DIR) + \
        [os.path.join(CSRC, "qed_runtime.cu")]
    jobs = jobs or min(len(sources), max(1, os.cpu_count() or 1))
    # largest translation unit first
    sources.sort(key=lambda s: -os.path.getsize(s))
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), sources))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    # FP64 peak microbenchmark (bench.py / profiles only; not part of the C ABI)
    peak_src = os.path.join(CSRC, "tools", "dfma_peak.cu")
    peak_lib = os.path.join(LIB_DIR, "libqed_peak.so")
    if force or not os.path.exists(peak_lib) or os.path.getmtime(peak_lib) < os.path.getmtime(peak_src):
        subprocess.run([nvcc()] + ARCH + ["-O3", "-shared", "-Xcompiler", "-fPIC", "-o", peak_lib + ".tmp", peak_src],
                       check=True)
        os.replace(peak_lib + ".tmp", peak_lib)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int)
    a = ap.parse_args()
    print(build(a.force, a.jobs))
