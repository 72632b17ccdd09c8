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
        [os.path.join(ROOT, "include", "qed.h"), os.path.join(ROOT, "include", "abc.h")]


def _compile(src: str, force: bool, extra=(), tag: str = "", log: bool = True) -> str:
    obj = os.path.join(OBJ_DIR, os.path.basename(src).replace(".cu", tag + ".o"))
    deps = [src] + _headers()
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc()] + NVCC_FLAGS + list(extra) + ["-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        logf = os.path.join(LIB_DIR, "ptxas_" + os.path.basename(src).replace(".cu", ".log"))
        with open(logf, "w") as f:   # (compile-time lines dropped: the tracked logs change only with the code)
            text = r.stdout + r.stderr
            f.write(" ".join(cmd) + "\n" + "".join(ln for ln in text.splitlines(True) if "Compile time" not in ln))
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    os.replace(obj + ".tmp", obj)
    return obj


SWEEP_N = 4                                   # the paper's Fig. 9 process, e- gamma^4 -> e- gamma
SWEEP_CHECK = [0.0, 0.125, 0.25, 0.5, 0.75, 1.0]   # fractions of the node reductions at which states are emitted
SWEEP_BUILDS = {"cse": [], "nocse": ["-DSWEEP_NOCSE"]}


def sweep_sources() -> tuple[list[str], str]:
    """Node-reduction sweep (§3.4 Fig. 9): one translation unit per
    partially reduced CDAG state of e- gamma^4 -> e- gamma (gen/sweep.py) and a timing entry point.
    Experiment libraries, not the product ABI: tests/test_reduction_sweep.py and tools/reduction_sweep.py
    load them.  Returns (sources, metadata json path)."""
    import json
    from paper_2511_19456_b200.gen.dag import paper_process
    from paper_2511_19456_b200.gen.sweep import emit_sweep_files, reduction_states
    proc = paper_process(SWEEP_N)
    files, meta = emit_sweep_files(proc, reduction_states(proc, SWEEP_CHECK, seed=1), f"qed_sweep_n{SWEEP_N}")
    out = []
    for name, src in files.items():
        path = os.path.join(GEN_DIR, name)
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        out.append(path)
    mpath = os.path.join(LIB_DIR, f"sweep_n{SWEEP_N}_meta.json")
    old = json.load(open(mpath)) if os.path.exists(mpath) else []
    keep = {m["state"]: m for m in old if "sass_cse" in m}
    for m in meta:   # SASS sizes (tools/reduction_sweep.py) survive a rebuild of identical states
        k = keep.get(m["state"])
        if k and k["nodes"] == m["nodes"] and k["predicted_flops"] == m["predicted_flops"]:
            m.update({x: k[x] for x in k if x.startswith("sass_")})
    with open(mpath, "w") as f:
        json.dump(meta, f, indent=1)
    return out, mpath


def build(force: bool = False, jobs: int | None = None) -> str:
    sys.path.insert(0, ROOT) if ROOT not in sys.path else None
    from paper_2511_19456_b200.gen.abc import generate_abc
    from paper_2511_19456_b200.gen.emit import generate_all
    from paper_2511_19456_b200.gen.emit_bg import generate_bg
    from paper_2511_19456_b200.gen.emit_regs import generate_regs

    os.makedirs(OBJ_DIR, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    sources = generate_all(GEN_DIR) + generate_regs(GEN_DIR) + generate_bg(GEN_DIR) + generate_abc(GEN_DIR) + \
        [os.path.join(CSRC, "qed_runtime.cu"), os.path.join(CSRC, "abc_runtime.cu")]
    sweep_src, _ = sweep_sources()
    units = [(s, (), "", True) for s in sources] + \
        [(s, fl, "_" + tag, False) for tag, fl in SWEEP_BUILDS.items() for s in sweep_src]
    jobs = jobs or min(len(units), max(1, os.cpu_count() or 1))
    # largest translation unit first
    units.sort(key=lambda u: -os.path.getsize(u[0]))
    with cf.ThreadPoolExecutor(jobs) as ex:
        done = dict(zip([u[0] + u[2] for u in units], ex.map(lambda u: _compile(u[0], force, u[1], u[2], u[3]), units)))
    objs = [done[s] for s in sources]
    for tag in SWEEP_BUILDS:
        sobjs = [done[s + "_" + tag] for s in sweep_src]
        slib = os.path.join(LIB_DIR, f"libqed_sweep_n{SWEEP_N}_{tag}.so")
        if force or not os.path.exists(slib) or os.path.getmtime(slib) < max(os.path.getmtime(o) for o in sobjs):
            subprocess.run([nvcc()] + ARCH + ["-shared", "-o", slib + ".tmp"] + sobjs + ["-lcudart"], check=True)
            os.replace(slib + ".tmp", slib)
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
