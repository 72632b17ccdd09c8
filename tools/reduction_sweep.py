"""NEXT #4: node-reduction sweep on B200 (Fig. 9 analogue, lines 190-201).

  build (here, no GPU):  python tools/reduction_sweep.py build   (build() compiles the libraries; this adds SASS sizes)
  run (GPU box):         python tools/reduction_sweep.py run [n]   -> gpurun_out/reduction_sweep_n{n}.json

Generates the fixed-spin CDAG of e- gamma^n -> e- gamma at several partial node-reduction states
(reductions applied one at a time in random order), emits one statement per node (gen/sweep.py),
compiles twice -- full optimisation (instruction-level CSE across nodes), and with volatile momentum
loads so that identical node computations cannot be merged by the compiler -- and
measures time per point against the FLOP prediction.  Parity of every state against the oracle.
"""
import ctypes
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GEN = os.path.join(ROOT, "paper_2511_19456_b200", "csrc", "generated")
LIB = os.path.join(ROOT, "paper_2511_19456_b200", "lib")


def build(n):
    """Compile (paper_2511_19456_b200.build, which also emits the states; n = 4 only) and record the
    SASS instruction count of every state's kernel in each build."""
    assert n == 4, "the sweep libraries are built for the paper's n = 4 process"
    from paper_2511_19456_b200 import build as b
    b.build()
    mpath = os.path.join(LIB, f"sweep_n{n}_meta.json")
    meta = json.load(open(mpath))
    for tag in ("cse", "nocse"):
        out = os.path.join(LIB, f"libqed_sweep_n{n}_{tag}.so")
        sass = subprocess.run(["cuobjdump", "-sass", out], capture_output=True, text=True).stdout
        counts, cur = {}, None
        for line in sass.splitlines():
            if "Function :" in line:
                cur = line.split("Function :")[1].strip()
                counts[cur] = 0
            elif cur and "/*" in line and ";" in line:
                counts[cur] += 1
        for m in meta:
            m[f"sass_{tag}"] = next((v for k_, v in counts.items() if f"k_state{m['state']}E" in k_), None)
    json.dump(meta, open(mpath, "w"), indent=1)
    print(json.dumps(meta, indent=1))


def run(n):
    import numpy as np
    import torch

    import oracle
    import synthetic
    meta = json.load(open(os.path.join(LIB, f"sweep_n{n}_meta.json")))
    P = 1 << 20
    mom = synthetic.rambo_cm(n, P, sqrt_s=5.0, seed=41 + n, device="cuda")
    rev = torch.cat([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], dim=1)   # e- gamma^n -> e- gamma
    soa = synthetic.to_soa(rev)
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    N = n + 1
    norm = (4 * math.pi / 137.035999084) ** N
    ref = oracle.msq(n, 1, rev[:64].cpu().numpy(), spec=[0] * (n + 3))
    res = {"process": f"e- gamma^{n} -> e- gamma, fixed spins/polarisations", "points": P, "states": []}
    for tag in ("cse", "nocse"):
        lib = ctypes.CDLL(os.path.join(LIB, f"libqed_sweep_n{n}_{tag}.so"))
        lib.sweep_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_double,
                                  ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
        for m in meta:
            ms = ctypes.c_float()
            rc = lib.sweep_run(m["state"], soa.data_ptr(), P, out.data_ptr(), norm, 10, ctypes.byref(ms))
            torch.cuda.synchronize()
            got = out[:64].cpu().numpy()
            err = float(np.max(np.abs(got / ref - 1)))
            res["states"].append(dict(m, build=tag, rc=rc, ms=ms.value, max_rel_err_vs_oracle=err))
    base = {t: next(s for s in res["states"] if s["build"] == t and s["state"] == 0) for t in ("cse", "nocse")}
    for s in res["states"]:
        s["speedup_measured"] = base[s["build"]]["ms"] / s["ms"]
        s["speedup_predicted_flops"] = base[s["build"]]["predicted_flops"] / s["predicted_flops"]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", f"reduction_sweep_n{n}.json"), "w"), indent=1)
    for s in res["states"]:
        print(f"{s['build']} red={s['reductions']:4d} nodes={s['nodes']:5d} flops={s['predicted_flops']:7d} "
              f"sass={s.get('sass_' + s['build'])} ms={s['ms']:.3f} speedup={s['speedup_measured']:.2f} "
              f"pred={s['speedup_predicted_flops']:.2f} err={s['max_rel_err_vs_oracle']:.1e}")


if __name__ == "__main__":
    mode = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    build(n) if mode == "build" else run(n)
