"""Parity oracle for tree-level n-photon Compton |M|^2 (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(paper_2511_19456_b200) never imports it, and it shares no code with it.

The arithmetic lives in ``qed_oracle.c`` (plain C, dense 4x4 Dirac algebra,
explicit enumeration of every Feynman diagram; see its header for the
PAPER.md citations).  This module only compiles it and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qed_oracle.c")
_LIBS = {
    "f64": os.path.join(_HERE, "liboracle_f64.so"),
    "f80": os.path.join(_HERE, "liboracle_f80.so"),
}
_DEFS = {"f64": "double", "f80": "long double"}
_ABC_SRC = os.path.join(_HERE, "abc_oracle.c")
_ABC_LIB = os.path.join(_HERE, "liboracle_abc.so")
_loaded: dict[str, ctypes.CDLL] = {}


def build(force: bool = False) -> None:
    """Compile the oracles (QED in double and long double, ABC model in double) with gcc."""
    jobs = [(path, _SRC, [f"-DORACLE_REAL={_DEFS[kind]}"]) for kind, path in _LIBS.items()]
    jobs.append((_ABC_LIB, _ABC_SRC, []))
    for path, src, defs in jobs:
        if not force and os.path.exists(path) and os.path.getmtime(path) >= os.path.getmtime(src):
            continue
        tmp = path + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=gnu11", "-shared", "-fPIC"] + defs + ["-o", tmp, src, "-lm", "-lpthread"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, path)


def _lib(kind: str = "f64") -> ctypes.CDLL:
    if kind not in _loaded:
        build()
        lib = ctypes.CDLL(_LIBS[kind])
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_msq.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_long,
                                   ctypes.POINTER(ctypes.c_int8), dp, ctypes.c_int]
        lib.oracle_msq.restype = ctypes.c_int
        lib.oracle_amps.argtypes = [ctypes.c_int, ctypes.c_int, dp, ctypes.c_long, dp, ctypes.c_int]
        lib.oracle_amps.restype = ctypes.c_int
        lib.oracle_diagram_sum_explicit.argtypes = [ctypes.c_int, dp, dp, dp, dp, dp, dp]
        lib.oracle_diagram_sum_explicit.restype = ctypes.c_long
        for f in ("oracle_spinor_u", "oracle_spinor_ubar", "oracle_polvec"):
            getattr(lib, f).argtypes = [dp, ctypes.c_int, dp]
            getattr(lib, f).restype = None
        lib.oracle_gammas.argtypes = [dp]
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
        lib.oracle_rambo_point.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, dp]
        lib.oracle_rambo_point.restype = ctypes.c_double
        lib.oracle_mc_sum.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, dp, ctypes.c_int]
        lib.oracle_mc_sum.restype = ctypes.c_int
        lib.oracle_coupling_e.restype = ctypes.c_double
        lib.oracle_real_bytes.restype = ctypes.c_int
        _loaded[kind] = lib
    return _loaded[kind]


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def msq(n_in_ph: int, n_out_ph: int, mom: np.ndarray, spec=None, threads: int | None = None,
        kind: str = "f64") -> np.ndarray:
    """|M|^2 per point.  mom: [n_points, n_ext, 4] float64, particle order
    e-_in, gamma_in..., e-_out, gamma_out...  spec: per-particle -1 (summed;
    averaged if initial) or fixed state 0/1; None = all summed."""
    mom = np.ascontiguousarray(mom, dtype=np.float64)
    n_ext = n_in_ph + n_out_ph + 2
    assert mom.ndim == 3 and mom.shape[1:] == (n_ext, 4), mom.shape
    out = np.empty(mom.shape[0], dtype=np.float64)
    sp = None
    if spec is not None:
        spa = np.asarray(spec, dtype=np.int8)
        assert spa.shape == (n_ext,)
        sp = spa.ctypes.data_as(ctypes.POINTER(ctypes.c_int8))
    rc = _lib(kind).oracle_msq(n_in_ph, n_out_ph, _dp(mom), mom.shape[0], sp, _dp(out),
                               threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_msq: bad arguments")
    return out


def amps(n_in_ph: int, n_out_ph: int, mom: np.ndarray, threads: int | None = None,
         kind: str = "f64") -> np.ndarray:
    """All 2^(n_ext) helicity amplitudes (including e^N) per point:
    complex [n_points, H]; bit j of h = state of external particle j."""
    mom = np.ascontiguousarray(mom, dtype=np.float64)
    n_ext = n_in_ph + n_out_ph + 2
    H = 1 << n_ext
    out = np.empty((mom.shape[0], H, 2), dtype=np.float64)
    rc = _lib(kind).oracle_amps(n_in_ph, n_out_ph, _dp(mom), mom.shape[0], _dp(out),
                                threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_amps: bad arguments")
    return out[..., 0] + 1j * out[..., 1]


def diagram_sum_explicit(q: np.ndarray, p: np.ndarray, u: np.ndarray, ubar: np.ndarray,
                         eps: np.ndarray, kind: str = "f64"):
    """Sum over all N! orderings for explicit wave functions (no coupling).
    q: [N,4] signed photon momenta; eps: complex [N,4]; u, ubar: complex [4].
    Returns (amplitude, number_of_diagrams)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    N = q.shape[0]
    p = np.ascontiguousarray(p, dtype=np.float64)
    uu = np.ascontiguousarray(np.stack([np.real(u), np.imag(u)], -1), dtype=np.float64)
    ub = np.ascontiguousarray(np.stack([np.real(ubar), np.imag(ubar)], -1), dtype=np.float64)
    ee = np.ascontiguousarray(np.stack([np.real(eps), np.imag(eps)], -1), dtype=np.float64)
    out = np.empty(2, dtype=np.float64)
    nd = _lib(kind).oracle_diagram_sum_explicit(N, _dp(q), _dp(p), _dp(uu), _dp(ub), _dp(ee), _dp(out))
    if nd < 0:
        raise ValueError("bad N")
    return complex(out[0], out[1]), int(nd)


def spinor_u(p, s, kind="f64"):
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.empty(8)
    _lib(kind).oracle_spinor_u(_dp(p), int(s), _dp(out))
    return out[0::2] + 1j * out[1::2]


def spinor_ubar(p, s, kind="f64"):
    p = np.ascontiguousarray(p, dtype=np.float64)
    out = np.empty(8)
    _lib(kind).oracle_spinor_ubar(_dp(p), int(s), _dp(out))
    return out[0::2] + 1j * out[1::2]


def polvec(k, lam, kind="f64"):
    k = np.ascontiguousarray(k, dtype=np.float64)
    out = np.empty(4)
    _lib(kind).oracle_polvec(_dp(k), int(lam), _dp(out))
    return out


def gammas(kind="f64"):
    out = np.empty(128)
    _lib(kind).oracle_gammas(_dp(out))
    c = out[0::2] + 1j * out[1::2]
    return c.reshape(4, 4, 4)


def coupling_e(kind="f64") -> float:
    return _lib(kind).oracle_coupling_e()


def philox4x32_10(ctr, key, kind="f64"):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    _lib(kind).oracle_philox4x32_10(c, k, o)
    return list(o)


def rambo_point(n_out_ph: int, sqrt_s: float, seed: int, index: int, kind="f64"):
    """(momenta [n+3, 4], weight) of point `index` of the MC sequence keyed by `seed`."""
    mom = np.empty((n_out_ph + 3) * 4)
    w = _lib(kind).oracle_rambo_point(n_out_ph, sqrt_s, seed, index, _dp(mom))
    return mom.reshape(n_out_ph + 3, 4), w


def mc_sum(n_out_ph: int, sqrt_s: float, omega_min: float, seed: int, first: int, count: int,
           chunk: int = 1024, threads: int | None = None, kind="f64") -> np.ndarray:
    """Chunk partial sums [n_chunks, 3] = (sum w|M|^2, sum (w|M|^2)^2, n_pass), n_chunks =
    ceil((first + count) / chunk) (chunks before `first` stay zero)."""
    n_chunks = (first + count + chunk - 1) // chunk
    out = np.zeros(3 * n_chunks)
    rc = _lib(kind).oracle_mc_sum(n_out_ph, sqrt_s, omega_min, seed, first, count, chunk, _dp(out),
                                  threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_mc_sum: bad arguments")
    return out.reshape(n_chunks, 3)


# ---------------------------------------------------------------- ABC model (abc_oracle.c)

def _abc():
    if "abc" not in _loaded:
        build()
        lib = ctypes.CDLL(_ABC_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.oracle_abc_msq.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       dp, ctypes.c_long, dp, ctypes.c_int]
        lib.oracle_abc_msq.restype = ctypes.c_int
        lib.oracle_abc_diagram_sum.argtypes = [ctypes.c_int, dp, dp, ctypes.c_double, ctypes.c_double, dp]
        lib.oracle_abc_diagram_sum.restype = ctypes.c_long
        _loaded["abc"] = lib
    return _loaded["abc"]


def abc_msq(n_in: int, n_out: int, mom: np.ndarray, m_a: float, m_c: float, g: float = 1.0,
            threads: int | None = None) -> np.ndarray:
    """|M|^2 per point of A + n_in B -> A + n_out B.  mom: [n_points, n_in + n_out + 2, 4], particle
    order A_in, B_in..., A_out, B_out...; the B mass enters only through the (on-shell) momenta."""
    mom = np.ascontiguousarray(mom, dtype=np.float64)
    assert mom.ndim == 3 and mom.shape[1:] == (n_in + n_out + 2, 4), mom.shape
    out = np.empty(mom.shape[0], dtype=np.float64)
    rc = _abc().oracle_abc_msq(n_in, n_out, m_a, m_c, g, _dp(mom), mom.shape[0], _dp(out),
                               threads or default_threads())
    if rc != 0:
        raise ValueError("oracle_abc_msq: bad arguments (the number of B-ons must be even)")
    return out


def abc_diagram_sum(q: np.ndarray, p_a: np.ndarray, m_a: float, m_c: float):
    """(sum over orderings of prod 1/(Q_l^2 - m_{X_l}^2), number of diagrams) for signed B momenta q [N, 4]."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    p_a = np.ascontiguousarray(p_a, dtype=np.float64)
    out = np.empty(1)
    nd = _abc().oracle_abc_diagram_sum(q.shape[0], _dp(q), _dp(p_a), m_a, m_c, _dp(out))
    if nd < 0:
        raise ValueError("bad N")
    return float(out[0]), int(nd)
