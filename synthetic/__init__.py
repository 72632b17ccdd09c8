"""Seeded synthetic phase-space inputs shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no spinors, propagators,
diagrams or |M|^2).  It only produces on-shell, momentum-conserving external
momenta with the distributions of the north-star workloads
(SURVEY.md §8(d) "Concrete synthetic inputs"):

* ``compton_lab``   -- n = 1, lab frame (electron at rest), omega log-uniform
  in [1e-2, 1e2] m_e, cos(theta) ~ U[-1, 1], phi ~ U[0, 2pi), outgoing photon
  from the Compton relation.  Used for the Klein-Nishina checks (config C1).
* ``rambo_cm``      -- e- gamma -> e- + n gamma in the CM frame at sqrt(s)
  (incoming photon along +z, electron along -z), final state from massive
  RAMBO (Kleiss, Stirling, Ellis, CPC 40 (1986) 359): n+1 isotropic massless
  momenta, boosted and scaled to (sqrt s, 0), then rescaled to the masses
  (1 massive electron + n photons) by Newton iteration on xi.  Configs C2-C5.

Momenta are float64 in units of m_e.  Layout helpers convert between the
point-major AoS array [n_points, n_ext, 4] (oracle side) and the SoA layout
``mom[(4*j + mu) * n_points + i]`` that the C-ABI takes.  Particle order:
e-_in, gamma_in..., e-_out, gamma_out...

Generation uses torch so that the large bench batches (2^22-2^26 points) can
be produced directly in device memory; the parity tests generate on the CPU
and copy the same array to both sides.
"""
from __future__ import annotations

import math

import torch


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def compton_lab(n_points: int, seed: int = 1, omega_range=(1e-2, 1e2), device="cpu") -> torch.Tensor:
    """[n_points, 4, 4] lab-frame Compton kinematics (order e_in, g_in, e_out, g_out)."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    f64 = torch.float64
    r = torch.rand((3, n_points), generator=g, device=dev, dtype=f64)
    lo, hi = math.log(omega_range[0]), math.log(omega_range[1])
    w = torch.exp(lo + (hi - lo) * r[0])
    c = 2 * r[1] - 1
    phi = 2 * math.pi * r[2]
    s = torch.sqrt(torch.clamp(1 - c * c, min=0))
    wp = w / (1 + w * (1 - c))
    mom = torch.zeros((n_points, 4, 4), dtype=f64, device=dev)
    mom[:, 0, 0] = 1.0
    mom[:, 1, 0] = w
    mom[:, 1, 3] = w
    kp = torch.stack([wp, wp * s * torch.cos(phi), wp * s * torch.sin(phi), wp * c], -1)
    mom[:, 3] = kp
    mom[:, 2] = mom[:, 0] + mom[:, 1] - kp
    return mom


def _rambo_massive(n_final: int, masses, sqrt_s: float, n_points: int, g, dev) -> torch.Tensor:
    f64 = torch.float64
    r = torch.rand((4, n_final, n_points), generator=g, device=dev, dtype=f64)
    c = 2 * r[0] - 1
    phi = 2 * math.pi * r[1]
    q0 = -torch.log(r[2] * r[3])
    st = torch.sqrt(torch.clamp(1 - c * c, min=0))
    q = torch.stack([q0, q0 * st * torch.cos(phi), q0 * st * torch.sin(phi), q0 * c], -1)  # [K, n, 4]
    Q = q.sum(0)
    M = torch.sqrt(Q[:, 0] ** 2 - (Q[:, 1:] ** 2).sum(-1))
    b = -Q[:, 1:] / M[:, None]
    x = sqrt_s / M
    gam = Q[:, 0] / M
    a = 1 / (1 + gam)
    bq = (b[None] * q[..., 1:]).sum(-1)  # [K, n]
    p0 = x * (gam * q[..., 0] + bq)
    pv = x[..., None] * (q[..., 1:] + b[None] * q[..., :1] + (a * bq)[..., None] * b[None])
    m = torch.tensor(masses, dtype=f64, device=dev)[:, None]
    xi = torch.full((n_points,), math.sqrt(max(0.0, 1 - (float(sum(masses)) / sqrt_s) ** 2)), dtype=f64,
                    device=dev)
    for _ in range(30):
        e = torch.sqrt(m * m + (xi * p0) ** 2)
        f = e.sum(0) - sqrt_s
        df = (xi * p0 * p0 / e).sum(0)
        xi = xi - f / df
    e = torch.sqrt(m * m + (xi * p0) ** 2)
    return torch.cat([e[..., None], xi[None, :, None] * pv], -1)  # [K, n, 4]


def rambo_cm(n_out_photons: int, n_points: int, sqrt_s: float = 5.0, seed: int = 2, device="cpu") -> torch.Tensor:
    """[n_points, n+3, 4] for e- gamma -> e- + n gamma at CM energy sqrt_s."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    f64 = torch.float64
    s = sqrt_s * sqrt_s
    kin = (s - 1.0) / (2 * sqrt_s)
    ein = (s + 1.0) / (2 * sqrt_s)
    n = n_out_photons
    mom = torch.empty((n_points, n + 3, 4), dtype=f64, device=dev)
    mom[:, 0] = torch.tensor([ein, 0.0, 0.0, -kin], dtype=f64, device=dev)
    mom[:, 1] = torch.tensor([kin, 0.0, 0.0, kin], dtype=f64, device=dev)
    fin = _rambo_massive(n + 1, [1.0] + [0.0] * n, sqrt_s, n_points, g, dev)
    mom[:, 2:] = fin.permute(1, 0, 2)
    return mom


# ABC model (App. F): masses of the A-, B- and C-on in units of m_A (reading A2)
ABC_MASSES = (1.0, 0.5, 1.2)


def abc_cm(n_out_b: int, n_points: int, sqrt_s: float = 5.0, seed: int = 2, masses=ABC_MASSES,
           device="cpu") -> torch.Tensor:
    """[n_points, n+3, 4] for A B -> A + n B in the CM frame at sqrt_s (incoming B along +z, A along -z),
    final state from massive RAMBO with masses (m_A, m_B x n)."""
    dev = torch.device(device)
    g = _gen(seed, dev)
    f64 = torch.float64
    mA, mB, _ = masses
    s = sqrt_s * sqrt_s
    kin = math.sqrt((s - (mA + mB) ** 2) * (s - (mA - mB) ** 2)) / (2 * sqrt_s)
    n = n_out_b
    mom = torch.empty((n_points, n + 3, 4), dtype=f64, device=dev)
    mom[:, 0] = torch.tensor([math.sqrt(mA * mA + kin * kin), 0.0, 0.0, -kin], dtype=f64, device=dev)
    mom[:, 1] = torch.tensor([math.sqrt(mB * mB + kin * kin), 0.0, 0.0, kin], dtype=f64, device=dev)
    fin = _rambo_massive(n + 1, [mA] + [mB] * n, sqrt_s, n_points, g, dev)
    mom[:, 2:] = fin.permute(1, 0, 2)
    return mom


def to_soa(mom: torch.Tensor) -> torch.Tensor:
    """[n_points, n_ext, 4] -> contiguous SoA [n_ext*4, n_points] (mom[(4j+mu)*n + i])."""
    n = mom.shape[0]
    return mom.permute(1, 2, 0).reshape(-1, n).contiguous()


def from_soa(soa: torch.Tensor, n_ext: int) -> torch.Tensor:
    n = soa.shape[-1]
    return soa.reshape(n_ext, 4, n).permute(2, 0, 1).contiguous()


def boost_rotate(mom: torch.Tensor, seed: int = 7, max_rapidity: float = 2.0) -> torch.Tensor:
    """Apply one random proper Lorentz transformation per point (rotation then
    boost).  Input-side helper for the Lorentz-invariance pin."""
    n = mom.shape[0]
    g = _gen(seed, "cpu")
    f64 = torch.float64
    r = torch.rand((6, n), generator=g, dtype=f64)
    # random rotation from a random unit quaternion
    qv = torch.randn((n, 4), generator=g, dtype=f64)
    qv = qv / qv.norm(dim=-1, keepdim=True)
    w, x, y, z = qv.unbind(-1)
    R = torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)], -1),
        torch.stack([2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)], -1),
        torch.stack([2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)], -1),
    ], -2)  # [n,3,3]
    out = mom.clone()
    out[..., 1:] = torch.einsum("nij,nkj->nki", R, mom[..., 1:])
    eta = max_rapidity * r[0]
    c = 2 * r[1] - 1
    phi = 2 * math.pi * r[2]
    st = torch.sqrt(1 - c * c)
    nvec = torch.stack([st * torch.cos(phi), st * torch.sin(phi), c], -1)  # [n,3]
    ch, sh = torch.cosh(eta), torch.sinh(eta)
    E = out[..., 0]
    pn = (out[..., 1:] * nvec[:, None]).sum(-1)
    E2 = ch[:, None] * E + sh[:, None] * pn
    pn2 = sh[:, None] * E + ch[:, None] * pn
    out2 = out.clone()
    out2[..., 0] = E2
    out2[..., 1:] = out[..., 1:] + (pn2 - pn)[..., None] * nvec[:, None]
    return out2
