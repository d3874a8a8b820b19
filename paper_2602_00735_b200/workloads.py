"""Seeded synthetic workloads (BASELINE.json configs c0..c4) -- shared by the product harness and the
oracle tests.  This module holds config literals and random draws only: none of the method's arithmetic
(grid sizing, widths, PML, assembly, solves) lives here, so the CUDA path and the oracle stay independent.

Recipe:
  * k, subdomain grid, source count and seed are BASELINE.json configs[0..4] (seed = k);
  * ppw = 10, 10 global PML cells per side, sigma0 = 5, GMRES(50), rtol 1e-6, x0 = 0;
  * sources: x_s ~ U(0.2, 0.8)^2, a_s ~ CN(0, 1), drawn in that order from numpy default_rng(seed);
    Gaussian width sigma = lambda / 4 = (2 pi / k) / 4 (BJ configs[0]);
  * apply / matvec probe vectors: N(0,1) + i N(0,1) per free node from default_rng(k + 1).
The paper's own workload is a single smoothed delta at (0.5, 0.5): this is a synthetic
stand-in with the same structure (localised sources well inside Omega_int), not a dataset.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    k: float
    nsub: int            # subdomains per axis (nsub x nsub Cartesian split)
    nsrc: int
    seed: int
    ppw: int = 10
    n_pml_global: int = 10
    sigma0: float = 5.0
    restart: int = 50
    rtol: float = 1e-6
    gpus: tuple = field(default=(1,))


CONFIGS = {
    "c0": Config("c0", 20.0, 2, 3, 20),
    "c1": Config("c1", 100.0, 4, 8, 100),
    "c2": Config("c2", 400.0, 16, 16, 400, gpus=(1, 2)),
    "c3": Config("c3", 1600.0, 64, 32, 1600, gpus=(1, 2, 4, 8)),
    "c4": Config("c4", 3200.0, 128, 64, 3200, gpus=(4, 8)),
}


def sources(cfg_or_seed, nsrc: int | None = None, k: float | None = None):
    """(xy[nsrc,2], amp[nsrc] complex, sigma) for a config (or an explicit seed / nsrc / k)."""
    if isinstance(cfg_or_seed, Config):
        seed, nsrc, k = cfg_or_seed.seed, cfg_or_seed.nsrc, cfg_or_seed.k
    else:
        seed = int(cfg_or_seed)
    rng = np.random.default_rng(seed)
    xy = rng.uniform(0.2, 0.8, (nsrc, 2))
    amp = (rng.standard_normal(nsrc) + 1j * rng.standard_normal(nsrc)) / math.sqrt(2.0)
    sigma = (2.0 * math.pi / k) / 4.0
    return np.ascontiguousarray(xy), np.ascontiguousarray(amp.astype(np.complex128)), sigma


def probe_vector(n: int, seed: int) -> np.ndarray:
    """N(0,1) + i N(0,1) entries (apply / matvec probes); seed = k + 1 for a config."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal(n)
    im = rng.standard_normal(n)
    return (re + 1j * im).astype(np.complex128)


# ------------------------------------------------------------------------------------------------------------------
# The paper's own experiment (Tables 1-4): Omega = (0,1)^2 on an n x n grid of Q1
# cells with n = 2k ("grid 600^2" at k = 300, ~12.6 points per wavelength), global PML of 3 wavelengths with
# g(x) = 10 k x^3, one smoothed delta at (0.5, 0.5), N = nsub^2 subdomains with `pml` / `ovlp` cells of local PML /
# overlap as printed in the tables, RAS-PML-Imp, linear-ramp PoU, rtol 1e-10.  Config literals only.
# ------------------------------------------------------------------------------------------------------------------
@dataclass(frozen=True)
class PaperConfig:
    name: str
    k: float
    nsub: int
    pml: int
    ovlp: int
    n_cells: int
    local_bc: int = 1      # 1 = impedance (RAS-PML-Imp), 0 = Dirichlet (RAS-PML-Drch)
    rtol: float = 1e-10
    maxit: int = 500


PAPER_CONFIGS = {
    # Table 1 / Table 2 rows (C_kappa = 3/8, C_delta = 1/6)
    "p300": PaperConfig("p300", 300.0, 2, 8, 4, 600),
    "p600": PaperConfig("p600", 600.0, 4, 11, 5, 1200),
    "p1200": PaperConfig("p1200", 1200.0, 8, 15, 6, 2400),
    "p2400": PaperConfig("p2400", 2400.0, 16, 18, 8, 4800),
    # Table 4 rows (C_kappa = 1/2, C_delta = 1/6): the paper's timed runs
    "t300": PaperConfig("t300", 300.0, 2, 12, 4, 600),
    "t600": PaperConfig("t600", 600.0, 4, 16, 5, 1200),
    "t1200": PaperConfig("t1200", 1200.0, 8, 21, 6, 2400),
    "t2400": PaperConfig("t2400", 2400.0, 16, 26, 8, 4800),
}


def paper_source(k: float):
    """The smoothed delta of P:217-218, f(x) = 16 k^2/pi^3 exp(-16 k^2 |x - x_c|^2 / pi^2), x_c = (0.5, 0.5),
    written as one unit-mass Gaussian (2 pi s^2)^-1 exp(-|x - x_c|^2 / (2 s^2)) with s = pi / (k sqrt(32)):
    returns (xy[1,2], amp[1], s) in the frame of Omega = (0,1)^2."""
    return (np.array([[0.5, 0.5]]), np.array([1.0 + 0.0j]), math.pi / (k * math.sqrt(32.0)))
