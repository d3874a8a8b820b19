"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
legs may import this module.  The product package ``paper_2602_00735_b200`` never imports it and shares
no code with it (the only shared module is ``paper_2602_00735_b200/workloads.py``, which holds seeded
input generators and config literals, none of the method's arithmetic).

Citations: ``P:n`` = /root/reference/PAPER.md line n; ``BJ`` = BASELINE.json; D-numbers = DESIGN.md
section 3 readings.

Contents
  * grid / widths from a config (O1, O2; D2, D8)             -- ``Oracle.from_config``
  * ctypes bindings to ``orc.c`` (PML, P1 assembly, RHS, matvec, band LU, RAS apply)
  * right-preconditioned restarted GMRES with modified Gram-Schmidt (O9), in numpy
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "orc.c")
_LIB = os.path.join(_HERE, "liborc.so")


def build(force: bool = False) -> str:
    """Compile orc.c -> liborc.so (plain gcc, OpenMP across subdomains only)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Params(C.Structure):
    _fields_ = [("k", C.c_double), ("sigma0", C.c_double), ("h", C.c_double),
                ("nix", C.c_int), ("niy", C.c_int), ("ng", C.c_int), ("kappa", C.c_double),
                ("px", C.c_int), ("py", C.c_int), ("novlp", C.c_int), ("npml", C.c_int), ("local_bc", C.c_int),
                ("pou", C.c_int), ("elem", C.c_int), ("frame", C.c_int), ("pml_c", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp, ip, dp, i64p = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.orc_create.restype = vp
        L.orc_create.argtypes = [C.POINTER(_Params), C.c_char_p, C.c_int]
        L.orc_destroy.argtypes = [vp]
        L.orc_dims.argtypes = [vp, ip]
        L.orc_subdomain.argtypes = [vp, C.c_int, ip]
        L.orc_gfun.argtypes = [C.c_double, C.c_double, C.c_double, dp]
        L.orc_gamma.argtypes = [vp, C.c_int, C.c_int, C.c_long, vp, vp]
        L.orc_gamma_q.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, vp, vp]
        L.orc_global_stencil.argtypes = [vp, vp]
        L.orc_matvec.argtypes = [vp, vp, vp]
        L.orc_matvec_rows.argtypes = [vp, vp, i64p, C.c_int, vp]
        L.orc_rhs.argtypes = [vp, C.c_int, dp, vp, C.c_double, vp]
        L.orc_local_band.restype = C.c_int64
        L.orc_local_band.argtypes = [vp, C.c_int, vp]
        L.orc_band_lu.restype = C.c_int64
        L.orc_band_lu.argtypes = [C.c_int64, C.c_int, vp]
        L.orc_band_solve.argtypes = [C.c_int64, C.c_int, vp, vp]
        L.orc_factor.restype = C.c_int
        L.orc_factor.argtypes = [vp, ip, C.c_int, i64p]
        L.orc_release.argtypes = [vp]
        L.orc_factor_dedup.restype = C.c_int
        L.orc_factor_dedup.argtypes = [vp, i64p, ip]
        L.orc_dedup_class.argtypes = [vp, C.c_int, ip]
        L.orc_chi1.restype = C.c_double
        L.orc_chi1.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.orc_apply.restype = C.c_int
        L.orc_apply.argtypes = [vp, vp, vp, ip, C.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def gfun(t: float, kappa: float, sigma0: float):
    """(g, g', g'') of the BJ profile (configs[0]): sigma0 t^3/(3 kappa^2), linear beyond kappa."""
    out = (C.c_double * 3)()
    lib().orc_gfun(t, kappa, sigma0, out)
    return out[0], out[1], out[2]


# ------------------------------------------------------------------------------------------------
# O1/O2: grid and widths from a BASELINE.json config (D2, D8)
# ------------------------------------------------------------------------------------------------
def round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


def n_int_from(k: float, ppw: int) -> int:
    """D2: n_int = round(ppw k / 2pi) cells on (0,1); h = 1/n_int (BJ: '10 points per wavelength gives a
    uniform 52x52-cell mesh' at k = 20 with 10 PML cells per side)."""
    return round_half_up(ppw * k / (2.0 * math.pi))


def width_from(k: float) -> int:
    """BJ configs[0]: overlap delta and local PML width are each max(2, round(1.59 ln k)) cells."""
    return max(2, round_half_up(1.59 * math.log(k)))


@dataclass
class Problem:
    k: float
    sigma0: float
    h: float
    nix: int
    niy: int
    ng: int
    kappa: float
    px: int
    py: int
    novlp: int
    npml: int
    local_bc: int = 0    # 0 RAS-PML-Drch, 1 RAS-PML-Imp
    pou: int = 0         # 0 owner indicator (D10), 1 linear ramps
    elem: int = 0        # 0 P1 (D1), 1 Q1 bilinear (D18)
    frame: int = 0       # 0 BJ frame (Omega_int = (0,1)^2 + ng PML cells), 1 paper frame (Omega = (0,1)^2; D19)
    pml_c: float = 0.0   # paper frame: g(t) = pml_c t^3


def problem_from_config(k, ppw=10, n_pml_global=10, sigma0=5.0, nsub_x=1, nsub_y=1,
                        n_ovlp=-1, n_pml=-1, local_bc=0, pou=0) -> Problem:
    n_int = n_int_from(k, ppw)
    h = 1.0 / n_int
    w = width_from(k)
    return Problem(k=float(k), sigma0=float(sigma0), h=h, nix=n_int, niy=n_int, ng=n_pml_global,
                   kappa=n_pml_global * h,  # D3: kappa_g = 1 wavelength ~ 10 cells at 10 ppw
                   px=nsub_x, py=nsub_y,
                   novlp=w if n_ovlp < 0 else n_ovlp, npml=w if n_pml < 0 else n_pml, local_bc=local_bc, pou=pou)


def problem_from_paper(k, nsub, pml, ovlp, local_bc=1, pou=1, n_cells=None, kappa_wavelengths=3.0,
                       pml_c=None) -> Problem:
    """The paper's own experiment (Tables 1-4): Omega = (0,1)^2 is a uniform n x n grid of Q1 cells
    (grid "600^2" at k = 300, i.e. n = 2k: D19), global PML of width kappa_g = 3 wavelengths inside Omega with
    g(x) = 10 k x^3, N = nsub^2 subdomains, `pml` / `ovlp` cells of local PML / overlap (the integers
    printed in the tables; D20), impedance (RAS-PML-Imp) or Dirichlet local faces, linear-ramp PoU."""
    n = int(round(2 * k)) if n_cells is None else int(n_cells)
    lam = 2.0 * math.pi / k
    return Problem(k=float(k), sigma0=0.0, h=1.0 / n, nix=n, niy=n, ng=0, kappa=kappa_wavelengths * lam,
                   px=nsub, py=nsub, novlp=ovlp, npml=pml, local_bc=local_bc, pou=pou, elem=1, frame=1,
                   pml_c=10.0 * k if pml_c is None else float(pml_c))


class OracleError(RuntimeError):
    pass


class Oracle:
    def __init__(self, prob: Problem):
        self.prob = prob
        p = _Params(prob.k, prob.sigma0, prob.h, prob.nix, prob.niy, prob.ng, prob.kappa,
                    prob.px, prob.py, prob.novlp, prob.npml, prob.local_bc, prob.pou, prob.elem, prob.frame,
                    prob.pml_c)
        self.ns = 9 if prob.elem == 1 else 7
        err = C.create_string_buffer(256)
        self._h = lib().orc_create(C.byref(p), err, 256)
        if not self._h:
            raise OracleError("layout: " + err.value.decode())
        d = (C.c_int * 7)()
        lib().orc_dims(self._h, d)
        self.N = (d[0], d[1])
        self.nf = (d[2], d[3])
        self.nfree = d[2] * d[3]
        self.nsub = d[4]

    @classmethod
    def from_config(cls, **kw) -> "Oracle":
        return cls(problem_from_config(**kw))

    @classmethod
    def from_paper(cls, **kw) -> "Oracle":
        return cls(problem_from_paper(**kw))

    def close(self):
        if getattr(self, "_h", None):
            lib().orc_destroy(self._h)
            self._h = None

    __del__ = close

    # -- layout ---------------------------------------------------------------------------------
    def subdomain(self, j: int) -> dict:
        o = (C.c_int * 20)()
        lib().orc_subdomain(self._h, j, o)
        keys = ["own_lo", "own_hi", "int_lo", "int_hi", "full_lo", "full_hi", "has_lo", "has_hi", "m", "node0"]
        return {k: (o[i], o[10 + i]) for i, k in enumerate(keys)}

    def chi(self, axis: int, block: int, x: int) -> float:
        """1-D partition-of-unity factor of `block` at node x (owner indicator or linear ramp)."""
        return lib().orc_chi1(self._h, axis, block, x)

    # -- PML ------------------------------------------------------------------------------------
    def gamma(self, axis: int, X3: int, sub: int = -1):
        g = np.zeros(1, np.complex128)
        dg = np.zeros(1, np.complex128)
        lib().orc_gamma(self._h, sub, axis, X3, _ptr(g), _ptr(dg))
        return complex(g[0]), complex(dg[0])

    def gamma_q(self, axis: int, ci: int, xi: float, sub: int = -1):
        """(gamma, gamma') at x = (ci + xi) h on the Q1 path (global, or subdomain `sub`'s local scaling)."""
        g = np.zeros(1, np.complex128)
        dg = np.zeros(1, np.complex128)
        lib().orc_gamma_q(self._h, sub, axis, ci, xi, _ptr(g), _ptr(dg))
        return complex(g[0]), complex(dg[0])

    # -- operators ------------------------------------------------------------------------------
    OFFSETS = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (-1, 1), (1, -1)]

    def stencil(self) -> np.ndarray:
        """Global matrix as [nfree, ns] slots: centre, E, W, N, S, NE, SW (+ NW, SE for Q1)."""
        out = np.zeros((self.nfree, self.ns), np.complex128)
        lib().orc_global_stencil(self._h, _ptr(out))
        return out

    def matrix(self):
        """Global A as scipy CSR (assembled from the 7 slots)."""
        import scipy.sparse as sp
        A7 = self.stencil()
        nfx, nfy = self.nf
        idx = np.arange(self.nfree)
        i = idx % nfx
        j = idx // nfx
        rows, cols, vals = [], [], []
        for s, (dx, dy) in enumerate(self.OFFSETS[:self.ns]):
            qi, qj = i + dx, j + dy
            ok = (qi >= 0) & (qi < nfx) & (qj >= 0) & (qj < nfy)
            rows.append(idx[ok]); cols.append((qi + nfx * qj)[ok]); vals.append(A7[ok, s])
        return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.nfree, self.nfree))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.complex128)
        y = np.empty(self.nfree, np.complex128)
        lib().orc_matvec(self._h, _ptr(x), _ptr(y))
        return y

    def matvec_rows(self, x: np.ndarray, rows: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.complex128)
        rows = np.ascontiguousarray(rows, np.int64)
        y = np.empty(len(rows), np.complex128)
        lib().orc_matvec_rows(self._h, _ptr(x), rows.ctypes.data_as(C.POINTER(C.c_int64)), len(rows), _ptr(y))
        return y

    def rhs(self, xy: np.ndarray, amp: np.ndarray, sigma: float) -> np.ndarray:
        xy = np.ascontiguousarray(xy, np.float64)
        amp = np.ascontiguousarray(amp, np.complex128)
        b = np.empty(self.nfree, np.complex128)
        lib().orc_rhs(self._h, len(amp), xy.ctypes.data_as(C.POINTER(C.c_double)), _ptr(amp), sigma, _ptr(b))
        return b

    def local_band(self, j: int):
        s = self.subdomain(j)
        mx, my = s["m"]
        p = mx + 1
        band = np.zeros((mx * my, 2 * p + 1), np.complex128)
        lib().orc_local_band(self._h, j, _ptr(band))
        return band, p

    def local_matrix(self, j: int) -> np.ndarray:
        """Dense A_j (small cases only)."""
        band, p = self.local_band(j)
        n = band.shape[0]
        A = np.zeros((n, n), np.complex128)
        for r in range(n):
            for off in range(-p, p + 1):
                c = r + off
                if 0 <= c < n:
                    A[r, c] = band[r, off + p]
        return A

    def factor(self, subs=None):
        zr = C.c_int64(-1)
        if subs is None:
            rc = lib().orc_factor(self._h, None, 0, C.byref(zr))
        else:
            arr = (C.c_int * len(subs))(*subs)
            rc = lib().orc_factor(self._h, arr, len(subs), C.byref(zr))
        if rc != 0:
            raise OracleError(f"zero pivot: subdomain {-rc - 1}, row {zr.value}")

    def factor_dedup(self) -> int:
        """Dedup mode (SURVEY 8(d) memory fallback): factor one representative per bitwise-distinct A_j, after
        asserting that every member is bitwise equal to its representative.  Returns the number of classes."""
        zr = C.c_int64(-1)
        nc = C.c_int(0)
        rc = lib().orc_factor_dedup(self._h, C.byref(zr), C.byref(nc))
        if rc != 0:
            if -rc - 1 < self.nsub:
                raise OracleError(f"zero pivot: subdomain {-rc - 1}, row {zr.value}")
            raise OracleError(f"dedup: subdomain {-rc - 1 - self.nsub} is not bitwise equal to its representative")
        self.nclasses = nc.value
        return nc.value

    def dedup_class(self, j: int):
        """(class, representative, class size) of subdomain j after factor_dedup."""
        o = (C.c_int * 3)()
        lib().orc_dedup_class(self._h, j, o)
        return o[0], o[1], o[2]

    def release(self):
        lib().orc_release(self._h)

    def apply(self, v: np.ndarray, subs=None, out: np.ndarray | None = None) -> np.ndarray:
        """z = sum_j R~_j^T A_j^-1 R_j v over all (or the listed) subdomains."""
        v = np.ascontiguousarray(v, np.complex128)
        z = np.zeros(self.nfree, np.complex128) if out is None else out
        if subs is None:
            rc = lib().orc_apply(self._h, _ptr(v), _ptr(z), None, 0)
        else:
            arr = (C.c_int * len(subs))(*subs)
            rc = lib().orc_apply(self._h, _ptr(v), _ptr(z), arr, len(subs))
        if rc != 0:
            raise OracleError("apply before factor")
        return z

    def owner_of(self, g: int) -> int:
        """Subdomain owning free node g (D10)."""
        nfx = self.nf[0]
        i, j = g % nfx + 1, g // nfx + 1
        for s in range(self.nsub):
            d = self.subdomain(s)
            if d["own_lo"][0] <= i < d["own_hi"][0] and d["own_lo"][1] <= j < d["own_hi"][1]:
                return s
        raise OracleError(f"node {g} has no owner")


# ------------------------------------------------------------------------------------------------
# Algorithm 1 RAS_IterSolve in its discrete form (eq. local-ras-discrete + eq. update1,
# P:130-142): u^{n+1} = u^n + sum_j R~_j^T A_j^{-1} R_j (f - A u^n) = u^n + B^{-1}(f - A u^n).
# Stops when ||f - A u|| <= rtol ||f||, at maxit, or flags divergence when the relative residual exceeds
# 1e6 or is not finite.
# ------------------------------------------------------------------------------------------------
@dataclass
class RichardsonResult:
    x: np.ndarray
    iterations: int
    status: int          # 0 converged, 2 maxit, 3 diverged
    relres: float
    history: list


def richardson(A, M, b: np.ndarray, rtol: float = 1e-6, maxit: int = 500, x0: np.ndarray | None = None,
               diverge: float = 1e6) -> RichardsonResult:
    b = np.asarray(b, np.complex128)
    x = np.zeros_like(b) if x0 is None else np.array(x0, np.complex128)
    beta0 = np.linalg.norm(b)
    if beta0 == 0.0:
        return RichardsonResult(np.zeros_like(b), 0, 0, 0.0, [])
    r = b - A(x)
    rel = np.linalg.norm(r) / beta0
    its, hist = 0, []
    while rel > rtol and its < maxit:
        x = x + M(r)                       # u^{n+1} = u^n + sum_j chi_j c_j
        its += 1
        r = b - A(x)
        rel = np.linalg.norm(r) / beta0
        hist.append(rel)
        if not np.isfinite(rel) or rel > diverge:
            return RichardsonResult(x, its, 3, rel, hist)
    return RichardsonResult(x, its, 0 if rel <= rtol else 2, rel, hist)


# ------------------------------------------------------------------------------------------------
# O9: right-preconditioned restarted GMRES(m), modified Gram-Schmidt, Hermitian inner products
# ("Algorithm 1 as a preconditioner for GMRES"; D13).
# ------------------------------------------------------------------------------------------------
@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    restarts: int
    status: int          # 0 converged, 2 maxit, 3 breakdown (NaN/Inf)
    relres_est: float
    relres_true: float
    history: list


def mgs(V, w: np.ndarray):
    """O9 step 2, modified Gram-Schmidt against every vector of V in order: h_i = v_i^H w; w -= h_i v_i.
    Returns (w, h)."""
    h = np.zeros(len(V), np.complex128)
    for i in range(len(V)):
        h[i] = np.vdot(V[i], w)
        w = w - h[i] * V[i]
    return w, h


def gmres(A, M, b: np.ndarray, restart: int = 50, rtol: float = 1e-6, maxit: int = 5000,
          x0: np.ndarray | None = None) -> GmresResult:
    """A, M: callables (vector -> vector).  Solves A M u = b, x = M u (right preconditioning)."""
    b = np.asarray(b, np.complex128)
    x = np.zeros_like(b) if x0 is None else np.array(x0, np.complex128)
    beta0 = np.linalg.norm(b)
    if beta0 == 0.0:
        return GmresResult(np.zeros_like(b), 0, 0, 0, 0.0, 0.0, [])
    r = b - A(x) if x0 is not None else b.copy()
    its, cycles, hist = 0, 0, []
    est = np.linalg.norm(r) / beta0
    while True:
        beta = np.linalg.norm(r)
        m = restart
        V = [r / beta]
        H = np.zeros((m + 1, m), np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, np.complex128)
        g = np.zeros(m + 1, np.complex128)
        g[0] = beta
        jend = 0
        for j in range(m):
            w = A(M(V[j]))
            its += 1
            w, H[:j + 1, j] = mgs(V, w)
            hn = np.linalg.norm(w)
            H[j + 1, j] = hn
            if not np.isfinite(hn):
                return GmresResult(x, its, cycles, 3, float("nan"), float("nan"), hist)
            if hn != 0.0:
                V.append(w / hn)
            for i in range(j):                           # previous rotations
                hi, hi1 = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * hi + sn[i] * hi1
                H[i + 1, j] = -np.conj(sn[i]) * hi + cs[i] * hi1
            a, bb = H[j, j], H[j + 1, j]                 # new rotation
            if a == 0:
                cs[j], sn[j] = 0.0, 1.0
                H[j, j] = bb
            else:
                rho = math.sqrt(abs(a) ** 2 + abs(bb) ** 2)
                cs[j] = abs(a) / rho
                sn[j] = (a / abs(a)) * np.conj(bb) / rho
                H[j, j] = (a / abs(a)) * rho
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1]) / beta0
            hist.append(est)
            jend = j + 1
            if abs(g[j + 1]) <= rtol * beta0 or hn == 0.0 or its >= maxit:
                break
        y = np.zeros(jend, np.complex128)                # back substitution H y = g
        for i in range(jend - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:jend] @ y[i + 1:jend]) / H[i, i]
        t = np.zeros_like(b)
        for i in range(jend):
            t += y[i] * V[i]
        x = x + M(t)
        r = b - A(x)
        true = np.linalg.norm(r) / beta0
        cycles += 1
        if true <= rtol:
            return GmresResult(x, its, cycles - 1, 0, est, true, hist)
        if its >= maxit:
            return GmresResult(x, its, cycles - 1, 2, est, true, hist)
