"""Thin Python binding of libhelm (include/helm.h): argument marshalling only.

Every step of the hot path runs in libhelm's CUDA kernels; this module converts torch tensors to device
pointers and ctypes structs.  PyTorch is used for device memory, streams and process groups only.  There is
no CPU fallback: if libhelm.so is missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_LIB = None


class HelmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"helm error {code}: {msg}")
        self.code = code


HELM_OK, HELM_NOT_CONVERGED, HELM_BREAKDOWN = 0, 2, 3


class Params(C.Structure):
    _fields_ = [("k", C.c_double), ("ppw", C.c_int), ("n_pml_global", C.c_int), ("sigma0", C.c_double),
                ("nsub_x", C.c_int), ("nsub_y", C.c_int), ("n_ovlp", C.c_int), ("n_pml", C.c_int),
                ("local_bc", C.c_int), ("gpu_grid_x", C.c_int), ("gpu_grid_y", C.c_int), ("pou", C.c_int),
                ("elem", C.c_int), ("n_cells", C.c_int), ("kappa_g", C.c_double), ("pml_c", C.c_double)]


class Layout(C.Structure):
    _fields_ = [("n_free_global", C.c_longlong), ("N_cells", C.c_int), ("n_int", C.c_int),
                ("n_ovlp", C.c_int), ("n_pml", C.c_int),
                ("owned_i0", C.c_int), ("owned_i1", C.c_int), ("owned_j0", C.c_int), ("owned_j1", C.c_int),
                ("n_local", C.c_longlong), ("n_sub", C.c_int), ("n_sub_local", C.c_int), ("m_max", C.c_int),
                ("local_unknowns", C.c_longlong), ("factor_bytes", C.c_longlong), ("apply_bytes", C.c_longlong),
                ("band_bytes", C.c_longlong), ("spmv_bytes", C.c_longlong), ("stencil_slots", C.c_int),
                ("overlap_interior", C.c_int), ("factor_flop", C.c_longlong)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class GmresInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("restarts", C.c_int), ("status", C.c_int), ("applies", C.c_int),
                ("relres_est", C.c_double), ("relres_true", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int)]


class RichardsonInfo(C.Structure):
    _fields_ = [("iterations", C.c_int), ("status", C.c_int), ("relres", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int)]


class Plan(C.Structure):
    _fields_ = [("gx", C.c_int), ("gy", C.c_int), ("rx", C.c_int), ("ry", C.c_int),
                ("owned_i0", C.c_int), ("owned_i1", C.c_int), ("owned_j0", C.c_int), ("owned_j1", C.c_int),
                ("ext_i0", C.c_int), ("ext_i1", C.c_int), ("ext_j0", C.c_int), ("ext_j1", C.c_int),
                ("halo_lo", C.c_int), ("halo_hi", C.c_int), ("nbr", C.c_int * 4), ("n_sub_local", C.c_int)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "nbr"}
        d["nbr"] = list(self.nbr)
        return d


class Msg(C.Structure):
    _fields_ = [("phase", C.c_int), ("peer", C.c_int),
                ("send_i0", C.c_int), ("send_i1", C.c_int), ("send_j0", C.c_int), ("send_j1", C.c_int),
                ("recv_i0", C.c_int), ("recv_i1", C.c_int), ("recv_j0", C.c_int), ("recv_j1", C.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["helm_setup", "helm_get_layout", "helm_rhs", "helm_factor", "helm_matvec", "helm_precond_apply",
           "helm_precond_apply_host", "helm_gmres", "helm_gmres_host", "helm_export_stencil",
           "helm_profile_enable", "helm_profile_read", "helm_last_error", "helm_destroy",
           "helm_plan_rank", "helm_halo_schedule", "helm_nccl_unique_id", "helm_precond_apply_ext",
           "helm_matvec_ext", "helm_richardson", "helm_probe_read_bandwidth", "helm_setup_loopback",
           "helm_probe_read_bandwidth_mode", "helm_set_orthogonalisation",
           "helm_get_krylov_basis", "helm_comm_info", "helm_probe_fp64_tflops", "helm_set_residual_band",
           "helm_comm_counters", "helm_halo_band_counts", "helm_halo_band_rects", "helm_nccl_selftest",
           "helm_factor_classes"]


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libhelm.so (building it in-tree if needed).  Raises if it cannot be built or loaded."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_missing:
        _build.build()
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"libhelm.so missing at {_build.LIB}; run __graft_entry__.build()")
    L = C.CDLL(_build.LIB)
    vp, i, d = C.c_void_p, C.c_int, C.c_double
    L.helm_setup.argtypes = [C.POINTER(Params), i, i, vp, vp, C.POINTER(vp)]
    L.helm_setup_loopback.argtypes = [C.POINTER(Params), i, i, i, vp, C.POINTER(vp)]
    L.helm_get_layout.argtypes = [vp, C.POINTER(Layout)]
    L.helm_rhs.argtypes = [vp, i, vp, vp, d, vp]
    L.helm_factor.argtypes = [vp]
    L.helm_matvec.argtypes = [vp, vp, vp]
    L.helm_precond_apply.argtypes = [vp, vp, vp]
    L.helm_precond_apply_host.argtypes = [vp, vp, vp]
    L.helm_gmres.argtypes = [vp, vp, vp, i, d, i, C.POINTER(GmresInfo)]
    L.helm_gmres_host.argtypes = [vp, vp, vp, i, d, i, C.POINTER(GmresInfo)]
    L.helm_set_orthogonalisation.argtypes = [vp, i]
    L.helm_get_krylov_basis.argtypes = [vp, i, vp]
    L.helm_export_stencil.argtypes = [vp, vp]
    L.helm_profile_enable.argtypes = [vp, i]
    L.helm_profile_read.argtypes = [vp, C.POINTER(d), C.POINTER(i), C.POINTER(i)]
    L.helm_plan_rank.argtypes = [C.POINTER(Params), i, i, C.POINTER(Plan)]
    L.helm_halo_schedule.argtypes = [C.POINTER(Params), i, i, i, C.POINTER(Msg), i]
    L.helm_nccl_unique_id.argtypes = [vp]
    L.helm_precond_apply_ext.argtypes = [vp, vp, vp]
    L.helm_matvec_ext.argtypes = [vp, vp, vp]
    L.helm_richardson.argtypes = [vp, vp, vp, d, i, C.POINTER(RichardsonInfo)]
    L.helm_probe_read_bandwidth.argtypes = [C.c_longlong, i, C.POINTER(d)]
    L.helm_probe_read_bandwidth_mode.argtypes = [C.c_longlong, i, i, C.POINTER(d)]
    L.helm_probe_fp64_tflops.argtypes = [i, C.POINTER(d)]
    L.helm_set_residual_band.argtypes = [vp, i]
    L.helm_nccl_selftest.argtypes = [vp, C.c_longlong, i, C.POINTER(C.c_longlong)]
    L.helm_comm_counters.argtypes = [vp, i, C.POINTER(C.c_longlong)]
    L.helm_halo_band_counts.argtypes = [C.POINTER(Params), i, i, C.POINTER(C.c_longlong)]
    L.helm_halo_band_rects.argtypes = [C.POINTER(Params), i, i, i, i, C.POINTER(i), i]
    L.helm_comm_info.argtypes = [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i)]
    L.helm_factor_classes.argtypes = [vp, C.POINTER(C.c_longlong), C.POINTER(i), i]
    L.helm_last_error.argtypes = [vp]
    L.helm_last_error.restype = C.c_char_p
    L.helm_destroy.argtypes = [vp]
    for name in EXPORTS:
        if name not in ("helm_last_error", "helm_destroy"):
            getattr(L, name).restype = C.c_int
    L.helm_destroy.restype = None
    _LIB = L
    return L


def _ptr(t) -> int:
    """Device (or host) address of a contiguous complex128 tensor / numpy array."""
    import numpy as np
    if isinstance(t, np.ndarray):
        assert t.dtype == np.complex128 and t.flags["C_CONTIGUOUS"]
        return t.ctypes.data
    import torch
    assert t.dtype == torch.complex128 and t.is_contiguous(), "complex128 contiguous tensors only"
    return t.data_ptr()


BC_DIRICHLET, BC_IMPEDANCE = 0, 1
POU_OWNER, POU_RAMP = 0, 1
ELEM_P1, ELEM_Q1 = 0, 1
ORTH_DCGS2, ORTH_CGS2 = 0, 1


def make_params(k, nsub_x, nsub_y=None, ppw=10, n_pml_global=10, sigma0=5.0, n_ovlp=-1, n_pml=-1,
                gpu_grid=(0, 0), local_bc=BC_DIRICHLET, pou=POU_OWNER, elem=ELEM_P1, n_cells=0, kappa_g=0.0,
                pml_c=0.0) -> Params:
    return Params(float(k), ppw, n_pml_global, float(sigma0), nsub_x, nsub_y if nsub_y is not None else nsub_x,
                  n_ovlp, n_pml, local_bc, gpu_grid[0], gpu_grid[1], pou, elem, n_cells, float(kappa_g),
                  float(pml_c))


def paper_params(k, nsub, pml, ovlp, n_cells=None, local_bc=BC_IMPEDANCE, pou=POU_RAMP, gpu_grid=(0, 0)) -> dict:
    """Keyword arguments of Context for the paper's own experiment (D18-D22): Q1 on an
    n x n grid of Omega = (0,1)^2 (n = 2k: "grid 600^2" at k = 300), kappa_g = 3 wavelengths, g(x) = 10 k x^3,
    nsub^2 subdomains with `pml` / `ovlp` cells, RAS-PML-Imp and the linear-ramp PoU by default."""
    import math
    return dict(k=float(k), nsub_x=nsub, nsub_y=nsub, n_ovlp=ovlp, n_pml=pml, local_bc=local_bc, pou=pou,
                elem=ELEM_Q1, n_cells=int(round(2 * k)) if n_cells is None else int(n_cells),
                kappa_g=3.0 * 2.0 * math.pi / k, pml_c=10.0 * k, gpu_grid=gpu_grid)


def plan_rank(params: Params, rank: int, nranks: int) -> dict:
    """This rank's owned / ghost-framed rectangles and neighbours (host logic of libhelm, no GPU needed)."""
    L = load()
    pl = Plan()
    rc = L.helm_plan_rank(C.byref(params), rank, nranks, C.byref(pl))
    if rc != 0:
        raise HelmError(rc, "helm_plan_rank")
    return pl.as_dict()


def halo_schedule(params: Params, rank: int, nranks: int, width: int) -> list:
    """The two-phase halo exchange libhelm performs for `rank` (list of message dicts)."""
    L = load()
    msgs = (Msg * 4)()
    n = L.helm_halo_schedule(C.byref(params), rank, nranks, width, msgs, 4)
    if n < 0:
        raise HelmError(n, "helm_halo_schedule")
    return [msgs[q].as_dict() for q in range(n)]


def halo_band_counts(params: Params, rank: int, nranks: int) -> dict:
    """This rank's apply-frame halo volume (complex elements): full and section 3(i) band, sent and received."""
    L = load()
    out = (C.c_longlong * 4)()
    rc = L.helm_halo_band_counts(C.byref(params), rank, nranks, out)
    if rc != 0:
        raise HelmError(rc, "helm_halo_band_counts")
    return {"sent_full": out[0], "sent_band": out[1], "recv_full": out[2], "recv_band": out[3]}


def halo_band_rects(params: Params, rank: int, nranks: int, msg: int, side: int) -> list:
    """Band sub-rectangles (i0, i1, j0, j1) of apply-frame message `msg` (side 0 send, 1 receive), packing order."""
    L = load()
    cap = 4096
    buf = (C.c_int * (4 * cap))()
    n = L.helm_halo_band_rects(C.byref(params), rank, nranks, msg, side, buf, cap)
    if n < 0:
        raise HelmError(n, "helm_halo_band_rects")
    return [tuple(buf[4 * q:4 * q + 4]) for q in range(min(n, cap))]


def probe_read_bandwidth(nbytes: int = 8 << 30, reps: int = 5, mode: int = 0) -> float:
    """GB/s of libhelm's bulk-copy read stream over an nbytes device buffer (roofline context for bench.py);
    mode 0 interleaved chunks, mode 1 one contiguous stream per CTA (the apply's pattern)."""
    L = load()
    g = C.c_double()
    rc = L.helm_probe_read_bandwidth_mode(int(nbytes), int(reps), int(mode), C.byref(g))
    if rc != 0:
        raise HelmError(rc, "helm_probe_read_bandwidth")
    return g.value


def probe_fp64_tflops(mode: int = 0) -> float:
    """Measured FP64 TFLOP/s of this GPU: mode 0 tensor-core DMMA, mode 1 DFMA (roofline context for the factorisation)."""
    L = load()
    g = C.c_double()
    rc = L.helm_probe_fp64_tflops(int(mode), C.byref(g))
    if rc != 0:
        raise HelmError(rc, "helm_probe_fp64_tflops")
    return g.value


def nccl_unique_id() -> bytes:
    L = load()
    buf = C.create_string_buffer(128)
    rc = L.helm_nccl_unique_id(buf)
    if rc != 0:
        raise HelmError(rc, "helm_nccl_unique_id (library built without NCCL?)")
    return buf.raw


class Context:
    """One rank's RAS-PML problem: owns the libhelm context (operators, factors, Krylov workspace)."""

    def __init__(self, k: float, nsub_x: int, nsub_y: int | None = None, *, ppw: int = 10, n_pml_global: int = 10,
                 sigma0: float = 5.0, n_ovlp: int = -1, n_pml: int = -1, rank: int = 0, nranks: int = 1,
                 gpu_grid=(0, 0), stream=None, nccl_id: bytes | None = None, local_bc: int = BC_DIRICHLET,
                 pou: int = POU_OWNER, elem: int = ELEM_P1, n_cells: int = 0, kappa_g: float = 0.0,
                 pml_c: float = 0.0, loopback_group: int | None = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libhelm needs a CUDA device (no CPU fallback)")
        self.L = load()
        self.params = make_params(k, nsub_x, nsub_y, ppw, n_pml_global, sigma0, n_ovlp, n_pml, gpu_grid, local_bc,
                                  pou, elem, n_cells, kappa_g, pml_c)
        self.rank, self.nranks = rank, nranks
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self._h = C.c_void_p()
        if loopback_group is not None:
            rc = self.L.helm_setup_loopback(C.byref(self.params), rank, nranks, int(loopback_group),
                                            C.c_void_p(self.stream.cuda_stream), C.byref(self._h))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            rc = self.L.helm_setup(C.byref(self.params), rank, nranks, idbuf, C.c_void_p(self.stream.cuda_stream),
                                   C.byref(self._h))
        self._check(rc)
        self.layout = self._layout()
        self.n = self.layout.n_local
        self.plan = plan_rank(self.params, rank, nranks)

    # ------------------------------------------------------------------------------------------ plumbing
    def _check(self, rc: int, ok=(0,)):
        if rc in ok:
            return rc
        msg = self.L.helm_last_error(self._h).decode() if self._h else ""
        raise HelmError(rc, msg)

    def _layout(self) -> Layout:
        lay = Layout()
        self._check(self.L.helm_get_layout(self._h, C.byref(lay)))
        return lay

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self.L.helm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self):
        import torch
        return torch.empty(self.n, dtype=torch.complex128, device="cuda")

    # ------------------------------------------------------------------------------------------ API
    def rhs(self, xy, amp, sigma: float, out=None):
        import numpy as np
        xy = np.ascontiguousarray(xy, np.float64)
        amp = np.ascontiguousarray(amp, np.complex128)
        b = self.empty() if out is None else out
        self._check(self.L.helm_rhs(self._h, len(amp), xy.ctypes.data, amp.ctypes.data, float(sigma), _ptr(b)))
        return b

    def factor(self):
        self._check(self.L.helm_factor(self._h))
        self.layout = self._layout()   # factor bytes / flops now count the factored classes (D28)

    def matvec(self, x, out=None):
        y = self.empty() if out is None else out
        self._check(self.L.helm_matvec(self._h, _ptr(x), _ptr(y)))
        return y

    def precond_apply(self, r, out=None):
        z = self.empty() if out is None else out
        self._check(self.L.helm_precond_apply(self._h, _ptr(r), _ptr(z)))
        return z

    def precond_apply_ext(self, ext, out=None):
        """Apply with a caller-filled ghost-framed input covering plan['ext_*'] (no communication)."""
        z = self.empty() if out is None else out
        self._check(self.L.helm_precond_apply_ext(self._h, _ptr(ext), _ptr(z)))
        return z

    def matvec_ext(self, ext1, out=None):
        """matvec with a caller-filled input covering the owned rectangle grown by 1 toward neighbours."""
        y = self.empty() if out is None else out
        self._check(self.L.helm_matvec_ext(self._h, _ptr(ext1), _ptr(y)))
        return y

    def precond_apply_host(self, r_host, z_host):
        self._check(self.L.helm_precond_apply_host(self._h, _ptr(r_host), _ptr(z_host)))
        return z_host

    def set_orthogonalisation(self, mode: int):
        """GMRES orthogonalisation: ORTH_DCGS2 (default, re-orthogonalisation delayed one step) or ORTH_CGS2."""
        self._check(self.L.helm_set_orthogonalisation(self._h, int(mode)))

    def krylov_basis(self, nv: int):
        """The first nv GMRES basis vectors of the last gmres call, as an (nv, n) device tensor."""
        import torch
        out = torch.empty(nv, self.n, dtype=torch.complex128, device="cuda")
        self._check(self.L.helm_get_krylov_basis(self._h, int(nv), _ptr(out)))
        return out

    def gmres(self, b, x=None, restart: int = 50, rtol: float = 1e-6, maxit: int = 5000, history: bool = False):
        import numpy as np
        if x is None:
            x = self.empty()
            x.zero_()
        info = GmresInfo()
        hist = None
        if history:
            hist = np.zeros(maxit, np.float64)
            info.history = hist.ctypes.data_as(C.POINTER(C.c_double))
            info.history_cap = maxit
        rc = self.L.helm_gmres(self._h, _ptr(b), _ptr(x), restart, float(rtol), maxit, C.byref(info))
        self._check(rc, ok=(0, 2))
        return x, info, (hist[:info.iterations].copy() if hist is not None else None)

    def richardson(self, b, x=None, rtol: float = 1e-6, maxit: int = 500, history: bool = False):
        """Algorithm 1 (RAS_IterSolve) on the device; returns (x, info, history or None)."""
        import numpy as np
        if x is None:
            x = self.empty()
            x.zero_()
        info = RichardsonInfo()
        hist = None
        if history:
            hist = np.zeros(max(maxit, 1), np.float64)
            info.history = hist.ctypes.data_as(C.POINTER(C.c_double))
            info.history_cap = maxit
        rc = self.L.helm_richardson(self._h, _ptr(b), _ptr(x), float(rtol), maxit, C.byref(info))
        self._check(rc, ok=(0, 2, 4))
        return x, info, (hist[:info.iterations].copy() if hist is not None else None)

    def gmres_host(self, b_host, x_host, restart: int = 50, rtol: float = 1e-6, maxit: int = 5000):
        info = GmresInfo()
        rc = self.L.helm_gmres_host(self._h, _ptr(b_host), _ptr(x_host), restart, float(rtol), maxit, C.byref(info))
        self._check(rc, ok=(0, 2))
        return x_host, info

    def export_stencil(self):
        import torch
        ns = self.layout.stencil_slots
        out = torch.empty(ns * self.n, dtype=torch.complex128, device="cuda")
        self._check(self.L.helm_export_stencil(self._h, _ptr(out)))
        return out.view(ns, self.n)

    def set_residual_band(self, on: bool):
        """Section 3(i) residual restriction + band-only halo in helm_richardson (default on, owner PoU)."""
        self._check(self.L.helm_set_residual_band(self._h, int(bool(on))))

    def nccl_selftest(self, nelem: int, nmsg: int = 2) -> int:
        """Grouped ncclSend/ncclRecv of the halo transport, every rank to itself; returns the mismatch count."""
        mm = C.c_longlong()
        self._check(self.L.helm_nccl_selftest(self._h, int(nelem), int(nmsg), C.byref(mm)))
        return mm.value

    def comm_counters(self, reset: bool = False) -> dict:
        out = (C.c_longlong * 4)()
        self._check(self.L.helm_comm_counters(self._h, int(bool(reset)), out))
        return {"sent": out[0], "recv": out[1], "msgs": out[2], "allreduces": out[3]}

    def factor_classes(self, with_members: bool = False) -> dict:
        """After factor(): {'classes', 'batched', 'tiles', 'factor_bytes', 'apply_flop', 'apply_flop_issued'} (D28),
        plus 'class_of' (one class index per local subdomain) when with_members."""
        out = (C.c_longlong * 6)()
        n = self._layout().n_sub_local if with_members else 0
        cls = (C.c_int * max(n, 1))()
        self._check(self.L.helm_factor_classes(self._h, out, cls if with_members else None, n))
        r = {"classes": out[0], "batched": bool(out[1]), "tiles": out[2], "factor_bytes": out[3],
             "apply_flop": out[4], "apply_flop_issued": out[5]}
        if with_members:
            r["class_of"] = list(cls[:n])
        return r

    TRANSPORTS = {0: "none", 1: "nccl", 2: "loopback", 3: "shard"}

    def comm_info(self) -> dict:
        """{'transport': none|nccl|loopback|shard, 'nranks': ..., 'rank': ...} as the transport reports them."""
        t, n, r = C.c_int(), C.c_int(), C.c_int()
        self._check(self.L.helm_comm_info(self._h, C.byref(t), C.byref(n), C.byref(r)))
        return {"transport": self.TRANSPORTS.get(t.value, str(t.value)), "nranks": n.value, "rank": r.value}

    def profile(self, on: bool = True):
        self._check(self.L.helm_profile_enable(self._h, int(on)))

    def profile_read(self):
        ms, na, nt = C.c_double(), C.c_int(), C.c_int()
        self._check(self.L.helm_profile_read(self._h, C.byref(ms), C.byref(na), C.byref(nt)))
        return ms.value, na.value, nt.value
