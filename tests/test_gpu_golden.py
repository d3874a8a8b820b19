"""The headline config c3 (k = 1600, 6.58 M unknowns, 64 x 64 subdomains; BASELINE.json configs[3]) at FULL size,
against the oracle: the whole assembled stencil, right-hand side, one apply and one matvec element by element (oracle
run live, its apply in dedup mode), and the
GMRES(50) solve against the oracle-only golden record tests/golden/c3_gmres.json (scripts/make_golden.py: MGS GMRES
on the dedup-mode oracle, written without libhelm) -- iterations +-1, the residual-estimate history to 1e-6 relative,
||x|| and a seeded 64-row sketch S x to 1e-6 (north_star: "GPU solutions matching the oracle ... on all five
configs"; GMRES P:240-242, B^-1 P:143-147, A P:58-62, b D14).  Launched exactly as bench.py times it (one rank,
the persistent k_apply, DCGS2).  -m gpu."""
import os

import numpy as np
import pytest

from golden_util import as_complex, golden_path, load_golden, sketch_rel
from oracle.oracle import Oracle
from paper_2602_00735_b200.workloads import CONFIGS, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402

_C = {}


@pytest.fixture(scope="module", autouse=True)
def _release_c3():
    """The c3 context holds ~58 GB of device memory: free it when this module is done."""
    yield
    ctx = _C.pop("ctx", None)
    if ctx is not None:
        ctx.close()
    _C.clear()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def c3():
    if "ctx" not in _C:
        cfg = CONFIGS["c3"]
        ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
        ctx.factor()
        _C["ctx"] = ctx
        _C["o"] = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    return _C["ctx"], _C["o"]


def test_c3_stencil_full_vector():
    """Every coefficient of the assembled 7-point operator (6.58 M rows x 7 slots) vs the oracle's assembly."""
    ctx, o = c3()
    A = ctx.export_stencil().cpu().numpy()          # [7][n]
    R = o.stencil().T
    assert A.shape == R.shape
    assert np.max(np.abs(A - R)) <= 1e-13 * np.max(np.abs(R))


def test_c3_apply_and_matvec_full_vector():
    """One RAS-PML apply and one matvec at c3, in the bench's launch configuration, against the oracle on EVERY node
    (the oracle's apply in dedup mode, D24 -- exact): apply <= 1e-10, matvec <= 1e-13 (north_star)."""
    ctx, o = c3()
    cfg = CONFIGS["c3"]
    from paper_2602_00735_b200.workloads import probe_vector
    v = probe_vector(ctx.n, int(cfg.k) + 1)
    vt = torch.from_numpy(v).cuda()
    z = ctx.precond_apply(vt).cpu().numpy()
    y = ctx.matvec(vt).cpu().numpy()
    assert o.factor_dedup() == 16
    zo = o.apply(v)
    o.release()
    yo = o.matvec(v)
    assert np.linalg.norm(z - zo) / np.linalg.norm(zo) <= 1e-10
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) <= 1e-13


def test_c3_rhs_full_vector():
    """b = M f_I on every free node vs the oracle, and its sketch vs the golden record."""
    ctx, o = c3()
    cfg = CONFIGS["c3"]
    xy, amp, sig = sources(cfg)
    b = ctx.rhs(xy, amp, sig).cpu().numpy()
    bo = o.rhs(xy, amp, sig)
    assert np.max(np.abs(b - bo)) <= 1e-13 * np.max(np.abs(bo))
    if os.path.exists(golden_path("c3")):
        g = load_golden("c3")
        assert abs(np.linalg.norm(b) - g["norm_b"]) <= 1e-13 * g["norm_b"]
        assert sketch_rel(b, g, "sketch_b") <= 1e-13


@pytest.mark.skipif(not os.path.exists(golden_path("c3")), reason="no c3 golden record")
def test_c3_gmres_matches_the_oracle_golden():
    ctx, _ = c3()
    g = load_golden("c3")
    cfg = CONFIGS["c3"]
    assert g["seed"] == cfg.seed and g["restart"] == cfg.restart and g["rtol"] == cfg.rtol
    b = ctx.rhs(*sources(cfg))
    x, info, hist = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"], history=True)
    assert info.status == g["status"] == 0
    assert abs(info.iterations - g["iterations"]) <= 1
    h_orc = np.asarray(g["history"])
    n = min(len(hist), len(h_orc))
    assert np.max(np.abs(hist[:n] - h_orc[:n]) / h_orc[:n]) <= 1e-6
    assert info.relres_true <= cfg.rtol
    xn = x.cpu().numpy()
    assert abs(np.linalg.norm(xn) - g["norm_x"]) <= 1e-6 * g["norm_x"]
    assert sketch_rel(xn, g) <= 1e-6


@pytest.mark.parametrize("name", ["c0", "c1", "c2"])
def test_small_configs_gmres_match_the_oracle_golden(name):
    """The same golden comparison at c0-c2 (BASELINE.json configs[0..2]): iterations +-1, history 1e-6, x sketch 1e-6."""
    g = load_golden(name)
    cfg = CONFIGS[name]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    b = ctx.rhs(*sources(cfg))
    x, info, hist = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"], history=True)
    assert info.status == g["status"] == 0 and abs(info.iterations - g["iterations"]) <= 1
    h_orc = np.asarray(g["history"])
    n = min(len(hist), len(h_orc))
    assert np.max(np.abs(hist[:n] - h_orc[:n]) / h_orc[:n]) <= 1e-6
    assert sketch_rel(x.cpu().numpy(), g) <= 1e-6
    ctx.close()


@pytest.mark.skipif(not os.path.exists(golden_path("c3_ramp")), reason="no c3 ramp-PoU golden record")
def test_c3_ramp_pou_gmres_matches_the_oracle_golden():
    """NEXT-3 at full size: GMRES(50) with the paper's linear-ramp partition of unity at c3 against the
    oracle-only golden record (scripts/make_golden.py c3 --pou ramp)."""
    from paper_2602_00735_b200.helm import POU_RAMP
    g = load_golden("c3_ramp")
    cfg = CONFIGS["c3"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, pou=POU_RAMP)
    ctx.factor()
    b = ctx.rhs(*sources(cfg))
    x, info, hist = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"], history=True)
    assert info.status == g["status"] == 0 and abs(info.iterations - g["iterations"]) <= 1
    h_orc = np.asarray(g["history"])
    n = min(len(hist), len(h_orc))
    assert np.max(np.abs(hist[:n] - h_orc[:n]) / h_orc[:n]) <= 1e-6
    assert sketch_rel(x.cpu().numpy(), g) <= 1e-6
    ctx.close()
    torch.cuda.empty_cache()


@pytest.mark.skipif(not os.path.exists(golden_path("c4")), reason="no c4 golden record")
def test_c4_gmres_on_one_gpu_matches_the_oracle_golden():
    """c4 (k = 3200, 26.1 M unknowns, 128 x 128 subdomains; BASELINE.json configs[4]) whole on ONE GPU: with the
    shared factors (D28: 16 classes, ~0.5 GB of inverses instead of 198 GB) the solve fits in HBM.  Against the
    oracle-only golden record (its first six GMRES(50) cycles, maxit = 300, status 2): the same 300 iterations, the
    residual-estimate history to 1e-6 relative, ||x|| and the seeded x sketch to 1e-6."""
    for k in list(_C):   # release c3 first
        if k == "ctx":
            _C[k].close()
        del _C[k]
    torch.cuda.empty_cache()
    g = load_golden("c4")
    cfg = CONFIGS["c4"]
    assert g["seed"] == cfg.seed and g["restart"] == cfg.restart
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    assert ctx.factor_classes()["classes"] == g["oracle_timing"]["classes"]
    b = ctx.rhs(*sources(cfg))
    x, info, hist = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"], history=True)
    assert info.status == g["status"] and info.iterations == g["iterations"]
    h_orc = np.asarray(g["history"])
    assert np.max(np.abs(hist - h_orc) / h_orc) <= 1e-6
    xn = x.cpu().numpy()
    assert abs(np.linalg.norm(xn) - g["norm_x"]) <= 1e-6 * g["norm_x"]
    assert sketch_rel(xn, g) <= 1e-6
    ctx.close()

