"""DCGS2 (the default GMRES orthogonalisation: CGS2 with the re-orthogonalisation of v_j delayed into step j + 1's
projection sweep) against the undelayed CGS2 on the same context: the same Krylov basis in exact
arithmetic, so the same iteration counts, residual histories to rounding and the same solutions.  Restart
boundaries, early convergence inside a cycle, restart = 1 and maxit cut-offs are covered.  -m gpu."""
import numpy as np
import pytest

from paper_2602_00735_b200.workloads import CONFIGS, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import ORTH_CGS2, ORTH_DCGS2, HelmError  # noqa: E402


def solve(ctx, b, mode, **kw):
    ctx.set_orthogonalisation(mode)
    return ctx.gmres(b, history=True, **kw)


@pytest.mark.parametrize("name,restart,rtol,maxit", [("c0", 50, 1e-10, 200), ("c1", 50, 1e-8, 500),
                                                     ("c1", 7, 1e-8, 500), ("c1", 1, 1e-3, 40),
                                                     ("c2", 50, 1e-6, 1000), ("c1", 50, 0.0, 23)])
def test_dcgs2_equals_cgs2(name, restart, rtol, maxit):
    cfg = CONFIGS[name]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    b = ctx.rhs(*sources(cfg))
    x1, i1, h1 = solve(ctx, b, ORTH_CGS2, restart=restart, rtol=rtol, maxit=maxit)
    x2, i2, h2 = solve(ctx, b, ORTH_DCGS2, restart=restart, rtol=rtol, maxit=maxit)
    assert i2.status == i1.status
    assert i2.iterations == i1.iterations and i2.restarts == i1.restarts
    assert i1.applies == i1.iterations + i1.restarts + 1   # CGS2: x += B^-1 (V y) costs one apply per cycle
    assert i2.applies == i2.iterations                      # DCGS2: x += Z R^-1 y from the steps' own applies
    assert np.allclose(h2, h1, rtol=1e-7, atol=0)
    rel = float(torch.linalg.norm(x2 - x1) / torch.linalg.norm(x1))
    assert rel <= 1e-9
    assert abs(i2.relres_true - i1.relres_true) <= 1e-6 * i1.relres_true + 1e-15
    ctx.close()


def test_dcgs2_basis_is_orthonormal():
    """After a full cycle the device basis v_0 .. v_{m-1} is orthonormal to rounding (slot m keeps the candidate
    u_m, whose re-orthogonalisation only closes the last Hessenberg column)."""
    cfg = CONFIGS["c1"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    b = ctx.rhs(*sources(cfg))
    m = 20
    ctx.gmres(b, restart=m, rtol=0.0, maxit=m)
    V = ctx.krylov_basis(m)
    G = V.conj() @ V.T
    assert float(torch.linalg.norm(G - torch.eye(m, dtype=G.dtype, device=G.device))) <= 1e-12
    ctx.close()


def test_orthogonalisation_mode_errors():
    cfg = CONFIGS["c0"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    with pytest.raises(HelmError):
        ctx.set_orthogonalisation(7)
    ctx.close()
