"""D28 -- shared factors and the tensor-core apply (k_apply_batch) against the oracle.

Subdomains whose assembled local operators A_j are bitwise equal form a class; libhelm factors one
representative per class (the exact local solves need A_j^-1, identical for identical matrices) and, when
the classes are large, applies each class to 16 subdomains at a time as complex GEMMs on the FP64 tensor cores.  The
oracle finds its classes independently (orc_factor_dedup: hashes of its own matrices, memcmp against the
representative).  Here, at sizes the oracle runs in seconds and with ragged tiles (class sizes not multiples of 16,
block widths not multiples of 8):
  * the GPU's class partition equals the oracle's (bit-exact integer work);
  * the tensor-core apply, forced on (HELM_APPLY_BATCH=1), matches the oracle apply to 1e-10 and GMRES to +-1
    iteration / 1e-6 (the north_star tolerances), with the owner write, RAS-PML-Imp and the ramp PoU;
  * one factorisation per subdomain (HELM_SHARE_FACTORS=0, the general path) and the shared path agree to 1e-13.
-m gpu."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, gmres as orc_gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import BC_IMPEDANCE, POU_RAMP  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make(cfg, env=None, **kw):
    """A factored context built with the given HELM_* environment (read at helm_setup), restored afterwards."""
    env = env or {}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        ctx = Context(cfg.k, cfg.nsub, cfg.nsub, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ctx.factor()
    return ctx


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_class_partition_equals_the_oracle_dedup(name):
    cfg = CONFIGS[name]
    ctx = make(cfg)
    info = ctx.factor_classes(with_members=True)
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    nc = o.factor_dedup()
    assert info["classes"] == nc == 9   # 4 corners, 4 edges, 1 interior class (uniform interior blocks)
    pairs = {(info["class_of"][j], o.dedup_class(j)[0]) for j in range(cfg.nsub ** 2)}
    assert len(pairs) == nc
    assert len({p[0] for p in pairs}) == nc and len({p[1] for p in pairs}) == nc
    ctx.close()


CASES = [("c1", {}, {}), ("c2", {}, {"HELM_BATCH_SPLIT": "0", "HELM_BATCH_W": "16"}),
         ("c1", {"local_bc": BC_IMPEDANCE}, {}), ("c2", {"pou": POU_RAMP}, {}),
         ("c2", {}, {"HELM_BATCH_SPLIT": "1"}), ("c1", {"pou": POU_RAMP}, {"HELM_BATCH_SPLIT": "1"}),
         ("c2", {}, {"HELM_APPLY_BATCH": "0"}), ("c2", {"local_bc": BC_IMPEDANCE}, {"HELM_SHARE_FACTORS": "0"})]


@pytest.mark.parametrize("name,kw,env", CASES, ids=["c1", "c2-w16", "c1-imp", "c2-ramp", "c2-split", "c1-ramp-split",
                                                    "c2-streaming", "c2-imp-per-subdomain"])
def test_tensor_core_apply_and_gmres_vs_oracle(name, kw, env):
    """The tensor-core apply forced on (split: every tile on a cluster of two CTAs, the twisted halves swapping carries
    through DSMEM; w16: one CTA per 16-wide tile), and the streaming apply on shared / per-subdomain factors, against
    the oracle."""
    cfg = CONFIGS[name]
    env = {"HELM_APPLY_BATCH": "1", **env}
    ctx = make(cfg, env, **kw)
    info = ctx.factor_classes()
    batched = env["HELM_APPLY_BATCH"] == "1" and env.get("HELM_SHARE_FACTORS") != "0"
    assert info["batched"] == batched
    assert not batched or info["tiles"] >= info["classes"]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, **kw)
    o.factor()
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    assert rel(z, o.apply(v)) <= 1e-10
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    ref = orc_gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol)
    x, ginfo, _ = ctx.gmres(torch.from_numpy(b).cuda(), restart=cfg.restart, rtol=cfg.rtol)
    assert ginfo.status == 0 and ref.status == 0
    assert abs(ginfo.iterations - ref.iterations) <= 1
    assert rel(x.cpu().numpy(), ref.x) <= 1e-6
    ctx.close()


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_shared_and_per_subdomain_factors_agree(name):
    """The general path (every subdomain factored, HELM_SHARE_FACTORS=0) and the default shared path: the same
    inverses, so the streaming apply is bitwise equal, and the tensor-core apply agrees to rounding."""
    cfg = CONFIGS[name]
    per = make(cfg, {"HELM_SHARE_FACTORS": "0"})
    v = torch.from_numpy(probe_vector(per.n, int(cfg.k) + 1)).cuda()
    assert per.factor_classes()["classes"] == cfg.nsub ** 2
    shared = make(cfg, {"HELM_APPLY_BATCH": "0"})
    batch = make(cfg, {"HELM_APPLY_BATCH": "1"})
    z0 = per.precond_apply(v).cpu().numpy()
    z1 = shared.precond_apply(v).cpu().numpy()
    z2 = batch.precond_apply(v).cpu().numpy()
    assert np.array_equal(z0, z1)
    assert rel(z2, z0) <= 1e-13
    for c in (per, shared, batch):
        c.close()


@pytest.mark.parametrize("bc", [0, 1], ids=["drch", "imp"])
def test_tensor_core_apply_q1_paper_frame_vs_oracle(bc):
    """The paper's own discretisation (Q1, 9-point couplings with the NW / SE terms, D18; RAS-PML-Imp and the ramp PoU
    by default) through the tensor-core apply, forced on, against the oracle."""
    from paper_2602_00735_b200.helm import paper_params
    kw = paper_params(100.0, 3, 4, 2, local_bc=bc)
    old = os.environ.get("HELM_APPLY_BATCH")
    os.environ["HELM_APPLY_BATCH"] = "1"
    try:
        ctx = Context(**kw)
    finally:
        if old is None:
            del os.environ["HELM_APPLY_BATCH"]
        else:
            os.environ["HELM_APPLY_BATCH"] = old
    ctx.factor()
    assert ctx.layout.stencil_slots == 9 and ctx.factor_classes()["batched"]
    o = Oracle.from_paper(k=100.0, nsub=3, pml=4, ovlp=2, local_bc=bc, pou=kw["pou"])
    o.factor()
    v = probe_vector(o.nfree, 11)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    assert rel(z, o.apply(v)) <= 1e-10
    ctx.close()
