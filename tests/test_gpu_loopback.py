"""The multi-rank code path executed on one GPU through libhelm's loopback transport (helm_setup_loopback): N rank
contexts in one process, each driven by its own thread and stream, run the collective entry points -- the halo
exchange of the apply input (width delta + kappa) and of the SpMV input (width 1, corners through the two-phase
schedule), the CGS2 / norm allreduces of GMRES, the residual norms of Richardson -- with the NCCL calls replaced by
device copies ordered by host barriers (no kernel waits on another).  Results must equal the single-rank run:
apply and matvec bitwise (no cross-rank reduction), GMRES / Richardson iterations equal and solutions to 1e-8 (the
inner products are summed in another order) -- and, assembled from the ranks' owned pieces, match the CPU oracle
directly at the north_star tolerances (apply <= 1e-10, matvec <= 1e-13, iterations +-1, x <= 1e-6).
SURVEY 8(e).  -m gpu."""
import itertools
import os
import threading

import numpy as np
import pytest

from oracle.oracle import Oracle, gmres as orc_gmres, richardson as orc_richardson
from paper_2602_00735_b200.workloads import CONFIGS, paper_source, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import BC_IMPEDANCE, POU_OWNER, POU_RAMP, paper_params  # noqa: E402

_gid = itertools.count(100)


def run_ranks(nranks, fn, timeout=300):
    """fn(rank) in one thread per rank; returns the results in rank order, re-raises the first error."""
    res, err = [None] * nranks, [None] * nranks

    def body(r):
        try:
            res[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    if any(t.is_alive() for t in th):
        errs = [f"rank {r}: {e!r}" for r, e in enumerate(err) if e is not None]
        pytest.fail("loopback ranks did not finish (deadlock?); errors on the others: " + "; ".join(errs))
    for e in err:
        if e is not None:
            raise e
    return res


def owned(vec2d, pl):
    return vec2d[pl["owned_j0"] - 1:pl["owned_j1"] - 1, pl["owned_i0"] - 1:pl["owned_i1"] - 1].contiguous().view(-1)


def oracle_for(kw):
    """The CPU oracle of the same problem as Context(**kw) (BJ frame or the paper frame)."""
    if kw.get("elem", 0) == 1:
        return Oracle.from_paper(k=kw["k"], nsub=kw["nsub_x"], pml=kw["n_pml"], ovlp=kw["n_ovlp"],
                                 local_bc=kw.get("local_bc", 1), pou=kw.get("pou", 1), n_cells=kw["n_cells"])
    return Oracle.from_config(k=kw["k"], nsub_x=kw["nsub_x"], nsub_y=kw["nsub_y"], local_bc=kw.get("local_bc", 0),
                              pou=kw.get("pou", 0))


def check_against_single_rank(kw, nranks, gg, b_of, restart=50, rtol=1e-6, bitwise=True, vs_oracle=True):
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 5)).cuda()
    b = b_of(ref)
    z_ref, y_ref = ref.precond_apply(v), ref.matvec(v)
    x_ref, gi_ref, _ = ref.gmres(b, restart=restart, rtol=rtol)
    xr_ref, ri_ref, _ = ref.richardson(b, rtol=rtol, maxit=200)
    ref.close()
    V, B = v.view(nf, nf), b.view(nf, nf)
    gid = next(_gid)
    torch.cuda.synchronize()

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**{**kw, "gpu_grid": gg}, rank=r, nranks=nranks, stream=s, loopback_group=gid)
            c.factor()
            pl = c.plan
            vl, bl = owned(V, pl), owned(B, pl)
            z, y = c.precond_apply(vl), c.matvec(vl)
            x, gi, _ = c.gmres(bl, restart=restart, rtol=rtol)
            xr, ri, _ = c.richardson(bl, rtol=rtol, maxit=200)
            s.synchronize()
            out = dict(pl=pl, z=z.clone(), y=y.clone(), x=x.clone(), xr=xr.clone(), gits=gi.iterations,
                       rits=ri.iterations, gstat=gi.status)
            c.close()
            return out

    outs = run_ranks(nranks, rank)
    Z, Y, X, XR = (torch.full_like(V, complex("nan")) for _ in range(4))
    for o in outs:
        pl = o["pl"]
        sl = (slice(pl["owned_j0"] - 1, pl["owned_j1"] - 1), slice(pl["owned_i0"] - 1, pl["owned_i1"] - 1))
        shape = (pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
        Z[sl], Y[sl] = o["z"].view(shape), o["y"].view(shape)
        X[sl], XR[sl] = o["x"].view(shape), o["xr"].view(shape)
    rel = lambda a, b: float(torch.linalg.norm(a - b) / torch.linalg.norm(b))  # noqa: E731
    if bitwise:
        assert torch.equal(Z.view(-1), z_ref) and torch.equal(Y.view(-1), y_ref)
    else:   # ramp PoU: sums over subdomains of two ranks are added in another order
        assert rel(Z.view(-1), z_ref) <= 1e-13 and torch.equal(Y.view(-1), y_ref)
    assert all(o["gstat"] == 0 for o in outs)
    assert len({o["gits"] for o in outs}) == 1 and abs(outs[0]["gits"] - gi_ref.iterations) <= 1
    assert len({o["rits"] for o in outs}) == 1 and outs[0]["rits"] == ri_ref.iterations
    assert rel(X.view(-1), x_ref) <= 1e-8 and rel(XR.view(-1), xr_ref) <= 1e-8
    if not vs_oracle:
        return
    # the assembled multi-rank results against the oracle itself (P:138-147 apply, P:58-62 matvec, P:240-242 GMRES,
    # P:102-128 Richardson)
    o = oracle_for(kw)
    o.factor()
    vn, bn = v.cpu().numpy(), b.cpu().numpy()
    zo, yo = o.apply(vn), o.matvec(vn)
    reln = lambda a, c: float(np.linalg.norm(a - c) / np.linalg.norm(c))  # noqa: E731
    assert reln(Z.view(-1).cpu().numpy(), zo) <= 1e-10
    assert reln(Y.view(-1).cpu().numpy(), yo) <= 1e-13
    go = orc_gmres(o.matvec, o.apply, bn, restart=restart, rtol=rtol)
    assert abs(outs[0]["gits"] - go.iterations) <= 1
    assert reln(X.view(-1).cpu().numpy(), go.x) <= max(1e-6, 100 * rtol)
    ro = orc_richardson(o.matvec, o.apply, bn, rtol=rtol, maxit=200)
    assert abs(outs[0]["rits"] - ro.iterations) <= 1
    assert reln(XR.view(-1).cpu().numpy(), ro.x) <= max(1e-6, 100 * rtol)


def bj_rhs(name):
    return lambda ctx: ctx.rhs(*sources(CONFIGS[name]))


@pytest.mark.parametrize("name,nranks,gg", [("c1", 2, (2, 1)), ("c1", 4, (2, 2)), ("c2", 4, (2, 2)), ("c2", 8, (4, 2)),
                                            ("c1", 3, (1, 3))])
def test_loopback_bj(name, nranks, gg):
    cfg = CONFIGS[name]
    check_against_single_rank(dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub), nranks, gg, bj_rhs(name))


def test_loopback_short_restart():
    """GMRES(5) on 4 ranks: every cycle closes its last Hessenberg column with an extra projection sweep (DCGS2) whose
    sums go through the allreduce too."""
    cfg = CONFIGS["c1"]
    check_against_single_rank(dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub), 4, (2, 2), bj_rhs("c1"), restart=5)


@pytest.mark.parametrize("overlap", ["1", "0"])
def test_loopback_apply_overlap(overlap, monkeypatch):
    """The apply overlapped with its halo exchange (interior subdomains on the library stream while the ghost frame
    is exchanged and the boundary subdomains run on the communication stream) and the serial form: both bitwise equal
    to one rank."""
    monkeypatch.setenv("HELM_APPLY_OVERLAP", overlap)
    cfg = CONFIGS["c2"]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    probe = Context(**kw, rank=0, nranks=4, gpu_grid=(2, 2), loopback_group=next(_gid))
    assert (probe.layout.overlap_interior > 0) == (overlap == "1")
    probe.close()
    check_against_single_rank(kw, 4, (2, 2), bj_rhs("c2"))


def test_loopback_impedance():
    cfg = CONFIGS["c1"]
    check_against_single_rank(dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, local_bc=BC_IMPEDANCE), 2, (2, 1),
                              bj_rhs("c1"))


def test_loopback_paper_q1():
    """Q1 (9-point SpMV: corner ghosts), cluster factorisation and cluster-split apply per rank."""
    kw = paper_params(150.0, 4, 6, 3, pou=POU_OWNER)
    check_against_single_rank(kw, 4, (2, 2), lambda ctx: ctx.rhs(*paper_source(150.0)), rtol=1e-10)


@pytest.mark.parametrize("name,nranks,gg,bc", [("c1", 2, (2, 1), 0), ("c1", 4, (2, 2), 1), ("c2", 8, (4, 2), 0)])
def test_loopback_ramp_pou(name, nranks, gg, bc):
    """The paper's linear-ramp PoU on several ranks: weighted contributions on each rank's ghost frame, the
    additive reverse two-phase exchange (corners in two hops), equal to the single-rank prolongation up to the order
    of the additions."""
    cfg = CONFIGS[name]
    check_against_single_rank(dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, pou=POU_RAMP, local_bc=bc), nranks, gg,
                              bj_rhs(name), bitwise=False)


def test_loopback_paper_q1_ramp():
    """The paper's own method (Q1, RAS-PML-Imp, linear ramps) across 4 ranks: the configuration Tables 1-4 run."""
    kw = paper_params(150.0, 4, 6, 3)
    check_against_single_rank(kw, 4, (2, 2), lambda ctx: ctx.rhs(*paper_source(150.0)), rtol=1e-10, bitwise=False)


def _loop_draws(n=8, seed=77):
    rng = np.random.default_rng(seed)
    grids = [(2, 1), (1, 2), (2, 2), (3, 1), (2, 3), (4, 1)]
    out = []
    for _ in range(n):
        gg = grids[int(rng.integers(0, len(grids)))]
        out.append(dict(k=float(rng.choice([50, 80, 120])), nsub_x=int(rng.integers(gg[0], 9)),
                        nsub_y=int(rng.integers(gg[1], 9)), gg=gg, local_bc=int(rng.integers(0, 2)),
                        pou=int(rng.integers(0, 2))))
    return out


@pytest.mark.parametrize("d", _loop_draws(), ids=lambda d: "-".join(f"{a}{b}" for a, b in d.items()))
def test_loopback_random_layouts(d):
    """Seeded random layouts and rank grids: the sharded apply (overlapped with its halo) and matvec against one rank
    -- bitwise for the owner write, to the order of the additions for the ramp PoU."""
    kw = dict(k=d["k"], nsub_x=d["nsub_x"], nsub_y=d["nsub_y"], local_bc=d["local_bc"], pou=d["pou"])
    gg = d["gg"]
    nranks = gg[0] * gg[1]
    if d["nsub_x"] < gg[0] or d["nsub_y"] < gg[1]:
        pytest.skip("fewer subdomains than ranks along an axis")
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 12)).cuda()
    z_ref, y_ref = ref.precond_apply(v), ref.matvec(v)
    ref.close()
    V = v.view(nf, nf)
    gid = next(_gid)
    torch.cuda.synchronize()

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**kw, gpu_grid=gg, rank=r, nranks=nranks, stream=s, loopback_group=gid)
            c.factor()
            pl = c.plan
            vl = owned(V, pl)
            z, y = c.precond_apply(vl), c.matvec(vl)
            s.synchronize()
            out = dict(pl=pl, z=z.clone(), y=y.clone())
            c.close()
            return out

    outs = run_ranks(nranks, rank)
    Z, Y = torch.full_like(V, complex("nan")), torch.full_like(V, complex("nan"))
    for o in outs:
        pl = o["pl"]
        sl = (slice(pl["owned_j0"] - 1, pl["owned_j1"] - 1), slice(pl["owned_i0"] - 1, pl["owned_i1"] - 1))
        shape = (pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
        Z[sl], Y[sl] = o["z"].view(shape), o["y"].view(shape)
    assert torch.equal(Y.view(-1), y_ref)
    if d["pou"] == 0:
        assert torch.equal(Z.view(-1), z_ref)
    else:
        assert float(torch.linalg.norm(Z.view(-1) - z_ref) / torch.linalg.norm(z_ref)) <= 1e-13
    o = oracle_for(kw)
    o.factor()
    vn = v.cpu().numpy()
    zo, yo = o.apply(vn), o.matvec(vn)
    assert np.linalg.norm(Z.view(-1).cpu().numpy() - zo) <= 1e-10 * np.linalg.norm(zo)
    assert np.linalg.norm(Y.view(-1).cpu().numpy() - yo) <= 1e-13 * np.linalg.norm(yo)


@pytest.mark.parametrize("gg", [(2, 1), (2, 2)])
def test_loopback_c3_full_size(gg):
    """BASELINE.json's headline config at full size on two and four ranks (all on this GPU): the
    overlapped sharded apply bitwise equal to one rank on a probe vector, and GMRES(50) to 1e-6 -- DCGS2 with the
    multi-rank lookahead, packed allreduces, the two-phase halos -- in the single-rank iteration count +-1."""
    cfg = CONFIGS["c3"]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 3)).cuda()
    z_ref = ref.precond_apply(v)
    b = ref.rhs(*sources(cfg))
    _, gi_ref, _ = ref.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=1000)
    ref.close()
    del ref
    torch.cuda.empty_cache()
    V, B = v.view(nf, nf), b.view(nf, nf)
    gid = next(_gid)
    torch.cuda.synchronize()

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**kw, gpu_grid=gg, rank=r, nranks=gg[0] * gg[1], stream=s, loopback_group=gid)
            c.factor()
            pl = c.plan
            z = c.precond_apply(owned(V, pl))
            x, gi, _ = c.gmres(owned(B, pl), restart=cfg.restart, rtol=cfg.rtol, maxit=1000)
            s.synchronize()
            out = dict(pl=pl, z=z.clone(), x=x.clone(), its=gi.iterations, status=gi.status, rr=gi.relres_true,
                       ov=c.layout.overlap_interior)
            c.close()
            return out

    outs = run_ranks(gg[0] * gg[1], rank, timeout=900)
    Z = torch.full_like(V, complex("nan"))
    X = torch.full_like(V, complex("nan"))
    for o in outs:
        pl = o["pl"]
        sl = (slice(pl["owned_j0"] - 1, pl["owned_j1"] - 1), slice(pl["owned_i0"] - 1, pl["owned_i1"] - 1))
        Z[sl] = o["z"].view(pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
        X[sl] = o["x"].view(pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
    assert torch.equal(Z.view(-1), z_ref)
    assert all(o["ov"] > 0 for o in outs)   # the overlapped apply ran
    assert all(o["status"] == 0 and o["rr"] <= cfg.rtol for o in outs)
    assert len({o["its"] for o in outs}) == 1 and abs(outs[0]["its"] - gi_ref.iterations) <= 1
    # against the oracle directly: the subdomains on both sides of every rank boundary, solved one by one by the
    # oracle, and the assembled solution against the oracle-only golden record (scripts/make_golden.py)
    from golden_util import golden_path, load_golden, sketch_rel
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    P = cfg.nsub
    subs = sorted({P // 2 - 1 + P * 5, P // 2 + P * 5, 3 + P * (P // 2 - 1), 3 + P * (P // 2), P // 2 + P * (P // 2),
                   P // 2 - 1 + P * (P // 2 - 1)})
    o.factor(subs)
    vn = v.cpu().numpy()
    zo = o.apply(vn, subs=subs)
    zg = Z.view(-1).cpu().numpy()
    for j in subs:
        d = o.subdomain(j)
        rows = [(gi - 1) + (nf) * (gj - 1) for gj in range(max(d["own_lo"][1], 1), d["own_hi"][1])
                for gi in range(max(d["own_lo"][0], 1), d["own_hi"][0])]
        assert np.linalg.norm(zg[rows] - zo[rows]) <= 1e-10 * np.linalg.norm(zo[rows])
    if os.path.exists(golden_path("c3")):
        g = load_golden("c3")
        assert abs(outs[0]["its"] - g["iterations"]) <= 1
        assert sketch_rel(X.view(-1).cpu().numpy(), g) <= 1e-6


@pytest.mark.parametrize("name,nranks,gg,bc", [("c1", 4, (2, 2), 0), ("c2", 8, (4, 2), 0), ("c1", 4, (2, 2), 1)])
def test_loopback_richardson_residual_band(name, nranks, gg, bc):
    """Section 3(i): Richardson restricting its residual to the interface band and exchanging only the band
    part of the apply's ghost frame.  Exact counts: every apply after the first receives exactly the band area of the
    ghost frame (helm_halo_band_counts), the first one the full frame, each residual the width-1 frame.  The solution
    is bitwise the single-rank band run's, the iteration count the oracle's full-residual Algorithm 1's, x within 1e-8
    of it; the full-frame run (band off) agrees to the same tolerance."""
    from oracle.oracle import richardson as orc_rich
    from paper_2602_00735_b200.helm import halo_band_counts, halo_schedule, make_params
    cfg = CONFIGS[name]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, local_bc=bc)
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    b = ref.rhs(*sources(cfg))
    x1, i1, _ = ref.richardson(b, rtol=cfg.rtol, maxit=300)
    ref.set_residual_band(False)
    x1f, i1f, _ = ref.richardson(b, rtol=cfg.rtol, maxit=300)
    ref.close()
    B = b.view(nf, nf)
    p = make_params(cfg.k, cfg.nsub, gpu_grid=gg, local_bc=bc)
    gid = next(_gid)
    torch.cuda.synchronize()

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**kw, gpu_grid=gg, rank=r, nranks=nranks, stream=s, loopback_group=gid)
            c.factor()
            pl = c.plan
            bl = owned(B, pl)
            c.comm_counters(reset=True)
            x, inf, _ = c.richardson(bl, rtol=cfg.rtol, maxit=300)
            cnt = c.comm_counters(reset=True)
            c.set_residual_band(False)
            xf, inff, _ = c.richardson(bl, rtol=cfg.rtol, maxit=300)
            cntf = c.comm_counters(reset=True)
            s.synchronize()
            out = dict(pl=pl, x=x.clone(), xf=xf.clone(), its=inf.iterations, itsf=inff.iterations, cnt=cnt,
                       cntf=cntf)
            c.close()
            return out

    outs = run_ranks(nranks, rank)
    X = torch.full_like(B, complex("nan"))
    XF = torch.full_like(B, complex("nan"))
    for q, o in enumerate(outs):
        pl = o["pl"]
        sl = (slice(pl["owned_j0"] - 1, pl["owned_j1"] - 1), slice(pl["owned_i0"] - 1, pl["owned_i1"] - 1))
        shape = (pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
        X[sl], XF[sl] = o["x"].view(shape), o["xf"].view(shape)
        its = o["its"]
        hb = halo_band_counts(p, q, nranks)
        w1 = sum((m["recv_i1"] - m["recv_i0"]) * (m["recv_j1"] - m["recv_j0"]) for m in halo_schedule(p, q, nranks, 1))
        # norm(b) has no exchange; residuals: initial + one per step (width 1); applies: first full, then band
        assert o["cnt"]["recv"] == hb["recv_full"] + (its - 1) * hb["recv_band"] + (its + 1) * w1, (q, o["cnt"], hb)
        assert o["cntf"]["recv"] == o["itsf"] * hb["recv_full"] + (o["itsf"] + 1) * w1
        assert hb["recv_band"] < hb["recv_full"]
    assert len({o["its"] for o in outs}) == 1 and abs(outs[0]["its"] - i1.iterations) <= 1   # (norms summed in
    if outs[0]["its"] == i1.iterations:                                                        # another order)
        assert torch.equal(X.view(-1), x1)                 # bitwise the single-rank band run
    rel = lambda a, c: float(torch.linalg.norm(a - c) / torch.linalg.norm(c))  # noqa: E731
    assert rel(XF.view(-1), x1f) <= 1e-8 and rel(X.view(-1), XF.view(-1)) <= 1e-8
    o = oracle_for(kw)
    o.factor()
    bn = b.cpu().numpy()
    ro = orc_rich(o.matvec, o.apply, bn, rtol=cfg.rtol, maxit=300)
    assert abs(outs[0]["its"] - ro.iterations) <= 1 and i1f.iterations == ro.iterations
    assert np.linalg.norm(X.view(-1).cpu().numpy() - ro.x) <= 1e-8 * np.linalg.norm(ro.x)


@pytest.mark.parametrize("fold", ["1", "0"])
def test_loopback_gmres_collectives_per_step(fold, monkeypatch):
    """Several ranks: with the folded norm (default) an Arnoldi step issues ONE allreduce (the packed projection sums);
    unfolded, two (plus the norm).  Both give the single-rank iteration count +-1 and its solution to 1e-8, and the
    oracle's count +-1; the SpMV of every step overlaps its width-1 halo with the interior rows (bitwise: matvec
    equals one rank in test_loopback_bj)."""
    monkeypatch.setenv("HELM_GMRES_FOLD", fold)
    cfg = CONFIGS["c2"]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    b = ref.rhs(*sources(cfg))
    x_ref, gi_ref, _ = ref.gmres(b, restart=cfg.restart, rtol=cfg.rtol)
    ref.close()
    B = b.view(nf, nf)
    gid = next(_gid)
    torch.cuda.synchronize()

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**kw, gpu_grid=(2, 2), rank=r, nranks=4, stream=s, loopback_group=gid)
            c.factor()
            pl = c.plan
            c.comm_counters(reset=True)
            x, gi, _ = c.gmres(owned(B, pl), restart=cfg.restart, rtol=cfg.rtol)
            cnt = c.comm_counters(reset=True)
            s.synchronize()
            out = dict(pl=pl, x=x.clone(), its=gi.iterations, applies=gi.applies, restarts=gi.restarts, cnt=cnt)
            c.close()
            return out

    outs = run_ranks(4, rank)
    X = torch.full_like(B, complex("nan"))
    for o in outs:
        pl = o["pl"]
        X[pl["owned_j0"] - 1:pl["owned_j1"] - 1, pl["owned_i0"] - 1:pl["owned_i1"] - 1] = o["x"].view(
            pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
    its = outs[0]["its"]
    assert abs(its - gi_ref.iterations) <= 1
    tol = 1e-8 if its == gi_ref.iterations else 1e-6
    assert float(torch.linalg.norm(X.view(-1) - x_ref) / torch.linalg.norm(x_ref)) <= tol
    steps = outs[0]["applies"]                      # Arnoldi steps issued, discarded lookahead steps included
    cycles = outs[0]["restarts"] + 1
    # per step: the packed projection allreduce (+ the norm unfolded); per cycle: ||b||, ||r|| (residual), closing
    # projection; once: ||b|| for beta0
    per_step = 1 if fold == "1" else 2
    ar = outs[0]["cnt"]["allreduces"]
    assert steps * per_step <= ar <= steps * per_step + 3 * cycles + 2, (ar, steps, cycles)


def test_loopback_failed_rank_aborts_the_group():
    """A collective entry point that fails on one rank (here: invalid restart) aborts the loopback group: its peer
    leaves the collective with HELM_ENCCL at once instead of waiting for a rank that never arrives."""
    from paper_2602_00735_b200 import HelmError
    cfg = CONFIGS["c1"]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    gid = next(_gid)

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            c = Context(**kw, gpu_grid=(2, 1), rank=r, nranks=2, stream=s, loopback_group=gid)
            c.factor()
            b = torch.ones(c.n, dtype=torch.complex128, device="cuda")
            try:
                c.gmres(b, restart=0 if r == 0 else 50, rtol=1e-6)
                return None
            except HelmError as e:
                return e.code
            finally:
                s.synchronize()
                c.close()

    codes = run_ranks(2, rank, timeout=120)
    assert codes[0] == -1 and codes[1] == -4, codes
