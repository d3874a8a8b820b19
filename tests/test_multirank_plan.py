"""Multi-rank host logic of libhelm (rank plan + two-phase halo schedule), checked on CPU: partition of the free
nodes, message pairing, coverage of every subdomain's full box, and the exchange itself executed over a gloo
process group (world size 2 and 4) on a synthetic global vector.  -m "not gpu"."""
import os
import socket

import numpy as np
import pytest

from oracle.oracle import Oracle
from paper_2602_00735_b200.helm import make_params, plan_rank, halo_schedule

CASES = [(100.0, 4, 2), (100.0, 4, 4), (400.0, 16, 2), (400.0, 16, 4), (400.0, 16, 8), (400.0, 16, 6),
         (1600.0, 64, 8), (100.0, 5, 3)]


@pytest.mark.parametrize("k,nsub,nranks", CASES)
def test_owned_rectangles_partition_the_free_nodes(k, nsub, nranks):
    p = make_params(k, nsub)
    plans = [plan_rank(p, r, nranks) for r in range(nranks)]
    nf = plans[0]["owned_i1"] if False else None
    o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub)
    nfx, nfy = o.nf
    cover = np.zeros((nfy + 2, nfx + 2), int)
    for pl in plans:
        cover[pl["owned_j0"]:pl["owned_j1"], pl["owned_i0"]:pl["owned_i1"]] += 1
        assert pl["gx"] * pl["gy"] == nranks
    assert np.all(cover[1:nfy + 1, 1:nfx + 1] == 1) and cover.sum() == nfx * nfy
    assert sum(pl["n_sub_local"] for pl in plans) == nsub * nsub


@pytest.mark.parametrize("k,nsub,nranks", CASES)
@pytest.mark.parametrize("bc", [0, 1])
def test_every_full_box_inside_its_ranks_ghost_frame(k, nsub, nranks, bc):
    """The ghost frame (delta + kappa - 1 below, delta + kappa above; one more each side for RAS-PML-Imp, whose
    face nodes are unknowns) is exactly what the edge subdomains' local unknowns need."""
    p = make_params(k, nsub, local_bc=bc)
    o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub, local_bc=bc)
    need = {r: [10 ** 9, -1, 10 ** 9, -1] for r in range(nranks)}
    plans = [plan_rank(p, r, nranks) for r in range(nranks)]
    for j in range(o.nsub):
        s = o.subdomain(j)
        gi, gj = max(s["own_lo"][0], 1), max(s["own_lo"][1], 1)
        r = next(q for q, pl in enumerate(plans) if pl["owned_i0"] <= gi < pl["owned_i1"] and pl["owned_j0"] <= gj < pl["owned_j1"])
        pl = plans[r]
        lo = s["node0"]
        hi = (s["node0"][0] + s["m"][0] - 1, s["node0"][1] + s["m"][1] - 1)
        assert pl["ext_i0"] <= lo[0] and hi[0] < pl["ext_i1"]
        assert pl["ext_j0"] <= lo[1] and hi[1] < pl["ext_j1"]
        n = need[r]
        n[0] = min(n[0], lo[0]); n[1] = max(n[1], hi[0])
        n[2] = min(n[2], lo[1]); n[3] = max(n[3], hi[1])
    for r, pl in enumerate(plans):   # and no wider than needed
        assert need[r] == [pl["ext_i0"], pl["ext_i1"] - 1, pl["ext_j0"], pl["ext_j1"] - 1]


@pytest.mark.parametrize("k,nsub,nranks", CASES)
@pytest.mark.parametrize("W", [0, 1])
def test_messages_pair_up(k, nsub, nranks, W):
    p = make_params(k, nsub)
    sched = {r: halo_schedule(p, r, nranks, W) for r in range(nranks)}
    for r, msgs in sched.items():
        for m in msgs:
            back = [q for q in sched[m["peer"]] if q["peer"] == r and q["phase"] == m["phase"]]
            assert len(back) == 1
            q = back[0]
            # what r sends is exactly what the peer receives, node for node
            assert (m["send_i0"], m["send_i1"], m["send_j0"], m["send_j1"]) == \
                   (q["recv_i0"], q["recv_i1"], q["recv_j0"], q["recv_j1"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, nranks, port, k, nsub, result_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        p = make_params(k, nsub)
        pl = plan_rank(p, rank, nranks)
        N = int(round(10 * k / (2 * np.pi))) + 20
        nf = N - 1
        gid = lambda i, j: (i - 1) + nf * (j - 1)   # noqa: E731  synthetic global vector value = index
        ok = True
        for W in (0, 1):
            lo, hi = (pl["halo_lo"], pl["halo_hi"]) if W == 0 else (W, W)
            e_i0, e_j0 = pl["ext_i0"], pl["ext_j0"]
            ew, eh = pl["ext_i1"] - e_i0, pl["ext_j1"] - e_j0
            buf = torch.full((eh, ew), -1.0, dtype=torch.float64)
            for j in range(pl["owned_j0"], pl["owned_j1"]):
                buf[j - e_j0, pl["owned_i0"] - e_i0:pl["owned_i1"] - e_i0] = torch.tensor(
                    [float(gid(i, j)) for i in range(pl["owned_i0"], pl["owned_i1"])])
            msgs = halo_schedule(p, rank, nranks, W)
            for phase in (0, 1):
                ops, recvs = [], []
                for m in msgs:
                    if m["phase"] != phase:
                        continue
                    send = buf[m["send_j0"] - e_j0:m["send_j1"] - e_j0, m["send_i0"] - e_i0:m["send_i1"] - e_i0].contiguous()
                    recv = torch.empty((m["recv_j1"] - m["recv_j0"], m["recv_i1"] - m["recv_i0"]), dtype=torch.float64)
                    ops.append(dist.P2POp(dist.isend, send, m["peer"]))
                    ops.append(dist.P2POp(dist.irecv, recv, m["peer"]))
                    recvs.append((m, recv))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                for m, recv in recvs:
                    buf[m["recv_j0"] - e_j0:m["recv_j1"] - e_j0, m["recv_i0"] - e_i0:m["recv_i1"] - e_i0] = recv
            # the (lo, hi) frame (incl. corners) must now hold the global values
            for j in range(pl["owned_j0"] - (lo if pl["nbr"][2] >= 0 else 0), pl["owned_j1"] + (hi if pl["nbr"][3] >= 0 else 0)):
                for i in range(pl["owned_i0"] - (lo if pl["nbr"][0] >= 0 else 0), pl["owned_i1"] + (hi if pl["nbr"][1] >= 0 else 0)):
                    if buf[j - e_j0, i - e_i0].item() != gid(i, j):
                        ok = False
        result_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 4])
def test_two_phase_exchange_over_gloo(nranks):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, nranks, port, 100.0, 4, q)) for r in range(nranks)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(nranks))
    for pr in procs:
        pr.join(timeout=60)
    assert all(res[r] for r in range(nranks)), res


@pytest.mark.parametrize("k,nsub,nranks", CASES)
@pytest.mark.parametrize("bc", [0, 1])
@pytest.mark.parametrize("W", [0, 1])
def test_exact_communication_counts(k, nsub, nranks, bc, W):
    """SURVEY 4.2 T3 (S:525 adapted): the elements a rank receives in one exchange equal the area of its ghost frame
    exactly -- the two phases neither miss nor double-count a node (corners arrive once, in phase 1) -- and every
    element sent is received."""
    p = make_params(k, nsub, local_bc=bc)
    sent = recv = 0
    for r in range(nranks):
        pl = plan_rank(p, r, nranks)
        lo, hi = (pl["halo_lo"], pl["halo_hi"]) if W == 0 else (W, W)
        nb = pl["nbr"]
        fw = (pl["owned_i1"] - pl["owned_i0"]) + (lo if nb[0] >= 0 else 0) + (hi if nb[1] >= 0 else 0)
        fh = (pl["owned_j1"] - pl["owned_j0"]) + (lo if nb[2] >= 0 else 0) + (hi if nb[3] >= 0 else 0)
        frame = fw * fh - (pl["owned_i1"] - pl["owned_i0"]) * (pl["owned_j1"] - pl["owned_j0"])
        msgs = halo_schedule(p, r, nranks, W)
        got = sum((m["recv_i1"] - m["recv_i0"]) * (m["recv_j1"] - m["recv_j0"]) for m in msgs)
        assert got == frame
        recv += got
        sent += sum((m["send_i1"] - m["send_i0"]) * (m["send_j1"] - m["send_j0"]) for m in msgs)
    assert sent == recv


@pytest.mark.parametrize("nranks,gg", [(2, (2, 1)), (4, (2, 2)), (8, (4, 2))])
def test_paper_frame_plans(nranks, gg):
    """The paper's Q1 frame (k = 600, grid 1200^2, 4 x 4 subdomains, pml 11 / ovlp 5, Imp): owned rectangles partition
    the free nodes and the ghost frames are covered exactly."""
    from paper_2602_00735_b200.helm import paper_params
    kw = paper_params(600.0, 4, 11, 5, gpu_grid=gg)
    p = make_params(kw["k"], 4, 4, n_ovlp=5, n_pml=11, gpu_grid=gg, local_bc=kw["local_bc"], pou=0, elem=kw["elem"],
                    n_cells=kw["n_cells"], kappa_g=kw["kappa_g"], pml_c=kw["pml_c"])
    nf = kw["n_cells"] - 1
    cover = np.zeros((nf + 2, nf + 2), int)
    for r in range(nranks):
        pl = plan_rank(p, r, nranks)
        cover[pl["owned_j0"]:pl["owned_j1"], pl["owned_i0"]:pl["owned_i1"]] += 1
        assert pl["halo_lo"] == 5 + 11 - 1 + 1 and pl["halo_hi"] == 5 + 11 + 1   # Imp: face nodes are unknowns
    assert np.all(cover[1:nf + 1, 1:nf + 1] == 1) and cover.sum() == nf * nf


def test_narrow_rank_strips_are_refused():
    """a rank sends halo_hi owned layers to its lower neighbour and halo_lo to its upper one, so its owned
    strip must be at least that wide.  k = 6 pi (N = 50 cells), 10 x 2 subdomains of 5 = delta + kappa cells, one rank
    per block column: with Dirichlet faces (halo 4 / 5; the edge ranks own 4 free nodes and send 4) the layout is
    valid; with impedance faces (halo 5 / 6) it is refused on every rank, as the oracle refuses it
    (tests/test_oracle_solvers.py).  Every accepted plan sends owned nodes only."""
    from paper_2602_00735_b200.helm import HelmError
    k = 6 * np.pi
    pimp = make_params(k, 10, 2, n_ovlp=2, n_pml=3, local_bc=1, gpu_grid=(10, 1))
    for r in range(10):
        with pytest.raises(HelmError):
            plan_rank(pimp, r, 10)
    pdir = make_params(k, 10, 2, n_ovlp=2, n_pml=3, local_bc=0, gpu_grid=(10, 1))
    for r in range(10):
        pl = plan_rank(pdir, r, 10)
        for m in halo_schedule(pdir, r, 10, 0):
            if m["phase"] == 0:
                assert pl["owned_i0"] <= m["send_i0"] and m["send_i1"] <= pl["owned_i1"]
    # five rank columns of two blocks (10 owned nodes >= 6): accepted
    pimp5 = make_params(k, 10, 2, n_ovlp=2, n_pml=3, local_bc=1, gpu_grid=(5, 1))
    for r in range(5):
        pl = plan_rank(pimp5, r, 5)
        assert pl["owned_i1"] - pl["owned_i0"] >= pl["halo_hi"]
    # every accepted plan sends only owned nodes (the schedule's send rectangles lie in the owned rectangle)
    for r in range(5):
        pl = plan_rank(pimp5, r, 5)
        for m in halo_schedule(pimp5, r, 5, 0):
            if m["phase"] == 0:
                assert pl["owned_i0"] <= m["send_i0"] and m["send_i1"] <= pl["owned_i1"]


# ------------------------------------------------------------------------------------------ section 3(i) band halo
def _band_sets(o):
    """Independent of libhelm: node indices whose stencil crosses a block boundary, per axis, from the oracle's
    ownership ranges (tests/test_oracle_richardson.py pins that the residual lives there)."""
    out = []
    for ax in (0, 1):
        starts = sorted({o.subdomain(j)["own_lo"][ax] for j in range(o.nsub)})
        out.append({v for s in starts[1:] for v in (s - 1, s)})
    return out


@pytest.mark.parametrize("k,nsub,nranks", CASES)
def test_band_halo_counts_equal_the_band_area(k, nsub, nranks):
    """Section 3(i): on the band exchange a rank receives exactly the band nodes of its ghost frame (ext rectangle minus
    owned rectangle, corners included), and everything sent is received."""
    from paper_2602_00735_b200.helm import halo_band_counts
    p = make_params(k, nsub)
    o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub)
    bx, by = _band_sets(o)
    tot_s = tot_r = full_r = 0
    for r in range(nranks):
        pl = plan_rank(p, r, nranks)
        c = halo_band_counts(p, r, nranks)
        area = 0
        for j in range(pl["ext_j0"], pl["ext_j1"]):
            for i in range(pl["ext_i0"], pl["ext_i1"]):
                own = pl["owned_i0"] <= i < pl["owned_i1"] and pl["owned_j0"] <= j < pl["owned_j1"]
                if not own and (i in bx or j in by):
                    area += 1
        assert c["recv_band"] == area, (r, c, area)
        assert c["recv_full"] == (pl["ext_i1"] - pl["ext_i0"]) * (pl["ext_j1"] - pl["ext_j0"]) - \
            (pl["owned_i1"] - pl["owned_i0"]) * (pl["owned_j1"] - pl["owned_j0"])
        tot_s += c["sent_band"]
        tot_r += c["recv_band"]
        full_r += c["recv_full"]
    assert tot_s == tot_r
    if nranks > 1:
        assert 0 < tot_r < full_r


@pytest.mark.parametrize("k,nsub,nranks", [(100.0, 4, 4), (400.0, 16, 8), (100.0, 5, 3)])
def test_band_rects_pair_up(k, nsub, nranks):
    """The sender's packing order (band sub-rectangles of its send rectangle) is the receiver's unpacking order."""
    from paper_2602_00735_b200.helm import halo_band_rects
    p = make_params(k, nsub)
    sched = {r: halo_schedule(p, r, nranks, 0) for r in range(nranks)}
    for r, msgs in sched.items():
        for q, m in enumerate(msgs):
            back = [t for t, x in enumerate(sched[m["peer"]]) if x["peer"] == r and x["phase"] == m["phase"]]
            assert len(back) == 1
            assert halo_band_rects(p, r, nranks, q, 0) == halo_band_rects(p, m["peer"], nranks, back[0], 1)


def _band_exchange_worker(rank, nranks, port, k, nsub, result_q):
    """The band exchange executed over gloo: every rank packs the band sub-rectangles of its send rectangles (libhelm's
    canonical order) from a synthetic global field, the peers unpack into a zeroed frame; afterwards the frame holds
    the global value at every band node and 0 elsewhere."""
    import torch
    import torch.distributed as dist

    from paper_2602_00735_b200.helm import halo_band_rects
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        p = make_params(k, nsub)
        pl = plan_rank(p, rank, nranks)
        o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub)
        bx, by = _band_sets(o)
        nf = o.nf[0]
        gid = lambda i, j: float((i - 1) + nf * (j - 1) + 1)   # noqa: E731
        e_i0, e_j0 = pl["ext_i0"], pl["ext_j0"]
        buf = torch.zeros((pl["ext_j1"] - e_j0, pl["ext_i1"] - e_i0), dtype=torch.float64)
        for j in range(pl["owned_j0"], pl["owned_j1"]):
            for i in range(pl["owned_i0"], pl["owned_i1"]):
                buf[j - e_j0, i - e_i0] = gid(i, j) if (i in bx or j in by) else 0.0   # the masked residual
        msgs = halo_schedule(p, rank, nranks, 0)
        for phase in (0, 1):
            ops, recvs = [], []
            for q, m in enumerate(msgs):
                if m["phase"] != phase:
                    continue
                srects = halo_band_rects(p, rank, nranks, q, 0)
                send = torch.cat([buf[j0 - e_j0:j1 - e_j0, i0 - e_i0:i1 - e_i0].reshape(-1)
                                  for i0, i1, j0, j1 in srects]) if srects else torch.zeros(0, dtype=torch.float64)
                rrects = halo_band_rects(p, rank, nranks, q, 1)
                recv = torch.empty(sum((i1 - i0) * (j1 - j0) for i0, i1, j0, j1 in rrects), dtype=torch.float64)
                ops.append(dist.P2POp(dist.isend, send.contiguous(), m["peer"]))
                ops.append(dist.P2POp(dist.irecv, recv, m["peer"]))
                recvs.append((rrects, recv))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for rrects, recv in recvs:
                off = 0
                for i0, i1, j0, j1 in rrects:
                    n = (i1 - i0) * (j1 - j0)
                    buf[j0 - e_j0:j1 - e_j0, i0 - e_i0:i1 - e_i0] = recv[off:off + n].view(j1 - j0, i1 - i0)
                    off += n
        ok = True
        for j in range(pl["ext_j0"], pl["ext_j1"]):
            for i in range(pl["ext_i0"], pl["ext_i1"]):
                want = gid(i, j) if (i in bx or j in by) else 0.0
                if buf[j - e_j0, i - e_i0].item() != want:
                    ok = False
        result_q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks,nsub", [(2, 4), (4, 5)])
def test_band_exchange_over_gloo(nranks, nsub):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_exchange_worker, args=(r, nranks, port, 100.0, nsub, q)) for r in range(nranks)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=240) for _ in range(nranks))
    for pr in procs:
        pr.join(timeout=60)
    assert all(res[r] for r in range(nranks)), res
