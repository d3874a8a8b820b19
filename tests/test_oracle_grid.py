"""Oracle pins: grid sizing and decomposition (O1, O2) against BASELINE.json's printed sizes and the
covering / PoU invariants of P:71-96.  -m "not gpu"."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError, Problem, problem_from_config, width_from
from paper_2602_00735_b200.workloads import CONFIGS

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bj_sizes.txt")


def _golden():
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        name, k, cells, unk, nsub, w = line.split()
        rows.append((name, float(k), cells, unk, int(nsub), int(w)))
    return rows


def _close(printed: str, value: float):
    if printed == "-":
        return True
    if printed.startswith("~"):
        return abs(value - float(printed[1:])) <= 0.025 * float(printed[1:])
    return value == float(printed)


@pytest.mark.parametrize("row", _golden(), ids=lambda r: r[0])
def test_sizes_match_baseline_json(row):
    name, k, cells, unk, nsub, w = row
    cfg = CONFIGS[name]
    assert cfg.k == k and cfg.nsub == nsub
    o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub)
    assert _close(cells, o.N[0]) and o.N[0] == o.N[1]
    assert _close(unk, o.nfree)
    assert width_from(k) == w
    assert o.prob.novlp == w and o.prob.npml == w


def test_c3_local_sizes():
    # BJ configs[3]: "~7.7k local unknowns, band ~ 88"; SURVEY D8 per-side overlap
    o = Oracle.from_config(k=1600, nsub_x=64, nsub_y=64)
    ms = set()
    nmax = 0
    for j in [0, 1, 2, 63, 64, 65, 64 * 32 + 17, 4095]:
        m = o.subdomain(j)["m"]
        ms.update(m)
        nmax = max(nmax, m[0] * m[1])
    assert ms <= {63, 64, 87, 88} and 88 in ms
    assert nmax == 7744


def test_c4_factor_bytes_per_subdomain():
    # BJ configs[4]: "complex128 factors (~25 MB per subdomain)"; band L+U = n * 2(mx+1) * 16 B
    o = Oracle.from_config(k=3200, nsub_x=128, nsub_y=128)
    m = o.subdomain(128 * 64 + 64)["m"]
    n = m[0] * m[1]
    mb = n * 2 * (m[0] + 1) * 16 / 1e6
    assert 23.0 < mb < 26.5


@pytest.mark.parametrize("px,py", [(1, 1), (2, 2), (3, 2), (4, 4), (5, 3)])
def test_owner_partition(px, py):
    """PoU = 0/1 owner indicator (D10): every free node owned exactly once, owned nodes inside the full
    box, full box inside Omega (P:95-96 supp chi_j subset Omega_j,int, sum chi_j = 1)."""
    o = Oracle.from_config(k=20, nsub_x=px, nsub_y=py)
    nfx, nfy = o.nf
    count = np.zeros((nfy + 2, nfx + 2), int)
    for j in range(o.nsub):
        s = o.subdomain(j)
        for ax in range(2):
            assert 0 <= s["full_lo"][ax] <= s["int_lo"][ax] <= s["own_lo"][ax]
            assert s["own_hi"][ax] <= s["int_hi"][ax] <= s["full_hi"][ax] <= o.N[ax]
            # owned free nodes strictly inside the full box (local free nodes)
            assert s["full_lo"][ax] < max(s["own_lo"][ax], 1)
            assert min(s["own_hi"][ax], o.N[ax]) - 1 < s["full_hi"][ax]
            # local PML only on faces not on dOmega
            assert s["has_lo"][ax] == (s["own_lo"][ax] > 0)
            assert s["has_hi"][ax] == (s["own_hi"][ax] < o.N[ax])
        count[s["own_lo"][1]:s["own_hi"][1], s["own_lo"][0]:s["own_hi"][0]] += 1
    assert np.all(count[1:nfy + 1, 1:nfx + 1] == 1)


def test_single_subdomain_is_omega():
    o = Oracle.from_config(k=20, nsub_x=1, nsub_y=1)
    s = o.subdomain(0)
    assert s["full_lo"] == (0, 0) and s["full_hi"] == o.N
    assert s["m"] == o.nf and s["has_lo"] == (0, 0) and s["has_hi"] == (0, 0)


def test_remainder_to_lowest_blocks():
    # c1: 179 cells into 4 blocks -> 45, 45, 45, 44 (S:83 remainder rule, D8)
    o = Oracle.from_config(k=100, nsub_x=4, nsub_y=4)
    sizes = [o.subdomain(j)["own_hi"][0] - o.subdomain(j)["own_lo"][0] for j in range(4)]
    assert sizes == [45, 45, 45, 44]


def test_layout_error_when_blocks_too_small():
    # delta + kappa = 10 cells per side but blocks of 52/8 = 6.5 cells: the extension would leave Omega
    with pytest.raises(OracleError):
        Oracle.from_config(k=20, nsub_x=8, nsub_y=8)
