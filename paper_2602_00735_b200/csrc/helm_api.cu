// helm_api.cu -- host side of libhelm: the C ABI of include/helm.h, grid / decomposition / rank plan, device
// memory, the NCCL halo exchange, and the restarted GMRES driver.  Every arithmetic step on vectors runs in
// this library's kernels; the host only sizes the problem, launches, and performs the O(restart^2) Givens /
// triangular-solve bookkeeping of GMRES on at most restart+1 scalars per iteration (D13).
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <complex>
#include <condition_variable>
#include <map>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

void raise_smem_attr(const void* fn, int smem, bool nonportable)
{
    static std::mutex mu;
    static std::map<const void*, int> cur;
    std::lock_guard<std::mutex> lk(mu);
    int& c = cur[fn];
    if (smem > c) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        c = smem;
    }
    if (nonportable) cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

// NVTX ranges (host-side, zero cost without a tool attached): setup, factor, apply, spmv, gmres, orth, comm
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

#ifdef HELM_HAVE_NCCL
#include <nccl.h>
#endif

typedef std::complex<double> cplx;

namespace {

constexpr int NVMAX = 64;
constexpr int M_LIMIT = 992;   // apply CTA: one consumer thread per block row entry, <= 31 consumer warps

int round_half_up(double x) { return (int)floor(x + 0.5); }

// Cartesian block starts: N cells into P blocks of floor/ceil size, larger blocks first (D8)
std::vector<int> block_starts(int N, int P)
{
    std::vector<int> s(P + 1, 0);
    const int q = N / P, r = N % P;
    for (int b = 0; b < P; b++) s[b + 1] = s[b] + q + (b < r ? 1 : 0);
    return s;
}

// Grid (O1/D2), covering (P:71-84/D8) and this rank's place in the rank grid -- pure host logic.
struct GridInfo {
    int n_int = 0, N = 0, nf = 0, ng = 0, wo = 0, wp = 0;
    double h = 0;
    int frame = 0, ns = 7;                    // paper frame (D19); stencil slots (7 P1, 9 Q1)
    double lo_u = 0, hi_u = 0;                // Omega_int in cell units (node 0 at 0)
    int P[2] = {1, 1};
    std::vector<int> st[2];
    int gx = 1, gy = 1, rx = 0, ry = 0;
    int bx0 = 0, bx1 = 0, by0 = 0, by1 = 0;
    int i0 = 1, i1 = 1, j0 = 1, j1 = 1;       // owned free nodes
    int halo_lo = 0, halo_hi = 0;             // ghost nodes below / above: delta + kappa - 1, delta + kappa
    int nbr[4] = {-1, -1, -1, -1};            // -x, +x, -y, +y
    int e_i0 = 1, e_i1 = 1, e_j0 = 1, e_j1 = 1;   // ext rectangle (apply input)
};

int compute_grid(const helm_params& p, int rank, int nranks, GridInfo& G, char* err, size_t errlen)
{
    if (!(p.k > 0) || p.nsub_x < 1 || p.nsub_y < 1 || p.sigma0 < 0) {
        snprintf(err, errlen, "invalid parameters (k, nsub, sigma0)");
        return HELM_EINVAL;
    }
    if (p.local_bc != HELM_BC_DIRICHLET && p.local_bc != HELM_BC_IMPEDANCE) {
        snprintf(err, errlen, "local_bc must be HELM_BC_DIRICHLET or HELM_BC_IMPEDANCE");
        return HELM_EINVAL;
    }
    if (nranks < 1 || rank < 0 || rank >= nranks) {
        snprintf(err, errlen, "bad rank %d / %d", rank, nranks);
        return HELM_EINVAL;
    }
    if (p.elem != HELM_ELEM_P1 && p.elem != HELM_ELEM_Q1) {
        snprintf(err, errlen, "elem must be HELM_ELEM_P1 or HELM_ELEM_Q1");
        return HELM_EINVAL;
    }
    G.ns = p.elem == HELM_ELEM_Q1 ? 9 : 7;
    if (p.n_cells > 0) {
        // paper frame (D19): Omega = (0,1)^2 is n_cells^2 cells, Omega_int = (kappa_g, 1 - kappa_g)^2
        if (p.elem != HELM_ELEM_Q1 || !(p.kappa_g >= 0.0) || !(2.0 * p.kappa_g < 1.0) || !(p.pml_c >= 0.0)) {
            snprintf(err, errlen, "paper frame needs Q1, 0 <= kappa_g < 1/2 and pml_c >= 0");
            return HELM_EINVAL;
        }
        G.frame = 1;
        G.N = G.n_int = p.n_cells;
        G.h = 1.0 / G.N;
        G.ng = 0;
        G.nf = G.N - 1;
        G.lo_u = p.kappa_g / G.h;
        G.hi_u = (double)G.N - G.lo_u;
    } else {
        // O1 / D2: n_int = round(ppw k / 2 pi) cells on (0,1), h = 1 / n_int, N = n_int + 2 n_g
        if (p.ppw < 1 || p.n_pml_global < 1) {
            snprintf(err, errlen, "invalid parameters (ppw, n_pml_global)");
            return HELM_EINVAL;
        }
        G.n_int = round_half_up(p.ppw * p.k / (2.0 * M_PI));
        if (G.n_int < 1) {
            snprintf(err, errlen, "k * ppw too small: no interior cell");
            return HELM_EINVAL;
        }
        G.h = 1.0 / G.n_int;
        G.ng = p.n_pml_global;
        G.N = G.n_int + 2 * G.ng;
        G.nf = G.N - 1;
        G.lo_u = G.ng;
        G.hi_u = G.N - G.ng;
    }
    // BJ configs[0]: delta = kappa = max(2, round(1.59 ln k)) cells unless given
    const int wdef = std::max(2, round_half_up(1.59 * log(p.k)));
    G.wo = p.n_ovlp < 0 ? wdef : p.n_ovlp;
    G.wp = p.n_pml < 0 ? wdef : p.n_pml;
    G.P[0] = p.nsub_x;
    G.P[1] = p.nsub_y;
    G.st[0] = block_starts(G.N, G.P[0]);
    G.st[1] = block_starts(G.N, G.P[1]);
    const int w = G.wo + G.wp;
    for (int ax = 0; ax < 2; ax++)
        for (int b = 0; b < G.P[ax]; b++) {
            const int sz = G.st[ax][b + 1] - G.st[ax][b];
            if (sz < 2 || (G.P[ax] > 1 && sz < w)) {
                snprintf(err, errlen, "block %d on axis %d has %d cells; needs >= delta + kappa = %d (and >= 2)", b, ax,
                         sz, w);
                return HELM_ELAYOUT;
            }
            if (p.pou == HELM_POU_RAMP && G.P[ax] > 1 && sz < 2 * G.wo) {
                snprintf(err, errlen, "ramp PoU: block %d on axis %d has %d cells < 2 delta = %d", b, ax, sz, 2 * G.wo);
                return HELM_ELAYOUT;
            }
        }
    if (p.pou != HELM_POU_OWNER && p.pou != HELM_POU_RAMP) {
        snprintf(err, errlen, "pou must be HELM_POU_OWNER or HELM_POU_RAMP");
        return HELM_EINVAL;
    }
    if (p.pou == HELM_POU_RAMP && G.wo < 1) {
        snprintf(err, errlen, "ramp PoU needs delta >= 1");
        return HELM_EINVAL;
    }
    // rank grid: default = most square factorisation with gx >= gy
    int gx = p.gpu_grid_x, gy = p.gpu_grid_y;
    if (gx <= 0 || gy <= 0) {
        gy = 1;
        for (int d = 1; d * d <= nranks; d++)
            if (nranks % d == 0) gy = d;
        gx = nranks / gy;
        if (gx > G.P[0] && gy <= G.P[0] && gx <= G.P[1]) std::swap(gx, gy);
    }
    if (gx * gy != nranks || gx > G.P[0] || gy > G.P[1]) {
        snprintf(err, errlen, "gpu grid %dx%d does not match %d ranks / %dx%d subdomains", gx, gy, nranks, G.P[0], G.P[1]);
        return HELM_EINVAL;
    }
    G.gx = gx;
    G.gy = gy;
    G.rx = rank % gx;
    G.ry = rank / gx;
    const std::vector<int> sbx = block_starts(G.P[0], gx), sby = block_starts(G.P[1], gy);
    G.bx0 = sbx[G.rx];
    G.bx1 = sbx[G.rx + 1];
    G.by0 = sby[G.ry];
    G.by1 = sby[G.ry + 1];
    // owned free nodes of this rank: union of its blocks' owned nodes (D10)
    G.i0 = std::max(G.st[0][G.bx0], 1);
    G.i1 = std::min(G.st[0][G.bx1], G.N);
    G.j0 = std::max(G.st[1][G.by0], 1);
    G.j1 = std::min(G.st[1][G.by1], G.N);
    // the full box of a block's subdomain spans nodes s_p - w + 1 .. s_{p+1} + w - 1 while the block owns
    // s_p .. s_{p+1} - 1 (half-open ownership, D10): w - 1 ghost nodes below, w above
    // (with the impedance variant the face nodes themselves are unknowns: one more on each side)
    const int imp = p.local_bc == HELM_BC_IMPEDANCE;
    G.halo_lo = w - 1 + imp;
    G.halo_hi = w + imp;
    G.nbr[0] = G.rx > 0 ? rank - 1 : -1;
    G.nbr[1] = G.rx < gx - 1 ? rank + 1 : -1;
    G.nbr[2] = G.ry > 0 ? rank - gx : -1;
    G.nbr[3] = G.ry < gy - 1 ? rank + gx : -1;
    // every rank's owned strip must be at least as wide as the ghost layers it sends: halo_hi owned layers to the
    // lower neighbour and halo_lo to the upper one, never reaching past its own nodes (impedance makes the frame
    // delta + kappa + 1 wide, one more than a block needs to be).  Checked for all ranks, so every rank
    // accepts or refuses the same layout.
    for (int ax = 0; ax < 2; ax++) {
        const int g = ax ? gy : gx;
        if (g < 2) continue;
        const std::vector<int> sb = block_starts(G.P[ax], g);
        for (int q = 0; q < g; q++) {
            const int lo = std::max(G.st[ax][sb[q]], 1), hi = std::min(G.st[ax][sb[q + 1]], G.N);
            const int need = std::max(q > 0 ? G.halo_hi : 0, q < g - 1 ? G.halo_lo : 0);
            if (hi - lo < need) {
                snprintf(err, errlen, "rank strip %d on axis %d owns %d nodes < the %d ghost layers it must send", q,
                         ax, hi - lo, need);
                return HELM_ELAYOUT;
            }
        }
    }
    G.e_i0 = G.i0 - (G.nbr[0] >= 0 ? G.halo_lo : 0);
    G.e_i1 = G.i1 + (G.nbr[1] >= 0 ? G.halo_hi : 0);
    G.e_j0 = G.j0 - (G.nbr[2] >= 0 ? G.halo_lo : 0);
    G.e_j1 = G.j1 + (G.nbr[3] >= 0 ? G.halo_hi : 0);
    return HELM_OK;
}

// Two-phase halo exchange filling lo ghost layers below and hi above the owned rectangle (x first, then y
// over the x-extended range, which carries the corners).  width 0 = the apply frame (halo_lo, halo_hi),
// width W > 0 = W layers on both sides.  A message's send and receive rectangles may differ in shape: a
// rank sends `hi` layers down (the lower neighbour's upper ghosts) and receives `lo` layers from below.
int halo_schedule(const GridInfo& G, int width, helm_msg* out, int cap)
{
    int lo, hi;
    if (width == 0) {
        lo = G.halo_lo;
        hi = G.halo_hi;
    } else {
        lo = hi = width;
    }
    if (width < 0 || lo < 0 || hi < 1 || hi > G.halo_hi) return HELM_EINVAL;
    int n = 0;
    auto add = [&](int phase, int peer, int s0, int s1, int t0, int t1, int r0, int r1, int q0, int q1) {
        if (n < cap) out[n] = helm_msg{phase, peer, s0, s1, t0, t1, r0, r1, q0, q1};
        n++;
    };
    if (G.nbr[0] >= 0) add(0, G.nbr[0], G.i0, G.i0 + hi, G.j0, G.j1, G.i0 - lo, G.i0, G.j0, G.j1);
    if (G.nbr[1] >= 0) add(0, G.nbr[1], G.i1 - lo, G.i1, G.j0, G.j1, G.i1, G.i1 + hi, G.j0, G.j1);
    const int x0 = G.i0 - (G.nbr[0] >= 0 ? lo : 0), x1 = G.i1 + (G.nbr[1] >= 0 ? hi : 0);
    if (G.nbr[2] >= 0) add(1, G.nbr[2], x0, x1, G.j0, G.j0 + hi, x0, x1, G.j0 - lo, G.j0);
    if (G.nbr[3] >= 0) add(1, G.nbr[3], x0, x1, G.j1 - lo, G.j1, x0, x1, G.j1, G.j1 + hi);
    return n;
}

// Section 3(i): "the right-hand side of eq. (local-ras-discrete) is nonzero only in overlapping regions, and
// thus the communication of the local residuals can be restricted to these regions".  With the restricted owner write
// the residual b - A u after a RAS step vanishes at every node whose stencil stays inside its own block (a_j = a there
// and the local solve satisfied the equation), i.e. outside the interface band: node indices s_p - 1 and s_p of every
// interior block boundary s_p, per axis (tests/test_oracle_richardson.py pins this on the oracle).
std::vector<unsigned char> band_flags(const GridInfo& G, int ax)
{
    std::vector<unsigned char> f(G.N + 1, 0);
    for (int p = 1; p < G.P[ax]; p++) {
        const int b = G.st[ax][p];
        if (b - 1 >= 0) f[b - 1] = 1;
        if (b <= G.N) f[b] = 1;
    }
    return f;
}

// Canonical decomposition of the band nodes of the rectangle [i0,i1) x [j0,j1) into disjoint sub-rectangles: row
// ranges in increasing j -- a run of band rows is one full-width rectangle, a run of other rows contributes its runs of
// band columns in increasing i.  Sender and receiver of a message decompose the same global rectangle, so their packing
// orders agree.
void band_rects(const std::vector<unsigned char>& bx, const std::vector<unsigned char>& by, int i0, int i1, int j0,
                int j1, std::vector<int4>& out)
{
    int j = j0;
    while (j < j1) {
        int je = j;
        const unsigned char t = by[j];
        while (je < j1 && by[je] == t) je++;
        if (t) {
            out.push_back(make_int4(i0, i1, j, je));
        } else {
            for (int i = i0; i < i1;) {
                if (!bx[i]) {
                    i++;
                    continue;
                }
                int ie = i;
                while (ie < i1 && bx[ie]) ie++;
                out.push_back(make_int4(i, ie, j, je));
                i = ie;
            }
        }
        j = je;
    }
}

long long rects_area(const std::vector<int4>& r)
{
    long long a = 0;
    for (const int4& q : r) a += (long long)(q.y - q.x) * (q.w - q.z);
    return a;
}

// In-process loopback transport (helm_setup_loopback): the ranks of a group are contexts in one process, each driven
// by its own host thread and stream on the same device.  Halo messages and allreduces go through device-to-device
// copies between the contexts' buffers, ordered by host barriers -- no kernel ever waits on another.  It executes the
// whole multi-rank code path (packing, schedules, ghost frames, reductions) except the NCCL calls themselves.
struct LoopGroup {
    int nranks = 0, members = 0;
    std::vector<struct helm_ctx*> ctx;
    std::vector<const double*> slot;   // buffer each rank contributes to the current allreduce
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    bool aborted = false;   // a rank failed inside a collective call: the others leave their barriers with an error
    // false if the group was aborted (a failed rank would otherwise leave its peers waiting forever)
    bool barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) return false;
        const long g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || aborted; });
        }
        return !aborted;
    }
    void abort()
    {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};
std::mutex g_loop_mu;
std::map<int, LoopGroup*> g_loops;

}  // namespace

struct helm_ctx {
    helm_params p{};
    int rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;
    char err[512] = {0};

    GridInfo G;
    Geom geom{};
    long long n_local = 0;

    // subdomains held by this rank
    std::vector<SubDesc> subs;
    int m_max = 0;
    long long max_n = 0, local_unknowns = 0, n_dinv = 0, n_stc = 0;
    long long apply_bytes = 0, band_bytes = 0;
    SubDesc* d_desc = nullptr;
    int* d_order = nullptr;
    z2* d_A7 = nullptr;
    z2* d_stc = nullptr;
    z2* d_dinv = nullptr;
    z2* d_scratch = nullptr;
    long long scratch_per_cta = 0;
    int* d_err = nullptr;
    bool factored = false;

    // apply launch configuration
    int ap_block = 0, ap_smem = 0, ap_slot = 0, ap_grid = 0, ap_occ = 0, ap_nslots = 2;   // ring depth: apply.cu
    // cluster-split apply (few large subdomains): G CTAs per chain, 2G per cluster; 0 = off
    int sp_G = 0, sp_block = 0, sp_smem = 0, sp_slot = 0, sp_ncw = 0, sp_nss = 0;

    // ramp partition of unity: weighted local solutions + per-axis covering blocks
    long long pou_len = 0;
    z2* d_pou = nullptr;
    z2* d_cext = nullptr;   // multi-rank ramp PoU: weighted contributions on the ghost-framed rectangle
    int* d_candx = nullptr;
    int* d_candy = nullptr;

    // multi-rank: ghost-framed buffer (ext rectangle), pack / unpack buffers, communicator
    bool multi = false, has_comm = false;
    LoopGroup* loop = nullptr;   // loopback transport (tests); nullptr with NCCL
    int loop_id = -1;
    double* d_loop_tmp = nullptr;
    z2* d_ext = nullptr;
    long long ext_stride = 0, n_ext = 0;
    z2* d_sendbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    z2* d_recvbuf[4] = {nullptr, nullptr, nullptr, nullptr};
    long long msg_cap = 0;
    double* d_sq = nullptr;
#ifdef HELM_HAVE_NCCL
    ncclComm_t comm = nullptr;
#endif
    // Section 3(i): band flags per node index, the band sub-rectangles of every apply-frame message (by schedule
    // index), and element counters of the halo traffic (helm_comm_counters)
    bool res_band = false;     // Richardson restricts its residual to the interface band (owner PoU only)
    bool band_xchg = false;    // the current apply exchanges only the band part of its ghost frame
    unsigned char *d_bandx = nullptr, *d_bandy = nullptr;
    struct BandMsg {
        int4* d_rects = nullptr;
        long long* d_off = nullptr;
        int n = 0;
        long long total = 0, max_area = 0;
    } band_send[4], band_recv[4];
    long long xc_sent = 0, xc_recv = 0, xc_msgs = 0, xc_allreduce = 0;

    // Krylov workspace
    z2* d_V = nullptr;
    int V_cap = 0;
    z2 *d_w = nullptr, *d_z = nullptr, *d_t = nullptr, *d_r = nullptr, *d_xb = nullptr, *d_bb = nullptr;
    z2 *d_h1 = nullptr, *d_h2 = nullptr, *d_Hcol = nullptr, *d_y = nullptr;
    double* d_norm = nullptr;
    z2* d_zpart = nullptr;
    double* d_dpart = nullptr;
    int nblk = 148 * 4;
    z2* h_pin = nullptr;   // pinned host staging for y / norms (NVMAX complex)
    z2* h_hc = nullptr;    // pinned host slots: Hessenberg columns (CGS2) / the DCGS2 step record
    // DCGS2: device Hessenberg (NVMAX + 1) x NVMAX, reduced sweep sums, sweep-2 coefficients, step
    // record for the host (final column j - 1, pending column j, nu_j, ||u_{j+1}||)
    z2 *d_H = nullptr, *d_dots = nullptr, *d_ca = nullptr, *d_ce = nullptr, *d_hout = nullptr;
    // B^-1 u_j of every step (DCGS2): x += B^-1 V y = Z (R^-1 y) at a cycle's end without another apply
    z2* d_Z = nullptr;
    int Z_cap = 0;
    double* d_sc = nullptr;
    bool orth_cgs2 = false;
    // HELM_GMRES_PHASES=1 (development aid): CUDA events between the phases of every DCGS2 step, totals to stderr
    bool phases = false;
    cudaEvent_t ev_ph[8] = {};
    double ph_ms[8] = {};
    // multi-rank apply overlapped with its halo exchange: subdomains whose full box lies inside the
    // owned rectangle run while the ghost frame is in flight; the rest run on the communication stream after it
    bool overlap = false;
    cudaStream_t cstream = nullptr;
    cudaEvent_t ev_ov[2] = {nullptr, nullptr};
    int* d_order_ov = nullptr;   // interior subdomains (cost-sorted), then boundary subdomains (cost-sorted)
    int n_int = 0, n_bnd = 0, grid_int = 0, grid_bnd = 0;   // helm_set_orthogonalisation(HELM_ORTH_CGS2): the undelayed CGS2
    cudaEvent_t ev_hc[2] = {nullptr, nullptr};

    // profiling of the apply kernel
    bool prof = false;
    std::vector<cudaEvent_t> ev_free;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used;
    int launches = 0;

    // shared factors (D28): classes of subdomains whose local operators are bitwise equal; one representative per
    // class is factored and every member's fac_off points at its factors.  HELM_SHARE_FACTORS=0 factors every
    // subdomain (the general path, e.g. for a variable wave speed where no two local operators agree).
    bool share = true;
    std::vector<int> cls_rep, cls_of;
    long long n_dinv_all = 0;   // factor complex entries without sharing (layout reporting)
    // shared-factor apply on the tensor cores (batch.cu): HELM_APPLY_BATCH = 0 / 1 forces it off / on; by default on
    // when the factors are shared, m_max <= 128 and the whole problem has at least one subdomain per SM (decided on
    // global quantities so that every rank of a decomposition takes the same path)
    bool batched = false;
    z2* d_dinvB = nullptr;
    BatchTile* d_tiles = nullptr;
    BatchClass* d_bcls = nullptr;
    int* d_members = nullptr;
    z2* d_bscr = nullptr;
    int bt_ntiles = 0, bt_nint = 0, bt_grid = 0, bt_grid_int = 0, bt_grid_bnd = 0;
    int bt_block = 0, bt_smem = 0, bt_slot = 0, bt_nslots = 0, bt_mpmax = 0, bt_occ = 0, bt_w = BATCH_NT, bt_split = 0;
    long long bt_scr_per_cta = 0, dinvB_len = 0;

    // constant interior stencil (rows with gamma = 1 on all six triangles) and its node range
    int cst[4] = {0, 0, 0, 0};
    z2 c7[9] = {};
    z2 lcS{}, lcSW{}, lcN{}, lcNE{}, lcSE{}, lcNW{};   // constant local couplings (apply)

    StencilGeom geom_for(int xi0, int xj0, long long xstride) const
    {
        StencilGeom s{};
        s.i0 = G.i0;
        s.j0 = G.j0;
        s.nx = G.i1 - G.i0;
        s.ny = G.j1 - G.j0;
        s.nf = G.nf;
        s.xi0 = xi0;
        s.xj0 = xj0;
        s.xstride = xstride;
        s.ci0 = cst[0];
        s.ci1 = cst[1];
        s.cj0 = cst[2];
        s.cj1 = cst[3];
        s.ns = G.ns;
        for (int q = 0; q < 9; q++) s.c7[q] = c7[q];
        return s;
    }
    StencilGeom owned_geom() const { return geom_for(G.i0, G.j0, G.i1 - G.i0); }
    StencilGeom ext_geom() const { return geom_for(G.e_i0, G.e_j0, ext_stride); }
};

static int set_err(helm_ctx* ctx, int code, const char* fmt, ...)
{
    if (ctx) {
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(ctx->err, sizeof(ctx->err), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define CK(expr) HELM_CUDA_OK(expr)

#ifdef HELM_HAVE_NCCL
#define NK(expr)                                                                                              \
    do {                                                                                                      \
        ncclResult_t r__ = (expr);                                                                            \
        if (r__ != ncclSuccess) return set_err(ctx, HELM_ENCCL, "%s: %s", #expr, ncclGetErrorString(r__));   \
    } while (0)
#endif

namespace {

template <class T>
int dalloc(helm_ctx* ctx, T** p, size_t count)
{
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ctx, HELM_ENOMEM, "cudaMalloc of %.3f GB failed: %s", count * sizeof(T) / 1e9,
                       cudaGetErrorString(e));
    }
    return HELM_OK;
}

int build_layout(helm_ctx* ctx)
{
    GridInfo& G = ctx->G;
    int rc = compute_grid(ctx->p, ctx->rank, ctx->nranks, G, ctx->err, sizeof(ctx->err));
    if (rc) return rc;
    Geom& g = ctx->geom;
    g.k = ctx->p.k;
    g.h = G.h;
    g.h3 = G.h / 3.0;
    g.sigma0 = ctx->p.sigma0;
    g.kappa = G.ng * G.h;   // D3: one profile, kappa = kappa_g
    g.N = G.N;
    g.nf = G.nf;
    g.ng = G.ng;
    g.lo3 = 3L * G.ng;
    g.hi3 = 3L * (G.N - G.ng);
    g.elem = ctx->p.elem;
    g.frame = G.frame;
    g.lo_u = G.lo_u;
    g.hi_u = G.hi_u;
    g.pml_c = ctx->p.pml_c;
    if (G.frame == 1) g.kappa = ctx->p.kappa_g;
    ctx->n_local = (long long)(G.i1 - G.i0) * (G.j1 - G.j0);

    long long fac = 0, stc = 0;
    ctx->subs.clear();
    for (int by = G.by0; by < G.by1; by++)
        for (int bx = G.bx0; bx < G.bx1; bx++) {
            const int bb[2] = {bx, by};
            int own_lo[2], own_hi[2], int_lo[2], int_hi[2], full_lo[2], full_hi[2], has_lo[2], has_hi[2];
            for (int ax = 0; ax < 2; ax++) {
                const int b = bb[ax];
                own_lo[ax] = G.st[ax][b];
                own_hi[ax] = G.st[ax][b + 1];
                has_lo[ax] = b > 0;
                has_hi[ax] = b < G.P[ax] - 1;
                int_lo[ax] = own_lo[ax] - (has_lo[ax] ? G.wo : 0);
                int_hi[ax] = own_hi[ax] + (has_hi[ax] ? G.wo : 0);
                full_lo[ax] = int_lo[ax] - (has_lo[ax] ? G.wp : 0);
                full_hi[ax] = int_hi[ax] + (has_hi[ax] ? G.wp : 0);
                if (full_lo[ax] < 0 || full_hi[ax] > G.N)
                    return set_err(ctx, HELM_ELAYOUT, "full box of subdomain (%d,%d) leaves Omega", bx, by);
            }
            SubDesc d{};
            // local unknowns: nodes strictly inside the full box (Dirichlet on dOmega_j) plus, for
            // RAS-PML-Imp, the nodes on faces carrying the impedance condition
            const int imp = ctx->p.local_bc == HELM_BC_IMPEDANCE;
            int node0[2], node1[2];
            for (int ax = 0; ax < 2; ax++) {
                node0[ax] = full_lo[ax] + ((imp && has_lo[ax]) ? 0 : 1);
                node1[ax] = full_hi[ax] - ((imp && has_hi[ax]) ? 0 : 1);
            }
            d.m = node1[0] - node0[0] + 1;
            d.nb = node1[1] - node0[1] + 1;
            d.gx0 = node0[0];
            d.gy0 = node0[1];
            d.fx0 = full_lo[0];
            d.fx1 = full_hi[0];
            d.fy0 = full_lo[1];
            d.fy1 = full_hi[1];
            d.imp = imp ? ((has_lo[0] ? 1 : 0) | (has_hi[0] ? 2 : 0) | (has_lo[1] ? 4 : 0) | (has_hi[1] ? 8 : 0)) : 0;
            if (ctx->p.pou == HELM_POU_RAMP) {
                // the solution is needed wherever chi_j > 0: the int box interior
                d.olo = std::max(int_lo[0] + (has_lo[0] ? 1 : 0), 1) - d.gx0;
                d.ohi = std::min(int_hi[0] - (has_hi[0] ? 1 : 0), G.N - 1) - d.gx0;
                d.lo = std::max(int_lo[1] + (has_lo[1] ? 1 : 0), 1) - d.gy0;
                d.hi = std::min(int_hi[1] - (has_hi[1] ? 1 : 0), G.N - 1) - d.gy0;
            } else {
                // restricted owner write (D10): the block's own nodes
                d.olo = std::max(own_lo[0], 1) - d.gx0;
                d.ohi = std::min(own_hi[0], G.N) - 1 - d.gx0;
                d.lo = std::max(own_lo[1], 1) - d.gy0;
                d.hi = std::min(own_hi[1], G.N) - 1 - d.gy0;
            }
            // twist row: any row in [lo, hi] gives the same nb + hi - lo streamed blocks; this one
            // balances the two chains' step counts (bottom: 2 tw - lo + 1, top: nb - 1 + hi - 2 tw + 1), which is the
            // critical path when the chains run concurrently (k_apply_split)
            d.tw = std::min(d.hi, std::max(d.lo, (d.nb - 1 + d.hi + d.lo + 2) / 4));
            d.s0x = own_lo[0];
            d.s1x = own_hi[0];
            d.s0y = own_lo[1];
            d.s1y = own_hi[1];
            d.pou_off = ctx->pou_len;
            if (ctx->p.pou == HELM_POU_RAMP) ctx->pou_len += (long long)(d.ohi - d.olo + 1) * (d.hi - d.lo + 1);
            d.ilo3 = 3 * int_lo[0];
            d.ihi3 = 3 * int_hi[0];
            d.jlo3 = 3 * int_lo[1];
            d.jhi3 = 3 * int_hi[1];
            d.flags = (has_lo[0] ? 1 : 0) | (has_hi[0] ? 2 : 0) | (has_lo[1] ? 4 : 0) | (has_hi[1] ? 8 : 0);
            d.ns = G.ns;
            {
                // constant-coupling node range: cells [max(a_j, ceil lo_u), min(b_j, floor hi_u)) have local
                // gamma = 1 (inside the int box where g_j = g_i, and inside Omega_int where g_i = 0)
                int c0[2], c1[2];
                for (int ax = 0; ax < 2; ax++) {
                    const int lo_cell = std::max(has_lo[ax] ? int_lo[ax] : 0, (int)ceil(G.lo_u));
                    const int hi_cell = std::min(has_hi[ax] ? int_hi[ax] : G.N, (int)floor(G.hi_u));
                    // nodes with both adjacent cells inside, and all neighbours free in Omega_j
                    c0[ax] = std::max(lo_cell + 1, full_lo[ax] + 2);
                    c1[ax] = std::min(hi_cell, full_hi[ax] - 1);
                }
                d.cx0 = std::max(c0[0] - d.gx0, 0);
                d.cx1 = std::max(std::min(c1[0] - d.gx0, d.m), d.cx0);
                d.cy0 = std::max(c0[1] - d.gy0, 0);
                d.cy1 = std::max(std::min(c1[1] - d.gy0, d.nb), d.cy0);
            }
            d.fac_off = fac;
            d.stc_off = stc;
            if (d.m > M_LIMIT)
                return set_err(ctx, HELM_EINVAL, "local block width %d exceeds %d (use more subdomains)", d.m, M_LIMIT);
            // every node the subdomain reads must lie in this rank's ext rectangle
            if (d.gx0 < G.e_i0 || d.gx0 + d.m > G.e_i1 || d.gy0 < G.e_j0 || d.gy0 + d.nb > G.e_j1)
                return set_err(ctx, HELM_ELAYOUT, "subdomain (%d,%d) reaches beyond the halo of rank %d", bx, by,
                               ctx->rank);
            fac += (long long)d.nb * d.m * d.m;
            stc += (long long)d.nb * G.ns * d.m;
            ctx->m_max = std::max(ctx->m_max, d.m);
            const long long n = (long long)d.m * d.nb;
            ctx->max_n = std::max(ctx->max_n, n);
            ctx->local_unknowns += n;
            ctx->scratch_per_cta = std::max(ctx->scratch_per_cta, (long long)(d.hi - d.lo + 1) * d.m);
            // algorithmic bytes of one apply of this subdomain
            const long long nblocks = d.nb + d.hi - d.lo;
            const long long owned = (long long)(d.ohi - d.olo + 1) * (d.hi - d.lo + 1);
            // coupling vectors loaded per block step (two, three for Q1; twice that at the twist), except at
            // constant-stencil nodes;
            // the first step of each chain reads none (T: i = nb-1, B: i = 0)
            long long cpl = 0;
            auto loaded = [&](int i) { return (long long)d.m - ((i >= d.cy0 && i < d.cy1) ? (d.cx1 - d.cx0) : 0); };
            const int cv = G.ns == 9 ? 3 : 2;                   // vectors per coupling matrix
            for (int i = 0; i < d.nb; i++) {
                int uses = 0;
                if (i > d.tw && i < d.nb - 1) uses += cv;       // T: U_i
                if (i < d.tw && i > 0) uses += cv;              // B: L_i
                if (i == d.tw) uses += (i > 0 ? cv : 0) + (i < d.nb - 1 ? cv : 0);   // Z: L and U
                if (i < d.tw && i >= d.lo) uses += cv;          // D: U_i
                if (i > d.tw && i <= d.hi) uses += cv;          // U: L_i
                cpl += uses * loaded(i);
            }
            ctx->apply_bytes += 16 * (nblocks * d.m * d.m       // explicit inverse blocks streamed
                                      + n                       // restriction gather
                                      + cpl                     // coupling vectors
                                      + 2LL * (d.hi - d.lo) * d.m   // y / z scratch written + read
                                      + owned);                 // owner write
            ctx->band_bytes += 16 * (n * (2LL * (d.m + 1) + 1) + n + owned);
            ctx->subs.push_back(d);
        }
    ctx->n_dinv = ctx->n_dinv_all = fac;
    ctx->n_stc = stc;
    // ramp PoU: the gather re-reads every weighted value once and writes z once
    if (ctx->p.pou == HELM_POU_RAMP) ctx->apply_bytes += 16 * (ctx->pou_len + ctx->n_local);
    return HELM_OK;
}

// work vectors, reduction buffers and pinned staging (restart = 0), plus a GMRES basis of restart + 1 vectors and
// the DCGS2 Z basis (restart > 0).  helm_factor calls it with 0 so that a solve's timing holds no allocation.
int ensure_krylov(helm_ctx* ctx, int restart)
{
    int rc;
    const long long n = ctx->n_local;
    if (!ctx->d_w) {
        if ((rc = dalloc(ctx, &ctx->d_w, n)) || (rc = dalloc(ctx, &ctx->d_z, n)) || (rc = dalloc(ctx, &ctx->d_t, n)) ||
            (rc = dalloc(ctx, &ctx->d_r, n)) || (rc = dalloc(ctx, &ctx->d_h1, NVMAX)) ||
            (rc = dalloc(ctx, &ctx->d_h2, NVMAX)) || (rc = dalloc(ctx, &ctx->d_Hcol, NVMAX)) ||
            (rc = dalloc(ctx, &ctx->d_y, NVMAX)) || (rc = dalloc(ctx, &ctx->d_norm, 4)) ||
            (rc = dalloc(ctx, &ctx->d_zpart, (size_t)ctx->nblk * 2 * NVMAX)) || (rc = dalloc(ctx, &ctx->d_dpart, ctx->nblk)) ||
            (rc = dalloc(ctx, &ctx->d_H, (size_t)(NVMAX + 1) * NVMAX)) || (rc = dalloc(ctx, &ctx->d_dots, 2 * NVMAX)) ||
            (rc = dalloc(ctx, &ctx->d_ca, NVMAX)) || (rc = dalloc(ctx, &ctx->d_ce, NVMAX)) ||
            (rc = dalloc(ctx, &ctx->d_hout, 3 * NVMAX + 2)) || (rc = dalloc(ctx, &ctx->d_sc, 4)))
            return rc;
        CK(cudaMallocHost((void**)&ctx->h_pin, sizeof(z2) * NVMAX));
        CK(cudaMallocHost((void**)&ctx->h_hc, sizeof(z2) * 2 * (3 * NVMAX + 2)));
        const char* ph = getenv("HELM_GMRES_PHASES");
        if (ph && ph[0] == '1') {
            ctx->phases = true;
            for (auto& e : ctx->ev_ph) CK(cudaEventCreate(&e));
        }


        for (auto& e : ctx->ev_hc) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (restart > 0 && restart + 1 > ctx->V_cap) {
        if (ctx->d_V) cudaFree(ctx->d_V);
        ctx->d_V = nullptr;
        ctx->V_cap = 0;
        if ((rc = dalloc(ctx, &ctx->d_V, (size_t)(restart + 1) * n))) return rc;
        ctx->V_cap = restart + 1;
    }
    if (restart > 0 && !ctx->orth_cgs2 && restart > ctx->Z_cap) {
        if (ctx->d_Z) cudaFree(ctx->d_Z);
        ctx->d_Z = nullptr;
        ctx->Z_cap = 0;
        if ((rc = dalloc(ctx, &ctx->d_Z, (size_t)restart * n))) return rc;
        ctx->Z_cap = restart;
    }
    return HELM_OK;
}

int need_comm(helm_ctx* ctx)
{
    if (ctx->multi && !ctx->has_comm)
        return set_err(ctx, HELM_ENCCL, "communication-free shard: use the _ext entry points");
    return HELM_OK;
}

// ---------------------------------------------------------------------------------------- collectives
// loopback: after the phase's messages are packed, copy each peer's send buffer addressed to this rank into the
// matching receive buffer (the peer's message index is recomputed from its own schedule)
int loop_sendrecv(helm_ctx* ctx, int W, int phase, const helm_msg* msgs, const int* idx, int k, bool reverse,
                  bool band, cudaStream_t st)
{
    LoopGroup* L = ctx->loop;
    CK(cudaStreamSynchronize(st));
    if (!L->barrier()) return set_err(ctx, HELM_ENCCL, "loopback group aborted by another rank");   // all packed
    for (int a = 0; a < k; a++) {
        const helm_msg& m = msgs[idx[a]];
        const helm_ctx* peer = L->ctx[m.peer];
        helm_msg pm[4];
        const int pn = halo_schedule(peer->G, W, pm, 4);
        int pa = 0, found = -1, fq = -1;   // position among the peer's phase messages (= its send buffer), index in pm
        for (int q = 0; q < pn; q++)
            if (pm[q].phase == phase) {
                if (pm[q].peer == ctx->rank) {
                    found = pa;
                    fq = q;
                }
                pa++;
            }
        if (found < 0) return set_err(ctx, HELM_ENCCL, "loopback: rank %d has no message for rank %d", m.peer, ctx->rank);
        // forward: the peer packed its send rectangle into my receive rectangle; reverse: its receive rectangle (its
        // ghost frame toward me) onto my send rectangle (my owned strip)
        size_t rcnt = reverse ? (size_t)(m.send_i1 - m.send_i0) * (m.send_j1 - m.send_j0)
                              : (size_t)(m.recv_i1 - m.recv_i0) * (m.recv_j1 - m.recv_j0);
        size_t scnt = reverse ? (size_t)(pm[fq].recv_i1 - pm[fq].recv_i0) * (pm[fq].recv_j1 - pm[fq].recv_j0)
                              : (size_t)(pm[fq].send_i1 - pm[fq].send_i0) * (pm[fq].send_j1 - pm[fq].send_j0);
        if (band) {   // band parts only (section 3(i)): my decomposition of the receive rectangle, the peer's of its send
            rcnt = (size_t)ctx->band_recv[idx[a]].total;
            scnt = (size_t)peer->band_send[fq].total;
        }
        if (scnt != rcnt) return set_err(ctx, HELM_ENCCL, "loopback: message size mismatch %zu vs %zu", scnt, rcnt);
        CK(cudaMemcpyAsync(ctx->d_recvbuf[a], peer->d_sendbuf[found], sizeof(z2) * rcnt, cudaMemcpyDeviceToDevice,
                           st));
    }
    CK(cudaStreamSynchronize(st));
    if (!L->barrier()) return set_err(ctx, HELM_ENCCL, "loopback group aborted by another rank");   // may refill
    return HELM_OK;
}

// The NCCL transport of one exchange phase: k grouped send/receive pairs of complex128 buffers (counts in complex
// elements) with the given peers, on stream st.
int nccl_sendrecv(helm_ctx* ctx, int k, const int* peers, z2* const* sendbuf, const size_t* scnt, z2* const* recvbuf,
                  const size_t* rcnt, cudaStream_t st)
{
#ifdef HELM_HAVE_NCCL
    if (!ctx->comm) return set_err(ctx, HELM_ENCCL, "no NCCL communicator");
    NK(ncclGroupStart());
    for (int a = 0; a < k; a++) {
        NK(ncclSend(sendbuf[a], 2 * scnt[a], ncclDouble, peers[a], ctx->comm, st));
        NK(ncclRecv(recvbuf[a], 2 * rcnt[a], ncclDouble, peers[a], ctx->comm, st));
    }
    NK(ncclGroupEnd());
    return HELM_OK;
#else
    (void)k; (void)peers; (void)sendbuf; (void)scnt; (void)recvbuf; (void)rcnt; (void)st;
    return set_err(ctx, HELM_ENCCL, "library built without NCCL");
#endif
}

// halo exchange of width W on a ghost-framed buffer `buf` (ext rectangle layout).  Forward (reverse = false): the
// owned strips travel to the neighbours' ghost frames, phase 0 (x) then phase 1 (y, carrying the corners).
// Reverse (reverse = true, the ramp PoU's additive exchange): the ghost frames travel back and are ADDED onto the
// neighbours' owned strips, phase 1 then phase 0, so corner contributions reach the diagonal rank in two hops.
int exchange_buf(helm_ctx* ctx, int W, z2* buf, bool reverse, cudaStream_t st)
{
    NvtxRange nv_(reverse ? "helm.comm.halo_add" : (W == 0 ? "helm.comm.halo_apply" : "helm.comm.halo_spmv"));
    helm_msg msgs[4];
    const int nm = halo_schedule(ctx->G, W, msgs, 4);
    const GridInfo& G = ctx->G;
    // section 3(i): only the interface-band part of the apply frame (the caller zeroed the rest of the frame)
    const bool band = ctx->band_xchg && W == 0 && !reverse;
    for (int ph = 0; ph < 2; ph++) {
        const int phase = reverse ? 1 - ph : ph;
        int idx[4], k = 0;
        for (int q = 0; q < nm; q++)
            if (msgs[q].phase == phase) idx[k++] = q;
        if (!k && !ctx->loop) continue;   // (loopback ranks meet at every phase's barriers)
        size_t scnt[4], rcnt[4];
        for (int a = 0; a < k; a++) {
            const helm_msg& m = msgs[idx[a]];
            const size_t sa = (size_t)(m.send_i1 - m.send_i0) * (m.send_j1 - m.send_j0);
            const size_t ra = (size_t)(m.recv_i1 - m.recv_i0) * (m.recv_j1 - m.recv_j0);
            scnt[a] = band ? (size_t)ctx->band_send[idx[a]].total : (reverse ? ra : sa);
            rcnt[a] = band ? (size_t)ctx->band_recv[idx[a]].total : (reverse ? sa : ra);
            if (band) {
                const auto& bm = ctx->band_send[idx[a]];
                launch_pack_rects(buf, G.e_i0, G.e_j0, ctx->ext_stride, bm.d_rects, bm.d_off, bm.n, bm.max_area,
                                  ctx->d_sendbuf[a], false, st);
            } else {
                const int i0 = reverse ? m.recv_i0 : m.send_i0, i1 = reverse ? m.recv_i1 : m.send_i1;
                const int j0 = reverse ? m.recv_j0 : m.send_j0, j1 = reverse ? m.recv_j1 : m.send_j1;
                launch_copy_rect(buf, G.e_i0, G.e_j0, ctx->ext_stride, ctx->d_sendbuf[a], i0, j0, i1 - i0, i0, i1, j0,
                                 j1, st);
            }
            ctx->launches++;
            ctx->xc_sent += (long long)scnt[a];
            ctx->xc_recv += (long long)rcnt[a];
            ctx->xc_msgs++;
        }
        if (ctx->loop) {
            int rc = loop_sendrecv(ctx, W, phase, msgs, idx, k, reverse, band, st);
            if (rc) return rc;
        } else {
            int peers[4];
            for (int a = 0; a < k; a++) peers[a] = msgs[idx[a]].peer;
            int rc = nccl_sendrecv(ctx, k, peers, ctx->d_sendbuf, scnt, ctx->d_recvbuf, rcnt, st);
            if (rc) return rc;
        }
        for (int a = 0; a < k; a++) {
            const helm_msg& m = msgs[idx[a]];
            if (band) {
                const auto& bm = ctx->band_recv[idx[a]];
                launch_pack_rects(buf, G.e_i0, G.e_j0, ctx->ext_stride, bm.d_rects, bm.d_off, bm.n, bm.max_area,
                                  ctx->d_recvbuf[a], true, st);
            } else {
                const int i0 = reverse ? m.send_i0 : m.recv_i0, i1 = reverse ? m.send_i1 : m.recv_i1;
                const int j0 = reverse ? m.send_j0 : m.recv_j0, j1 = reverse ? m.send_j1 : m.recv_j1;
                launch_copy_rect(ctx->d_recvbuf[a], i0, j0, i1 - i0, buf, G.e_i0, G.e_j0, ctx->ext_stride, i0, i1, j0,
                                 j1, st, reverse);
            }
            ctx->launches++;
        }
    }
    return HELM_OK;
}

int exchange(helm_ctx* ctx, int W) { return exchange_buf(ctx, W, ctx->d_ext, false, ctx->stream); }

// in-place sum over ranks of `count` doubles on the device
int allreduce(helm_ctx* ctx, double* buf, size_t count)
{
    if (!ctx->multi) return HELM_OK;
    ctx->xc_allreduce++;
    NvtxRange nv_("helm.comm.allreduce");
    if (ctx->loop) {
        // loopback: every rank sums all ranks' buffers in rank order (identical bits everywhere)
        LoopGroup* L = ctx->loop;
        if (count > 4 * NVMAX) return set_err(ctx, HELM_EINVAL, "loopback allreduce of %zu doubles", count);
        CK(cudaStreamSynchronize(ctx->stream));
        L->slot[ctx->rank] = buf;
        if (!L->barrier()) return set_err(ctx, HELM_ENCCL, "loopback group aborted by another rank");
        launch_sum_ranks(L->slot.data(), L->nranks, (int)count, ctx->d_loop_tmp, ctx->stream);
        ctx->launches++;
        CK(cudaStreamSynchronize(ctx->stream));
        if (!L->barrier()) return set_err(ctx, HELM_ENCCL, "loopback group aborted by another rank");   // all read
        CK(cudaMemcpyAsync(buf, ctx->d_loop_tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
        return HELM_OK;
    }
#ifdef HELM_HAVE_NCCL
    NK(ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return HELM_OK;
#else
    (void)buf;
    (void)count;
    return set_err(ctx, HELM_ENCCL, "library built without NCCL");
#endif
}

// owned vector -> interior of d_ext, then exchange ghost layers (W = 0: the apply frame)
int fill_ext(helm_ctx* ctx, const z2* v, int W)
{
    const GridInfo& G = ctx->G;
    if (ctx->band_xchg && W == 0)   // the frame's non-band nodes are zero, not last exchange's values
        CK(cudaMemsetAsync(ctx->d_ext, 0, sizeof(z2) * ctx->n_ext, ctx->stream));
    launch_copy_rect(v, G.i0, G.j0, G.i1 - G.i0, ctx->d_ext, G.e_i0, G.e_j0, ctx->ext_stride, G.i0, G.i1, G.j0, G.j1,
                     ctx->stream);
    ctx->launches++;
    return exchange(ctx, W);
}

// ------------------------------------------------------------------------------------------- operators
// apply timing (helm_profile_enable): a pair of events on the library stream around each apply
int prof_begin(helm_ctx* ctx, cudaEvent_t* e0, cudaEvent_t* e1)
{
    if (!ctx->prof) return HELM_OK;
    if (ctx->ev_free.size() < 2) {
        cudaEvent_t a0, a1;
        CK(cudaEventCreate(&a0));
        CK(cudaEventCreate(&a1));
        ctx->ev_free.push_back(a0);
        ctx->ev_free.push_back(a1);
    }
    *e1 = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    *e0 = ctx->ev_free.back();
    ctx->ev_free.pop_back();
    CK(cudaEventRecord(*e0, ctx->stream));
    return HELM_OK;
}
int prof_end(helm_ctx* ctx, cudaEvent_t e0, cudaEvent_t e1)
{
    if (!ctx->prof) return HELM_OK;
    CK(cudaEventRecord(e1, ctx->stream));
    ctx->ev_used.push_back({e0, e1});
    return HELM_OK;
}

ApplyArgs apply_args(helm_ctx* ctx, const z2* in, int in_i0, int in_j0, long long in_stride, z2* z)
{
    ApplyArgs a{};
    a.desc = ctx->d_desc;
    a.order = ctx->d_order;
    a.nsub = (int)ctx->subs.size();
    a.dinv = ctx->d_dinv;
    a.stencil = ctx->d_stc;
    a.in = in;
    a.in_i0 = in_i0;
    a.in_j0 = in_j0;
    a.in_stride = in_stride;
    a.out = z;
    a.out_i0 = ctx->G.i0;
    a.out_j0 = ctx->G.j0;
    a.out_stride = ctx->G.i1 - ctx->G.i0;
    a.scratch = ctx->d_scratch;
    a.scratch_per_cta = ctx->scratch_per_cta;
    a.cS = ctx->lcS;
    a.cSW = ctx->lcSW;
    a.cN = ctx->lcN;
    a.cNE = ctx->lcNE;
    a.cSE = ctx->lcSE;
    a.cNW = ctx->lcNW;
    a.ns = ctx->G.ns;
    a.pou_buf = ctx->d_pou;
    a.delta = ctx->G.wo;
    return a;
}

// shared-factor apply (batch.cu) over tiles [t0, t0 + nt) with `grid` CTAs whose scratch starts at CTA slot `slot0`
BatchArgs batch_args(helm_ctx* ctx, const z2* in, int in_i0, int in_j0, long long in_stride, z2* z, int t0, int nt,
                     int slot0)
{
    BatchArgs b{};
    b.desc = ctx->d_desc;
    b.tiles = ctx->d_tiles + t0;
    b.ntiles = nt;
    b.members = ctx->d_members;
    b.cls = ctx->d_bcls;
    b.dinvB = ctx->d_dinvB;
    b.stencil = ctx->d_stc;
    b.in = in;
    b.in_i0 = in_i0;
    b.in_j0 = in_j0;
    b.in_stride = in_stride;
    b.out = z;
    b.out_i0 = ctx->G.i0;
    b.out_j0 = ctx->G.j0;
    b.out_stride = ctx->G.i1 - ctx->G.i0;
    b.scratch = ctx->d_bscr + (long long)slot0 * ctx->bt_scr_per_cta;
    b.scratch_per_cta = ctx->bt_scr_per_cta;
    b.cc = CplConst{ctx->lcS, ctx->lcSW, ctx->lcN, ctx->lcNE, ctx->lcSE, ctx->lcNW, ctx->G.ns};
    b.pou_buf = ctx->d_pou;
    b.delta = ctx->G.wo;
    return b;
}

int launch_batch(helm_ctx* ctx, const BatchArgs& b, int grid, cudaStream_t st)
{
    const int e = launch_apply_batch(b, grid, ctx->bt_block, ctx->bt_smem, ctx->bt_slot, ctx->bt_nslots, ctx->bt_mpmax,
                                     ctx->bt_split, st);
    if (e != 0) {
        cudaGetLastError();
        return set_err(ctx, HELM_ECUDA, "tensor-core apply launch: %s", cudaGetErrorString((cudaError_t)e));
    }
    return HELM_OK;
}

int apply_raw(helm_ctx* ctx, const z2* in, int in_i0, int in_j0, long long in_stride, z2* z)
{
    if (!ctx->factored) return set_err(ctx, HELM_ESTATE, "preconditioner applied before helm_factor");
    const ApplyArgs a = apply_args(ctx, in, in_i0, in_j0, in_stride, z);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    int rc;
    if ((rc = prof_begin(ctx, &e0, &e1))) return rc;
    if (ctx->batched) {
        const int grid = std::min(ctx->bt_ntiles * (ctx->bt_split ? 2 : 1), ctx->bt_grid_int + ctx->bt_grid_bnd);
        if ((rc = launch_batch(ctx, batch_args(ctx, in, in_i0, in_j0, in_stride, z, 0, ctx->bt_ntiles, 0), grid,
                               ctx->stream)))
            return rc;
    } else if (ctx->sp_G > 0) {
        const int e = launch_apply_split(a, (int)ctx->subs.size(), ctx->sp_G, ctx->sp_block, ctx->sp_smem, ctx->sp_slot,
                                         ctx->sp_ncw, ctx->m_max, ctx->sp_nss, ctx->stream);
        if (e != 0) {
            cudaGetLastError();   // the failed launch is reported here, not to the next caller
            return set_err(ctx, HELM_ECUDA, "cluster apply launch: %s", cudaGetErrorString((cudaError_t)e));
        }
    } else {
        launch_apply(a, ctx->ap_grid, ctx->ap_block, ctx->ap_smem, ctx->ap_slot, ctx->ap_nslots, ctx->stream);
    }
    CK(cudaGetLastError());
    ctx->launches++;
    if (ctx->d_pou && !ctx->multi) {
        const GridInfo& G = ctx->G;
        launch_pou_gather(ctx->d_desc, ctx->d_candx, ctx->d_candy, G.bx0, G.bx1, G.by0, G.by1, ctx->d_pou, z, G.i0,
                          G.j0, G.i1 - G.i0, G.i0, G.i1, G.j0, G.j1, ctx->stream);
        CK(cudaGetLastError());
        ctx->launches++;
    }
    return prof_end(ctx, e0, e1);
}

// z = B^-1 r for an owned input vector (exchanging the halo when sharded)
int apply_impl(helm_ctx* ctx, const z2* r, z2* z)
{
    NvtxRange nv_("helm.apply");
    int rc;
    if ((rc = need_comm(ctx))) return rc;
    if (!ctx->multi) return apply_raw(ctx, r, ctx->G.i0, ctx->G.j0, ctx->G.i1 - ctx->G.i0, z);
    if (ctx->overlap) {
        if (!ctx->factored) return set_err(ctx, HELM_ESTATE, "preconditioner applied before helm_factor");
        const GridInfo& G = ctx->G;
        if (ctx->band_xchg) CK(cudaMemsetAsync(ctx->d_ext, 0, sizeof(z2) * ctx->n_ext, ctx->stream));
        launch_copy_rect(r, G.i0, G.j0, G.i1 - G.i0, ctx->d_ext, G.e_i0, G.e_j0, ctx->ext_stride, G.i0, G.i1, G.j0,
                         G.j1, ctx->stream);
        CK(cudaEventRecord(ctx->ev_ov[0], ctx->stream));
        cudaEvent_t e0 = nullptr, e1 = nullptr;   // timed: both parts and the exchange they hide
        if ((rc = prof_begin(ctx, &e0, &e1))) return rc;
        ApplyArgs a = apply_args(ctx, ctx->d_ext, G.e_i0, G.e_j0, ctx->ext_stride, z);
        auto part = [&](int grid, cudaStream_t st) -> int {
            if (ctx->batched) {
                const bool inner = st == ctx->stream;   // interior tiles on the library stream, the rest after the halo
                const int t0 = inner ? 0 : ctx->bt_nint, nt = inner ? ctx->bt_nint : ctx->bt_ntiles - ctx->bt_nint;
                const int rc2 = launch_batch(ctx, batch_args(ctx, ctx->d_ext, G.e_i0, G.e_j0, ctx->ext_stride, z, t0, nt,
                                                             inner ? 0 : ctx->bt_grid_int),
                                             inner ? ctx->bt_grid_int : ctx->bt_grid_bnd, st);
                if (rc2) return rc2;
            } else if (ctx->sp_G > 0) {
                const int e = launch_apply_split(a, a.nsub, ctx->sp_G, ctx->sp_block, ctx->sp_smem, ctx->sp_slot,
                                                 ctx->sp_ncw, ctx->m_max, ctx->sp_nss, st);
                if (e != 0) {
                    cudaGetLastError();
                    return set_err(ctx, HELM_ECUDA, "cluster apply launch: %s", cudaGetErrorString((cudaError_t)e));
                }
            } else {
                launch_apply(a, grid, ctx->ap_block, ctx->ap_smem, ctx->ap_slot, ctx->ap_nslots, st);
            }
            CK(cudaGetLastError());
            return HELM_OK;
        };
        a.order = ctx->d_order_ov;   // interior subdomains: owned input only
        a.nsub = ctx->n_int;
        if ((rc = part(ctx->grid_int, ctx->stream))) return rc;
        CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_ov[0], 0));
        if ((rc = exchange_buf(ctx, 0, ctx->d_ext, false, ctx->cstream))) return rc;
        a.order = ctx->d_order_ov + ctx->n_int;   // boundary subdomains, once the ghost frame is in
        a.nsub = ctx->n_bnd;
        // scratch slots after the interior launch's (plain: one per CTA; split: one per CTA of each cluster)
        a.scratch = ctx->d_scratch + (ctx->sp_G > 0 ? (long long)ctx->n_int * 2 * ctx->sp_G : (long long)ctx->grid_int) *
                                         ctx->scratch_per_cta;
        if ((rc = part(ctx->grid_bnd, ctx->cstream))) return rc;
        CK(cudaEventRecord(ctx->ev_ov[1], ctx->cstream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_ov[1], 0));
        if ((rc = prof_end(ctx, e0, e1))) return rc;
        ctx->launches += 3;
    } else {
        if ((rc = fill_ext(ctx, r, 0))) return rc;
        if ((rc = apply_raw(ctx, ctx->d_ext, ctx->G.e_i0, ctx->G.e_j0, ctx->ext_stride, z))) return rc;
    }
    if (!ctx->d_pou) return HELM_OK;
    // ramp PoU on several ranks: this rank's weighted contributions on its ghost-framed rectangle, the
    // additive reverse exchange of the frames (width delta), then the owned part is the prolongation
    const GridInfo& G = ctx->G;
    launch_pou_gather(ctx->d_desc, ctx->d_candx, ctx->d_candy, G.bx0, G.bx1, G.by0, G.by1, ctx->d_pou, ctx->d_cext,
                      G.e_i0, G.e_j0, ctx->ext_stride, G.e_i0, G.e_i1, G.e_j0, G.e_j1, ctx->stream);
    ctx->launches++;
    if ((rc = exchange_buf(ctx, G.wo, ctx->d_cext, true, ctx->stream))) return rc;
    launch_copy_rect(ctx->d_cext, G.e_i0, G.e_j0, ctx->ext_stride, z, G.i0, G.j0, G.i1 - G.i0, G.i0, G.i1, G.j0, G.j1,
                     ctx->stream);
    ctx->launches++;
    CK(cudaGetLastError());
    return HELM_OK;
}

// y = A x for an owned input vector
int spmv_impl(helm_ctx* ctx, const z2* x, z2* y)
{
    NvtxRange nv_("helm.spmv");
    int rc;
    if ((rc = need_comm(ctx))) return rc;
    if (!ctx->multi) {
        launch_spmv(ctx->d_A7, x, y, ctx->owned_geom(), ctx->stream);
    } else if (ctx->overlap) {
        // rows whose stencil stays in the owned rectangle run while the width-1 frame is exchanged on the communication
        // stream; the frame rows follow (each row computes exactly what the serial form does: bitwise equal)
        const GridInfo& G = ctx->G;
        const int a0 = G.nbr[0] >= 0, a1 = G.nbr[1] >= 0, b0 = G.nbr[2] >= 0, b1 = G.nbr[3] >= 0;
        launch_copy_rect(x, G.i0, G.j0, G.i1 - G.i0, ctx->d_ext, G.e_i0, G.e_j0, ctx->ext_stride, G.i0, G.i1, G.j0,
                         G.j1, ctx->stream);
        CK(cudaEventRecord(ctx->ev_ov[0], ctx->stream));
        launch_spmv(ctx->d_A7, ctx->d_ext, y, ctx->ext_geom(), ctx->stream, a0, a1, b0, b1);
        CK(cudaStreamWaitEvent(ctx->cstream, ctx->ev_ov[0], 0));
        if ((rc = exchange_buf(ctx, 1, ctx->d_ext, false, ctx->cstream))) return rc;
        CK(cudaEventRecord(ctx->ev_ov[1], ctx->cstream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_ov[1], 0));
        launch_spmv_frame(ctx->d_A7, ctx->d_ext, y, ctx->ext_geom(), a0, a1, b0, b1, ctx->stream);
        ctx->launches += 2;
    } else {
        if ((rc = fill_ext(ctx, x, 1))) return rc;
        launch_spmv(ctx->d_A7, ctx->d_ext, y, ctx->ext_geom(), ctx->stream);
    }
    ctx->launches++;
    return HELM_OK;
}

// global ||.||^2 partials -> norm on the device (d_norm) and optionally a Hessenberg slot
int finish_norm(helm_ctx* ctx, z2* slot)
{
    if (!ctx->multi) {
        launch_reduce_norm(ctx->d_dpart, ctx->nblk, slot, ctx->d_norm, ctx->stream);
        ctx->launches++;
        return HELM_OK;
    }
    launch_reduce_sq(ctx->d_dpart, ctx->nblk, ctx->d_sq, ctx->stream);
    int rc;
    if ((rc = allreduce(ctx, ctx->d_sq, 1))) return rc;
    launch_finish_norm(ctx->d_sq, slot, ctx->d_norm, ctx->stream);
    ctx->launches += 2;
    return HELM_OK;
}

int fetch_norm(helm_ctx* ctx, double* out)
{
    CK(cudaMemcpyAsync(ctx->h_pin, ctx->d_norm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    memcpy(out, ctx->h_pin, sizeof(double));
    return HELM_OK;
}

// ||v|| (global) to the host (synchronises)
int norm_host(helm_ctx* ctx, const z2* v, double* out)
{
    launch_norm_partial(v, ctx->n_local, ctx->d_dpart, ctx->nblk, ctx->stream);
    ctx->launches++;
    int rc;
    if ((rc = finish_norm(ctx, nullptr))) return rc;
    return fetch_norm(ctx, out);
}

// r = b - A x and ||r|| (host)
int residual_host(helm_ctx* ctx, const z2* b, const z2* x, z2* r, double* out)
{
    int rc;
    if (!ctx->multi) {
        launch_residual(ctx->d_A7, x, b, r, ctx->owned_geom(), ctx->d_dpart, ctx->nblk, ctx->stream);
    } else {
        if ((rc = fill_ext(ctx, x, 1))) return rc;
        launch_residual(ctx->d_A7, ctx->d_ext, b, r, ctx->ext_geom(), ctx->d_dpart, ctx->nblk, ctx->stream);
    }
    ctx->launches++;
    if ((rc = finish_norm(ctx, nullptr))) return rc;
    return fetch_norm(ctx, out);
}

// Right-preconditioned restarted GMRES (O9 of DESIGN.md), classical Gram-Schmidt with one
// re-orthogonalisation pass (CGS2) on the device, Givens rotations on the host one step behind the device.
int gmres_impl(helm_ctx* ctx, const z2* b, z2* x, int restart, double rtol, int maxit, helm_gmres_info* info)
{
    NvtxRange nv_("helm.gmres");
    if (!ctx->factored) return set_err(ctx, HELM_ESTATE, "gmres before helm_factor");
    if (restart < 1 || restart + 1 > NVMAX || maxit < 0)
        return set_err(ctx, HELM_EINVAL, "restart must be in [1, %d], maxit >= 0", NVMAX - 1);
    int rc;
    if ((rc = need_comm(ctx))) return rc;
    if ((rc = ensure_krylov(ctx, restart))) return rc;
    const long long n = ctx->n_local;
    cudaStream_t s = ctx->stream;
    helm_gmres_info loc{};
    helm_gmres_info* inf = info ? info : &loc;
    inf->iterations = inf->restarts = inf->applies = 0;
    inf->status = HELM_OK;
    inf->relres_est = inf->relres_true = 0.0;

    double beta0;
    if ((rc = norm_host(ctx, b, &beta0))) return rc;
    if (!(beta0 > 0.0)) {
        if (beta0 == 0.0) {   // b = 0 -> x = 0, no iteration
            CK(cudaMemsetAsync(x, 0, sizeof(z2) * n, s));
            CK(cudaStreamSynchronize(s));
            return HELM_OK;
        }
        inf->status = HELM_BREAKDOWN;
        return set_err(ctx, HELM_BREAKDOWN, "non-finite ||b||");
    }
    double beta;
    if ((rc = residual_host(ctx, b, x, ctx->d_r, &beta))) return rc;
    if (!std::isfinite(beta)) {
        inf->status = HELM_BREAKDOWN;
        return set_err(ctx, HELM_BREAKDOWN, "non-finite initial residual");
    }
    if (beta == 0.0 || (rtol > 0 && beta <= rtol * beta0)) {   // the initial guess already solves the system
        inf->relres_est = inf->relres_true = beta / beta0;
        return HELM_OK;
    }
    if (maxit == 0) {   // no iteration allowed: x is the initial guess, not converged
        inf->relres_est = inf->relres_true = beta / beta0;
        inf->status = HELM_NOT_CONVERGED;
        return HELM_NOT_CONVERGED;
    }
    const int m = restart;
    std::vector<cplx> H((size_t)(m + 1) * m), g(m + 1), sn(m), y(m);
    std::vector<double> cs(m);
    auto Hij = [&](int i, int j) -> cplx& { return H[(size_t)i * m + j]; };
    int its = 0, cycles = 0;
    double est = beta / beta0;
    z2* V = ctx->d_V;
    std::vector<cplx> Hraw((size_t)(m + 1) * m), gkeep(m + 1);
    std::vector<cplx> Rz((size_t)m * m);   // DCGS2: U = V R (u_j = nu_j v_j + V_j a^(j)), upper triangular
    auto Rzi = [&](int i, int j) -> cplx& { return Rz[(size_t)i * m + j]; };
    auto Rij = [&](int i, int j) -> cplx& { return Hraw[(size_t)i * m + j]; };
    // Givens rotation of column jc from its unrotated copy (DCGS2 revisits a column once it is final)
    auto rotate_col = [&](int jc) {
        for (int i = 0; i <= jc + 1; i++) Hij(i, jc) = Rij(i, jc);
        for (int i = 0; i < jc; i++) {
            const cplx a = Hij(i, jc), c = Hij(i + 1, jc);
            Hij(i, jc) = cs[i] * a + sn[i] * c;
            Hij(i + 1, jc) = -std::conj(sn[i]) * a + cs[i] * c;
        }
        const cplx a = Hij(jc, jc), bb = Hij(jc + 1, jc);
        if (a == cplx(0, 0)) {
            cs[jc] = 0.0;
            sn[jc] = 1.0;
            Hij(jc, jc) = bb;
        } else {
            const double rho = sqrt(std::norm(a) + std::norm(bb));
            const cplx ph = a / std::abs(a);
            cs[jc] = std::abs(a) / rho;
            sn[jc] = ph * std::conj(bb) / rho;
            Hij(jc, jc) = ph * rho;
        }
        Hij(jc + 1, jc) = 0.0;
        const cplx gs = gkeep[jc];
        g[jc] = cs[jc] * gs;
        g[jc + 1] = -std::conj(sn[jc]) * gs;
        gkeep[jc + 1] = g[jc + 1];
    };
    while (true) {
        int jend = 0;
        if (ctx->orth_cgs2) {
            // v_0 = r / ||r||
            memcpy(ctx->h_pin, &beta, sizeof(double));
            CK(cudaMemcpyAsync(ctx->d_norm, ctx->h_pin, sizeof(double), cudaMemcpyHostToDevice, s));
            launch_scale_by_norm(ctx->d_r, ctx->d_norm, V, n, s);
            ctx->launches++;
            std::fill(g.begin(), g.end(), cplx(0, 0));
            g[0] = beta;
            // (a one-step lookahead -- enqueueing step j + 1 before the host's Givens update of column j -- was
            // measured: no gain at c3, one discarded apply per solve)
            auto enqueue_step = [&](int j) -> int {
                z2* vj = V + (long long)j * n;
                int rc2;
                if ((rc2 = apply_impl(ctx, vj, ctx->d_z))) return rc2;
                inf->applies++;
                if ((rc2 = spmv_impl(ctx, ctx->d_z, ctx->d_w))) return rc2;
                // CGS2: h1 = V^H w; w -= V h1; h2 = V^H w; w -= V h2; H(:,j) = h1 + h2; H(j+1,j) = ||w||
                // (the first update and the second projection share one sweep over V: k_axpy_dot)
                NvtxRange nv_o("helm.orth");
                launch_multidot(V, n, j + 1, ctx->d_w, n, ctx->d_zpart, ctx->nblk, s);
                launch_reduce_z(ctx->d_zpart, ctx->nblk, j + 1, ctx->d_h1, nullptr, nullptr, s);
                if ((rc2 = allreduce(ctx, (double*)ctx->d_h1, 2 * (size_t)(j + 1)))) return rc2;
                launch_axpy_dot(V, n, j + 1, ctx->d_h1, ctx->d_w, n, ctx->d_zpart, ctx->nblk, s);
                if (!ctx->multi) {
                    launch_reduce_z(ctx->d_zpart, ctx->nblk, j + 1, ctx->d_h2, ctx->d_Hcol, ctx->d_h1, s);
                } else {
                    launch_reduce_z(ctx->d_zpart, ctx->nblk, j + 1, ctx->d_h2, nullptr, nullptr, s);
                    if ((rc2 = allreduce(ctx, (double*)ctx->d_h2, 2 * (size_t)(j + 1)))) return rc2;
                    launch_zadd(ctx->d_h1, ctx->d_h2, ctx->d_Hcol, j + 1, s);
                    ctx->launches++;
                }
                launch_multiaxpy(V, n, j + 1, ctx->d_h2, ctx->d_w, n, ctx->d_dpart, ctx->nblk, s);
                ctx->launches += 5;   // multidot, axpy_dot, 2x reduce, multiaxpy
                if ((rc2 = finish_norm(ctx, ctx->d_Hcol + j + 1))) return rc2;
                launch_scale_by_norm(ctx->d_w, ctx->d_norm, V + (long long)(j + 1) * n, n, s);
                ctx->launches++;
                CK(cudaGetLastError());
                CK(cudaMemcpyAsync(ctx->h_hc + (j & 1) * NVMAX, ctx->d_Hcol, sizeof(z2) * (j + 2),
                                   cudaMemcpyDeviceToHost, s));
                CK(cudaEventRecord(ctx->ev_hc[j & 1], s));
                return HELM_OK;
            };
            for (int j = 0; j < m; j++) {
                if ((rc = enqueue_step(j))) return rc;
                its++;
                CK(cudaEventSynchronize(ctx->ev_hc[j & 1]));
                const z2* hc = ctx->h_hc + (j & 1) * NVMAX;
                for (int i = 0; i <= j + 1; i++) Hij(i, j) = cplx(hc[i].x, hc[i].y);
                const double hn = Hij(j + 1, j).real();
                if (!std::isfinite(hn)) {
                    inf->iterations = its;
                    inf->status = HELM_BREAKDOWN;
                    return set_err(ctx, HELM_BREAKDOWN, "non-finite Arnoldi norm at iteration %d", its);
                }
                for (int i = 0; i < j; i++) {   // previous rotations
                    const cplx a = Hij(i, j), c = Hij(i + 1, j);
                    Hij(i, j) = cs[i] * a + sn[i] * c;
                    Hij(i + 1, j) = -std::conj(sn[i]) * a + cs[i] * c;
                }
                const cplx a = Hij(j, j), bb = Hij(j + 1, j);   // new rotation
                if (a == cplx(0, 0)) {
                    cs[j] = 0.0;
                    sn[j] = 1.0;
                    Hij(j, j) = bb;
                } else {
                    const double rho = sqrt(std::norm(a) + std::norm(bb));
                    const cplx ph = a / std::abs(a);
                    cs[j] = std::abs(a) / rho;
                    sn[j] = ph * std::conj(bb) / rho;
                    Hij(j, j) = ph * rho;
                }
                Hij(j + 1, j) = 0.0;
                g[j + 1] = -std::conj(sn[j]) * g[j];
                g[j] = cs[j] * g[j];
                est = std::abs(g[j + 1]) / beta0;
                if (inf->history && its - 1 < inf->history_cap) inf->history[its - 1] = est;
                jend = j + 1;
                if ((rtol > 0 && std::abs(g[j + 1]) <= rtol * beta0) || hn == 0.0 || its >= maxit) break;
            }
        } else {
        // DCGS2: u_0 = r; step j applies the operator to the candidate u_j (V slot j), then one
        // projection sweep and one update sweep over V; column j - 1 becomes final in step j, column j is used
        // tentatively (its subdiagonal = ||u_{j+1}|| before re-orthogonalisation) for the convergence test and is
        // closed with one extra projection sweep when the cycle ends.
        launch_copy(V, ctx->d_r, n, s);
        ctx->launches++;
        std::fill(g.begin(), g.end(), cplx(0, 0));
        constexpr int REC = 3 * NVMAX + 2;   // step record: final column j - 1, pending column j, nu_j, ||u_{j+1}||,
                                             // then a (column j of R)
        auto mark = [&](int k) { if (ctx->phases) cudaEventRecord(ctx->ev_ph[k], s); };
        // Several ranks: step j + 1 (it needs only device data) is queued before the host's update of step j, so the
        // devices never wait for the host's turnaround.  One rank: the turnaround is 0.3 % of a c3 step (93.59 vs
        // 93.56 applies/s with and without; with the tensor-core apply 386.5 vs 385.2), not worth a discarded apply at
        // convergence.
        const bool lookahead = ctx->multi && !ctx->phases;
        // folded norm (several ranks, HELM_GMRES_FOLD=0 disables): one collective per Arnoldi step -- the convergence
        // test uses column j - 1 once step j's record has made it final, one step later than the tentative test; the
        // price is one more discarded step at convergence
        const char* fenv = getenv("HELM_GMRES_FOLD");
        const bool lookahead_folded = lookahead && !(fenv && fenv[0] == '0');
        auto enqueue_step = [&](int j) -> int {
            z2* uj = V + (long long)j * n;
            int rc2;
            z2* zj = ctx->d_Z + (long long)j * n;   // B^-1 u_j, kept for the cycle's solution update
            mark(0);
            if ((rc2 = apply_impl(ctx, uj, zj))) return rc2;
            inf->applies++;
            mark(1);
            if ((rc2 = spmv_impl(ctx, zj, ctx->d_w))) return rc2;
            mark(2);
            NvtxRange nv_o("helm.orth");
            launch_multidot2(V, n, j + 1, uj, ctx->d_w, n, ctx->d_zpart, ctx->nblk, s);
            mark(3);
            launch_reduce_z2(ctx->d_zpart, ctx->nblk, j + 1, ctx->d_dots, s);
            if ((rc2 = allreduce(ctx, (double*)ctx->d_dots, 4 * (size_t)(j + 1)))) return rc2;   // both groups
            launch_dcgs2_coef(ctx->d_dots, j, ctx->d_H, ctx->d_ca, ctx->d_ce, ctx->d_sc, ctx->d_hout, s);
            mark(4);
            launch_dcgs2_update(V, n, j, ctx->d_w, ctx->d_ca, ctx->d_ce, ctx->d_sc, n, ctx->d_dpart, ctx->nblk, s);
            mark(5);
            ctx->launches += 4;
            // ||u_{j+1}|| feeds only the host's tentative convergence test.  On several ranks (lookahead) it costs a
            // collective of its own; the next step's projection sweep computes alpha_{j+1} = ||u_{j+1}||^2 inside the
            // one packed allreduce anyway, so the host tests the FINAL column instead and this norm is not formed.
            if (!lookahead_folded && (rc2 = finish_norm(ctx, ctx->d_hout + 2 * NVMAX + 1))) return rc2;
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(ctx->h_hc + (j & 1) * REC, ctx->d_hout, sizeof(z2) * REC, cudaMemcpyDeviceToHost, s));
            mark(6);
            CK(cudaEventRecord(ctx->ev_hc[j & 1], s));
            return HELM_OK;
        };
        // (lookahead: when step j turns out to be the cycle's last, step j + 1 is discarded and its record supplies the
        // final column j)
        if (lookahead && (rc = enqueue_step(0))) return rc;
        for (int j = 0; j < m; j++) {
            if (ctx->phases && j > 0) {   // the previous step's end (mark 6, kept in slot 7) to this step's start
                CK(cudaEventRecord(ctx->ev_ph[0], s));
                CK(cudaEventSynchronize(ctx->ev_ph[0]));
                float g = 0.f;
                cudaEventElapsedTime(&g, ctx->ev_ph[7], ctx->ev_ph[0]);
                ctx->ph_ms[7] += g;
            }
            const bool ahead = lookahead && j + 1 < m && its + 2 <= maxit;
            if (!lookahead && (rc = enqueue_step(j))) return rc;
            if (ahead && (rc = enqueue_step(j + 1))) return rc;
            its++;
            CK(cudaEventSynchronize(ctx->ev_hc[j & 1]));
            if (ctx->phases) {
                for (int k = 0; k < 6; k++) {
                    float t = 0.f;
                    cudaEventElapsedTime(&t, ctx->ev_ph[k], ctx->ev_ph[k + 1]);
                    ctx->ph_ms[k] += t;
                }
                std::swap(ctx->ev_ph[6], ctx->ev_ph[7]);
            }
            const z2* hc = ctx->h_hc + (j & 1) * REC;
            const double nu = hc[2 * NVMAX].x, un = lookahead_folded ? 1.0 : hc[2 * NVMAX + 1].x;
            if (!std::isfinite(nu) || !std::isfinite(un)) {
                inf->iterations = its;
                inf->status = HELM_BREAKDOWN;
                return set_err(ctx, HELM_BREAKDOWN, "non-finite Arnoldi norm at iteration %d", its);
            }
            Rzi(j, j) = nu;
            for (int i = 0; i < j; i++) Rzi(i, j) = cplx(hc[2 * NVMAX + 2 + i].x, hc[2 * NVMAX + 2 + i].y);
            if (j == 0) {
                g[0] = gkeep[0] = nu;   // ||r|| from the same sweep that normalises v_0
            } else {
                for (int i = 0; i <= j; i++) Rij(i, j - 1) = cplx(hc[i].x, hc[i].y);
                rotate_col(j - 1);
                est = std::abs(g[j]) / beta0;
                if (inf->history && its - 2 < inf->history_cap) inf->history[its - 2] = est;
                if (nu == 0.0) {   // invariant subspace found one column late: step j is discarded
                    its--;
                    jend = j;
                    break;
                }
                if (lookahead_folded && rtol > 0 && std::abs(g[j]) <= rtol * beta0) {
                    // folded norm: the final column j - 1 meets rtol -> steps j (and j + 1 if queued) are discarded
                    its--;
                    jend = j;
                    break;
                }
            }
            for (int i = 0; i <= j; i++) Rij(i, j) = cplx(hc[NVMAX + i].x, hc[NVMAX + i].y);
            jend = j + 1;
            if (!lookahead_folded) {
                Rij(j + 1, j) = un;   // tentative
                rotate_col(j);
                est = std::abs(g[j + 1]) / beta0;
                if (inf->history && its - 1 < inf->history_cap) inf->history[its - 1] = est;
            }
            const bool done_tent = !lookahead_folded && ((rtol > 0 && std::abs(g[j + 1]) <= rtol * beta0) || un == 0.0);
            if (done_tent || its >= maxit || j == m - 1) {
                if (ahead) {   // the queued step j + 1 (discarded) has closed column j
                    CK(cudaEventSynchronize(ctx->ev_hc[(j + 1) & 1]));
                    const z2* h1 = ctx->h_hc + ((j + 1) & 1) * REC;
                    for (int i = 0; i <= j + 1; i++) Rij(i, j) = cplx(h1[i].x, h1[i].y);
                    rotate_col(j);
                    est = std::abs(g[j + 1]) / beta0;
                    if (inf->history && its - 1 < inf->history_cap) inf->history[its - 1] = est;
                    break;
                }
                // close column j: re-orthogonalise u_{j+1} against V_{j+1}
                launch_multidot(V, n, j + 2, V + (long long)(j + 1) * n, n, ctx->d_zpart, ctx->nblk, s);
                launch_reduce_z(ctx->d_zpart, ctx->nblk, j + 2, ctx->d_dots, nullptr, nullptr, s);
                if ((rc = allreduce(ctx, (double*)ctx->d_dots, 2 * (size_t)(j + 2)))) return rc;
                launch_dcgs2_close(ctx->d_dots, j, ctx->d_H, ctx->d_hout, s);
                ctx->launches += 3;
                CK(cudaMemcpyAsync(ctx->h_pin, ctx->d_hout, sizeof(z2) * (j + 2), cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                for (int i = 0; i <= j + 1; i++) Rij(i, j) = cplx(ctx->h_pin[i].x, ctx->h_pin[i].y);
                rotate_col(j);
                est = std::abs(g[j + 1]) / beta0;
                if (inf->history && its - 1 < inf->history_cap) inf->history[its - 1] = est;
                break;
            }
        }
        }
        // H y = g (upper triangular), t = V y, x += B^-1 t
        for (int i = jend - 1; i >= 0; i--) {
            cplx acc = g[i];
            for (int c = i + 1; c < jend; c++) acc -= Hij(i, c) * y[c];
            y[i] = acc / Hij(i, i);
        }
        if (!ctx->orth_cgs2) {
            // B^-1 V y = B^-1 U R^-1 y = Z c with R c = y: the steps' preconditioned candidates, no extra apply
            for (int i = jend - 1; i >= 0; i--) {
                cplx acc = y[i];
                for (int c = i + 1; c < jend; c++) acc -= Rzi(i, c) * y[c];
                y[i] = acc / Rzi(i, i);
            }
            for (int i = 0; i < jend; i++) ctx->h_pin[i] = zmk(y[i].real(), y[i].imag());
            CK(cudaMemcpyAsync(ctx->d_y, ctx->h_pin, sizeof(z2) * jend, cudaMemcpyHostToDevice, s));
            launch_combine(ctx->d_Z, n, jend, ctx->d_y, ctx->d_t, n, s);
            launch_axpy(x, ctx->d_t, n, s);
            ctx->launches += 2;
        } else {
            for (int i = 0; i < jend; i++) ctx->h_pin[i] = zmk(y[i].real(), y[i].imag());
            CK(cudaMemcpyAsync(ctx->d_y, ctx->h_pin, sizeof(z2) * jend, cudaMemcpyHostToDevice, s));
            launch_combine(V, n, jend, ctx->d_y, ctx->d_t, n, s);
            ctx->launches++;
            if ((rc = apply_impl(ctx, ctx->d_t, ctx->d_z))) return rc;
            inf->applies++;
            launch_axpy(x, ctx->d_z, n, s);
            ctx->launches++;
        }
        double rn;
        if ((rc = residual_host(ctx, b, x, ctx->d_r, &rn))) return rc;
        cycles++;
        const double tr = rn / beta0;
        inf->iterations = its;
        inf->restarts = cycles - 1;
        inf->relres_est = est;
        inf->relres_true = tr;
        if (!std::isfinite(tr)) {
            inf->status = HELM_BREAKDOWN;
            return set_err(ctx, HELM_BREAKDOWN, "non-finite residual");
        }
        if (tr == 0.0 || (rtol > 0 && tr <= rtol)) {   // (an exactly zero residual ends the solve even at rtol = 0)
            inf->status = HELM_OK;
            return HELM_OK;
        }
        if (its >= maxit) {
            inf->status = HELM_NOT_CONVERGED;
            return HELM_NOT_CONVERGED;
        }
        beta = rn;
    }
}

// Algorithm 1: u <- u + B^-1 (b - A u)
int richardson_impl(helm_ctx* ctx, const z2* b, z2* x, double rtol, int maxit, helm_richardson_info* info)
{
    NvtxRange nv_("helm.richardson");
    if (!ctx->factored) return set_err(ctx, HELM_ESTATE, "richardson before helm_factor");
    if (maxit < 0) return set_err(ctx, HELM_EINVAL, "maxit >= 0");
    int rc;
    if ((rc = need_comm(ctx))) return rc;
    if ((rc = ensure_krylov(ctx, 0))) return rc;
    helm_richardson_info loc{};
    helm_richardson_info* inf = info ? info : &loc;
    inf->iterations = 0;
    inf->status = HELM_OK;
    inf->relres = 0.0;
    double beta0;
    if ((rc = norm_host(ctx, b, &beta0))) return rc;
    if (beta0 == 0.0) {
        CK(cudaMemsetAsync(x, 0, sizeof(z2) * ctx->n_local, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        return HELM_OK;
    }
    double rn;
    if ((rc = residual_host(ctx, b, x, ctx->d_r, &rn))) return rc;
    double rel = rn / beta0;
    int its = 0;
    // section 3(i): after a RAS step the residual lives on the interface band; restrict it there exactly
    // (the rest is rounding noise) and exchange only the band part of the apply's ghost frame
    const bool band = ctx->res_band && ctx->p.pou == HELM_POU_OWNER;
    while (rel > rtol && its < maxit) {
        if (band && its > 0) {
            const GridInfo& G = ctx->G;
            launch_band_mask(ctx->d_r, G.i0, G.i1, G.j0, G.j1, ctx->d_bandx, ctx->d_bandy, ctx->stream);
            ctx->launches++;
            ctx->band_xchg = ctx->multi;
        }
        rc = apply_impl(ctx, ctx->d_r, ctx->d_z);   // sum_j chi_j c_j
        ctx->band_xchg = false;
        if (rc) return rc;
        launch_axpy(x, ctx->d_z, ctx->n_local, ctx->stream);
        ctx->launches++;
        its++;
        if ((rc = residual_host(ctx, b, x, ctx->d_r, &rn))) return rc;
        rel = rn / beta0;
        if (inf->history && its - 1 < inf->history_cap) inf->history[its - 1] = rel;
        if (!std::isfinite(rel) || rel > 1e6) {
            inf->iterations = its;
            inf->relres = rel;
            inf->status = HELM_DIVERGED;
            return HELM_DIVERGED;
        }
    }
    inf->iterations = its;
    inf->relres = rel;
    inf->status = rel <= rtol ? HELM_OK : HELM_NOT_CONVERGED;
    return inf->status;
}

}  // namespace

// ===================================================================================================== C ABI

int helm_get_krylov_basis(helm_ctx* ctx, int nv, helm_z* out_dev)
{
    if (!ctx) return HELM_EINVAL;
    if (!ctx->d_V) return set_err(ctx, HELM_ESTATE, "helm_get_krylov_basis before helm_gmres");
    if (nv < 1 || nv > ctx->V_cap || !out_dev) return set_err(ctx, HELM_EINVAL, "helm_get_krylov_basis: nv %d", nv);
    CK(cudaMemcpyAsync(out_dev, ctx->d_V, sizeof(z2) * ctx->n_local * nv, cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return HELM_OK;
}

int helm_set_orthogonalisation(helm_ctx* ctx, int mode)
{
    if (!ctx) return HELM_EINVAL;
    if (mode != HELM_ORTH_DCGS2 && mode != HELM_ORTH_CGS2)
        return set_err(ctx, HELM_EINVAL, "helm_set_orthogonalisation: mode %d", mode);
    ctx->orth_cgs2 = mode == HELM_ORTH_CGS2;
    return HELM_OK;
}

// A collective entry point that fails on one rank of a loopback group aborts the group, so that its peers leave their
// barriers with an error instead of waiting forever (with NCCL the peers would hang in the collective; with the
// loopback transport they can be told).
static int coll(helm_ctx* ctx, int rc)
{
    if (rc < 0 && ctx && ctx->loop) ctx->loop->abort();
    return rc;
}

int helm_richardson(helm_ctx* ctx, const helm_z* b_dev, helm_z* x_dev, double rtol, int maxit,
                    helm_richardson_info* info)
{
    if (!ctx || !b_dev || !x_dev || (const void*)b_dev == (void*)x_dev)
        return coll(ctx, set_err(ctx, HELM_EINVAL, "helm_richardson: bad arguments"));
    return coll(ctx, richardson_impl(ctx, (const z2*)b_dev, (z2*)x_dev, rtol, maxit, info));
}
extern "C" {

int helm_plan_rank(const helm_params* params, int rank, int nranks, helm_plan* out)
{
    if (!params || !out) return HELM_EINVAL;
    GridInfo G;
    char err[256];
    int rc = compute_grid(*params, rank, nranks, G, err, sizeof(err));
    if (rc) return rc;
    out->gx = G.gx;
    out->gy = G.gy;
    out->rx = G.rx;
    out->ry = G.ry;
    out->owned_i0 = G.i0;
    out->owned_i1 = G.i1;
    out->owned_j0 = G.j0;
    out->owned_j1 = G.j1;
    out->ext_i0 = G.e_i0;
    out->ext_i1 = G.e_i1;
    out->ext_j0 = G.e_j0;
    out->ext_j1 = G.e_j1;
    out->halo_lo = G.halo_lo;
    out->halo_hi = G.halo_hi;
    for (int q = 0; q < 4; q++) out->nbr[q] = G.nbr[q];
    out->n_sub_local = (G.bx1 - G.bx0) * (G.by1 - G.by0);
    return HELM_OK;
}

int helm_halo_schedule(const helm_params* params, int rank, int nranks, int width, helm_msg* out, int cap)
{
    if (!params || (!out && cap > 0)) return HELM_EINVAL;
    GridInfo G;
    char err[256];
    int rc = compute_grid(*params, rank, nranks, G, err, sizeof(err));
    if (rc) return rc;
    return halo_schedule(G, width, out, cap);
}

int helm_nccl_unique_id(void* out128)
{
#ifdef HELM_HAVE_NCCL
    if (!out128) return HELM_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HELM_ENCCL;
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
    memcpy(out128, &id, sizeof(id));
    return HELM_OK;
#else
    (void)out128;
    return HELM_ENCCL;
#endif
}

static int setup_impl(const helm_params* params, int rank, int nranks, const void* nccl_unique_id, int loop_group,
                      void* cuda_stream, helm_ctx** out)
{
    NvtxRange nv_("helm.setup");
    if (!params || !out) return HELM_EINVAL;
    *out = nullptr;
    helm_ctx* ctx = new helm_ctx();
    ctx->p = *params;
    ctx->rank = rank;
    ctx->nranks = nranks;
    ctx->stream = (cudaStream_t)cuda_stream;
    *out = ctx;
    int rc = build_layout(ctx);
    if (rc) return rc;
    // nranks == 1 with an NCCL id: the multi-rank code path over a one-rank NCCL communicator (ghost-framed buffers,
    // NCCL allreduce of every inner product) -- the NCCL data plane exercised on a single GPU
    ctx->multi = nranks > 1 || (nranks == 1 && nccl_unique_id && loop_group < 0);
    if (ctx->multi && loop_group >= 0) {
        std::lock_guard<std::mutex> lk(g_loop_mu);
        LoopGroup*& L = g_loops[loop_group];
        if (!L) {
            L = new LoopGroup();
            L->nranks = nranks;
            L->ctx.assign(nranks, nullptr);
            L->slot.assign(nranks, nullptr);
        }
        if (L->nranks != nranks || L->ctx[rank])
            return set_err(ctx, HELM_EINVAL, "loopback group %d: rank %d of %d already taken or size mismatch", loop_group,
                           rank, nranks);
        L->ctx[rank] = ctx;
        L->members++;
        ctx->loop = L;
        ctx->loop_id = loop_group;
        ctx->has_comm = true;
        if ((rc = dalloc(ctx, &ctx->d_loop_tmp, 4 * NVMAX))) return rc;
    } else if (ctx->multi && nccl_unique_id) {
#ifdef HELM_HAVE_NCCL
        ncclUniqueId id;
        memcpy(&id, nccl_unique_id, sizeof(id));
        NK(ncclCommInitRank(&ctx->comm, nranks, id, rank));
        ctx->has_comm = true;
#else
        return set_err(ctx, HELM_ENCCL, "library built without NCCL");
#endif
    }
    // device buffers: global stencil, local stencils, descriptors
    const int nsub = (int)ctx->subs.size();
    if ((rc = dalloc(ctx, &ctx->d_A7, ctx->G.ns * (size_t)ctx->n_local)) || (rc = dalloc(ctx, &ctx->d_stc, ctx->n_stc)) ||
        (rc = dalloc(ctx, &ctx->d_desc, nsub)) || (rc = dalloc(ctx, &ctx->d_order, nsub)) ||
        (rc = dalloc(ctx, &ctx->d_err, 4)) || (rc = dalloc(ctx, &ctx->d_sq, 2)))
        return rc;
    if (ctx->multi) {
        const GridInfo& G = ctx->G;
        ctx->ext_stride = G.e_i1 - G.e_i0;
        ctx->n_ext = ctx->ext_stride * (G.e_j1 - G.e_j0);
        ctx->msg_cap = (long long)std::max(G.i1 - G.i0 + G.halo_lo + G.halo_hi, G.j1 - G.j0) * G.halo_hi;
        if ((rc = dalloc(ctx, &ctx->d_ext, ctx->n_ext))) return rc;
        CK(cudaMemsetAsync(ctx->d_ext, 0, sizeof(z2) * ctx->n_ext, ctx->stream));
        for (int q = 0; q < 4; q++)
            if ((rc = dalloc(ctx, &ctx->d_sendbuf[q], ctx->msg_cap)) || (rc = dalloc(ctx, &ctx->d_recvbuf[q], ctx->msg_cap)))
                return rc;
    }
    {
        // section 3(i): band flags, and the band sub-rectangles of every apply-frame message (send and receive side)
        const GridInfo& G = ctx->G;
        const std::vector<unsigned char> bx = band_flags(G, 0), by = band_flags(G, 1);
        if ((rc = dalloc(ctx, &ctx->d_bandx, G.N + 1)) || (rc = dalloc(ctx, &ctx->d_bandy, G.N + 1))) return rc;
        CK(cudaMemcpyAsync(ctx->d_bandx, bx.data(), G.N + 1, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(ctx->d_bandy, by.data(), G.N + 1, cudaMemcpyHostToDevice, ctx->stream));
        ctx->res_band = ctx->p.pou == HELM_POU_OWNER;
        if (ctx->multi && ctx->has_comm) {
            helm_msg msgs[4];
            const int nm = halo_schedule(G, 0, msgs, 4);
            for (int q = 0; q < nm; q++)
                for (int side = 0; side < 2; side++) {
                    const helm_msg& m = msgs[q];
                    std::vector<int4> rects;
                    if (side == 0) band_rects(bx, by, m.send_i0, m.send_i1, m.send_j0, m.send_j1, rects);
                    else band_rects(bx, by, m.recv_i0, m.recv_i1, m.recv_j0, m.recv_j1, rects);
                    auto& bm = side == 0 ? ctx->band_send[q] : ctx->band_recv[q];
                    std::vector<long long> off(rects.size() + 1, 0);
                    for (size_t r = 0; r < rects.size(); r++) {
                        const long long a = (long long)(rects[r].y - rects[r].x) * (rects[r].w - rects[r].z);
                        off[r + 1] = off[r] + a;
                        bm.max_area = std::max(bm.max_area, a);
                    }
                    bm.n = (int)rects.size();
                    bm.total = off.back();
                    if (bm.n > 0) {
                        if ((rc = dalloc(ctx, &bm.d_rects, bm.n)) || (rc = dalloc(ctx, &bm.d_off, bm.n + 1))) return rc;
                        CK(cudaMemcpyAsync(bm.d_rects, rects.data(), sizeof(int4) * bm.n, cudaMemcpyHostToDevice,
                                           ctx->stream));
                        CK(cudaMemcpyAsync(bm.d_off, off.data(), sizeof(long long) * (bm.n + 1), cudaMemcpyHostToDevice,
                                           ctx->stream));
                    }
                }
            CK(cudaStreamSynchronize(ctx->stream));   // the host vectors die here
        }
        CK(cudaStreamSynchronize(ctx->stream));
    }
    // processing order: most expensive first (static round-robin over persistent CTAs)
    std::vector<int> order(nsub);
    for (int i = 0; i < nsub; i++) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const SubDesc &x = ctx->subs[a], &y = ctx->subs[b];
        return (long long)(x.nb + x.hi - x.lo) * x.m * x.m > (long long)(y.nb + y.hi - y.lo) * y.m * y.m;
    });
    CK(cudaMemcpyAsync(ctx->d_desc, ctx->subs.data(), sizeof(SubDesc) * nsub, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_order, order.data(), sizeof(int) * nsub, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(ctx->d_err, 0, 4 * sizeof(int), ctx->stream));
    launch_assemble_global(ctx->geom, ctx->d_A7, ctx->G.ns, ctx->G.i0, ctx->G.i1, ctx->G.j0, ctx->G.j1, ctx->stream);
    launch_assemble_local(ctx->geom, ctx->d_desc, nsub, ctx->d_stc, (int)ctx->max_n, ctx->stream);
    CK(cudaGetLastError());
    {
        // constant interior stencil: nodes whose cells all lie in Omega_int (ceil lo_u + 1 .. floor hi_u - 1) have
        // gamma = 1 everywhere around them; copy the coefficients of one such owned row from A so the SpMV fast
        // path is bitwise identical to A
        const GridInfo& G = ctx->G;
        const int clo = (int)ceil(G.lo_u) + 1, chi = (int)floor(G.hi_u);
        const int a = std::max(G.i0, clo), b = std::min(G.i1, chi);
        const int c = std::max(G.j0, clo), d = std::min(G.j1, chi);
        if (a < b && c < d) {
            const long long r = (long long)(a - G.i0) + (long long)(G.i1 - G.i0) * (c - G.j0);
            for (int q = 0; q < G.ns; q++)
                CK(cudaMemcpyAsync(&ctx->c7[q], ctx->d_A7 + q * ctx->n_local + r, sizeof(z2), cudaMemcpyDeviceToHost,
                                   ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            ctx->cst[0] = a;
            ctx->cst[1] = b;
            ctx->cst[2] = c;
            ctx->cst[3] = d;
        }
        // the same for the local operators: couplings of one constant-range node of the first subdomain that
        // has one (all such nodes are computed from gamma = 1 with exact arithmetic: identical bits)
        for (const SubDesc& sd : ctx->subs) {
            if (sd.cx0 >= sd.cx1 || sd.cy0 >= sd.cy1) continue;
            const z2* row = ctx->d_stc + sd.stc_off + (long long)sd.cy0 * sd.ns * sd.m + sd.cx0;
            z2* dst[6] = {&ctx->lcS, &ctx->lcSW, &ctx->lcN, &ctx->lcNE, &ctx->lcSE, &ctx->lcNW};
            const int sl[6] = {SL_S, SL_SW, SL_N, SL_NE, SL_SE, SL_NW};
            for (int q = 0; q < (sd.ns == 9 ? 6 : 4); q++)
                CK(cudaMemcpyAsync(dst[q], row + sl[q] * sd.m, sizeof(z2), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            break;
        }
    }
    // apply launch configuration
    int nsm = 148;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // the one-CTA-per-subdomain kernel may not fit very wide blocks (its ring holds whole columns); that is only an
    // error when the cluster-split kernel below does not take over
    apply_configure(ctx->m_max, ctx->ap_nslots, &ctx->ap_block, &ctx->ap_smem, &ctx->ap_slot, &ctx->ap_occ);
    if (cudaGetLastError() != cudaSuccess) ctx->ap_occ = 0;
    // Ring depth: two slots when every SM hosts as many CTAs as fit (many subdomains); with fewer subdomains than CTA
    // slots each CTA may stream deeper -- take the deepest ring (<= 6 slots) that still leaves one CTA slot per SM to
    // spare over the CTAs the subdomains need.  c2 (256 subdomains, ~2 CTAs/SM): 2 slots 0.617 ms, 3 0.522, 4 0.499,
    // 6 0.518, 8 (one CTA/SM) 0.838.  HELM_APPLY_SLOTS overrides.
    if (const char* e = getenv("HELM_APPLY_SLOTS")) {
        ctx->ap_nslots = std::max(2, atoi(e));
        apply_configure(ctx->m_max, ctx->ap_nslots, &ctx->ap_block, &ctx->ap_smem, &ctx->ap_slot, &ctx->ap_occ);
        if (cudaGetLastError() != cudaSuccess) ctx->ap_occ = 0;
    } else if (ctx->ap_occ > 0) {
        const int cps = (std::min(nsub, nsm * ctx->ap_occ) + nsm - 1) / nsm;   // CTAs per SM the grid needs
        for (int ns = 6; ns > 2; ns--) {
            int blk, sm, sl, occ = 0;
            apply_configure(ctx->m_max, ns, &blk, &sm, &sl, &occ);
            if (cudaGetLastError() != cudaSuccess) continue;
            if (occ >= cps + 1) {
                ctx->ap_nslots = ns;
                ctx->ap_block = blk;
                ctx->ap_smem = sm;
                ctx->ap_slot = sl;
                ctx->ap_occ = occ;
                break;
            }
        }
    }
    // persistent CTAs: as many as fit, then trimmed so that every CTA gets the same number of subdomains (round-robin
    // over the cost-sorted order); measured at c3 (apply ms): 1 GPU 296 CTAs 9.63 -> 293 9.33; the 1/4 shard
    // (1024 subdomains) 296 -> 256 CTAs 2.56 -> 2.28; the 1/8 shard 1.24 -> 1.15 (scripts/shard_timing.py)
    ctx->ap_grid = std::min(nsub, nsm * std::max(ctx->ap_occ, 1));
    {
        const int per = (nsub + ctx->ap_grid - 1) / std::max(ctx->ap_grid, 1);
        ctx->ap_grid = (nsub + per - 1) / per;
    }
    ctx->nblk = nsm * 4;
    // Fewer subdomains than SMs (the paper's regime): split every subdomain over a cluster of 2G CTAs (G per chain).
    // Among the G <= 8 whose clusters are all resident at once, take the smallest that keeps >= 80 % of the SMs
    // streaming (more G only adds exchange partners), else the largest; each CTA's ring takes the shared memory its
    // share of an SM leaves.  HELM_SPLIT_G overrides (0 = off).
    // D28: factor sharing, and the shared-factor apply on the tensor cores when the classes are large
    if (const char* e = getenv("HELM_SHARE_FACTORS")) ctx->share = e[0] != '0';
    {
        const long long nsub_global = (long long)ctx->G.P[0] * ctx->G.P[1];
        bool b = nsub_global >= nsm;   // c2 (256 subdomains): 0.365 vs 0.455 ms streaming; c1 (16): 0.31 vs 0.10
        if (const char* e = getenv("HELM_APPLY_BATCH")) b = e[0] == '1';
        ctx->batched = b && ctx->share && ctx->m_max <= 128;
    }
    const char* env_g = getenv("HELM_SPLIT_G");
    const int gforce = env_g ? atoi(env_g) : -1;
    if (!ctx->batched && (nsub < nsm || gforce > 0)) {
        int gbest = 0, cbest = 1;
        for (int G = 1; G <= 8; G++) {
            if (gforce >= 0 && G != gforce) continue;
            const int cps = (nsub * 2 * G + nsm - 1) / nsm;   // CTAs per SM if all are resident
            int blk, sm, sl, ncw, nss;
            if (split_configure(ctx->m_max, G, cps, &blk, &sm, &sl, &ncw, &nss)) continue;
            if (gforce > 0 || max_split_clusters(G, blk, sm) >= nsub) {
                gbest = G;
                cbest = cps;
                if (5 * nsub * 2 * G >= 4 * nsm) break;
            }
        }
        if (gbest > 0 && !split_configure(ctx->m_max, gbest, cbest, &ctx->sp_block, &ctx->sp_smem, &ctx->sp_slot,
                                          &ctx->sp_ncw, &ctx->sp_nss))
            ctx->sp_G = gbest;
        cudaGetLastError();
    }
    if (ctx->sp_G == 0 && ctx->ap_occ < 1)
        return set_err(ctx, HELM_ECUDA, "apply kernel does not fit on an SM (smem %d)", ctx->ap_smem);
    // overlap of the multi-rank apply with its halo exchange: split the subdomains into those whose full box lies in
    // the owned rectangle (no ghost input) and the rest, and the persistent CTA slots in proportion to their bytes
    const char* ovl = getenv("HELM_APPLY_OVERLAP");
    if (ctx->multi && ctx->has_comm && !(ovl && ovl[0] == '0')) {
        const GridInfo& G = ctx->G;
        std::vector<int> oi, ob;
        double ci = 0, cb = 0;
        for (int w : order) {
            const SubDesc& sd = ctx->subs[w];
            const bool inside = sd.gx0 >= G.i0 && sd.gx0 + sd.m <= G.i1 && sd.gy0 >= G.j0 && sd.gy0 + sd.nb <= G.j1;
            const double c = (double)(sd.nb + sd.hi - sd.lo) * sd.m * sd.m;
            if (inside) {
                oi.push_back(w);
                ci += c;
            } else {
                ob.push_back(w);
                cb += c;
            }
        }
        const int S = nsm * std::max(ctx->ap_occ, 1);
        if (!oi.empty() && !ob.empty() && S >= 2) {
            int sb = (int)std::lround(S * cb / (ci + cb));
            sb = std::max(1, std::min(S - 1, sb));
            auto trim = [](int n, int slots) {
                slots = std::max(1, std::min(slots, n));
                const int per = (n + slots - 1) / slots;
                return (n + per - 1) / per;
            };
            ctx->n_int = (int)oi.size();
            ctx->n_bnd = (int)ob.size();
            ctx->grid_int = trim(ctx->n_int, S - sb);
            ctx->grid_bnd = trim(ctx->n_bnd, sb);
            oi.insert(oi.end(), ob.begin(), ob.end());
            if ((rc = dalloc(ctx, &ctx->d_order_ov, nsub))) return rc;
            CK(cudaMemcpyAsync(ctx->d_order_ov, oi.data(), sizeof(int) * nsub, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
            for (auto& e : ctx->ev_ov) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->overlap = true;
        }
    }
    if (const char* dbg = getenv("HELM_DEBUG_CONFIG"))   // diagnostic: the apply configuration this rank chose
        if (dbg[0] == '1')
            fprintf(stderr,
                    "helm rank %d: %d subdomains, m_max %d; apply %s: grid %d block %d smem %d slot %d slots %d "
                    "(occ %d); split G %d block %d smem %d slot %d slots %d; overlap %d (%d interior)\n",
                    ctx->rank, nsub, ctx->m_max, ctx->sp_G > 0 ? "cluster-split" : "k_apply", ctx->ap_grid,
                    ctx->ap_block, ctx->ap_smem, ctx->ap_slot, ctx->ap_nslots, ctx->ap_occ, ctx->sp_G, ctx->sp_block,
                    ctx->sp_smem, ctx->sp_slot, ctx->sp_nss, (int)ctx->overlap, ctx->n_int);
    long long scr = (size_t)std::max(ctx->ap_grid, ctx->grid_int + ctx->grid_bnd) * ctx->scratch_per_cta;
    if (ctx->sp_G > 0) {
        long long per = 0;
        for (const SubDesc& sd : ctx->subs) per = std::max(per, (long long)(sd.hi - sd.lo + 1) * ((sd.m + ctx->sp_G - 1) / ctx->sp_G));
        ctx->scratch_per_cta = per;
        scr = (long long)nsub * 2 * ctx->sp_G * per;
    }
    if ((rc = dalloc(ctx, &ctx->d_scratch, (size_t)scr))) return rc;
    if (ctx->p.pou == HELM_POU_RAMP) {
        // per axis and node index: the (<= 2, ascending) blocks whose ramp chi is positive there
        const GridInfo& G = ctx->G;
        if ((rc = dalloc(ctx, &ctx->d_pou, ctx->pou_len)) || (rc = dalloc(ctx, &ctx->d_candx, 2 * (G.N + 1))) ||
            (rc = dalloc(ctx, &ctx->d_candy, 2 * (G.N + 1))))
            return rc;
        if (ctx->multi) {
            // the sum over covering subdomains crosses rank boundaries: it needs the additive reverse exchange, so
            // communication-free shards (the _ext entry points) cannot run the ramp PoU
            if (!ctx->has_comm) return set_err(ctx, HELM_EINVAL, "ramp PoU on several ranks needs a communicator");
            if ((rc = dalloc(ctx, &ctx->d_cext, ctx->n_ext))) return rc;
        }
        for (int ax = 0; ax < 2; ax++) {
            std::vector<int> cand(2 * (G.N + 1), -1);
            for (int x = 0; x <= G.N; x++) {
                int k = 0;
                for (int b = 0; b < G.P[ax] && k < 2; b++)
                    if (chi_ramp(x, G.st[ax][b], G.st[ax][b + 1], G.wo, b > 0, b < G.P[ax] - 1) > 0.0) cand[2 * x + k++] = b;
            }
            CK(cudaMemcpyAsync(ax ? ctx->d_candy : ctx->d_candx, cand.data(), sizeof(int) * cand.size(),
                               cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return HELM_OK;
}

int helm_factor_classes(const helm_ctx* ctx, long long* out6, int* class_of, int cap)
{
    if (!ctx || !out6) return HELM_EINVAL;
    if (!ctx->factored) return HELM_ESTATE;
    out6[0] = (long long)ctx->cls_rep.size();
    out6[1] = ctx->batched ? 1 : 0;
    out6[2] = ctx->bt_ntiles;
    out6[3] = 16LL * (ctx->n_dinv + ctx->dinvB_len);
    // algorithmic flops of one apply: 8 m^2 real flops (one complex m x m GEMV) per block step of every subdomain
    long long fl = 0, issued = 0;
    for (const SubDesc& d : ctx->subs) fl += 8LL * d.m * d.m * (d.nb + d.hi - d.lo);
    if (ctx->batched)
        for (int c = 0; c < (int)ctx->cls_rep.size(); c++) {
            // the tensor-core apply computes full padded tiles: ceil(members / 16) tiles of 16 columns, mp x mp blocks
            const SubDesc& d = ctx->subs[ctx->cls_rep[c]];
            long long nm = 0;
            for (int k : ctx->cls_of) nm += k == c;
            const long long mp = (d.m + 7) / 8 * 8;
            issued += (nm + ctx->bt_w - 1) / ctx->bt_w * ctx->bt_w * 8LL * mp * mp * (d.nb + d.hi - d.lo);
        }
    out6[4] = fl;
    out6[5] = issued;
    if (class_of)
        for (int j = 0; j < (int)ctx->cls_of.size() && j < cap; j++) class_of[j] = ctx->cls_of[j];
    return HELM_OK;
}

int helm_comm_info(const helm_ctx* ctx, int* transport, int* comm_nranks, int* comm_rank)
{
    if (!ctx) return HELM_EINVAL;
    int t = HELM_TRANSPORT_NONE, n = 1, r = 0;
    if (ctx->loop) {
        t = HELM_TRANSPORT_LOOPBACK;
        n = ctx->loop->nranks;
        r = ctx->rank;
    } else if (ctx->multi && !ctx->has_comm) {
        t = HELM_TRANSPORT_SHARD;
        n = ctx->nranks;
        r = ctx->rank;
    }
#ifdef HELM_HAVE_NCCL
    else if (ctx->comm) {
        t = HELM_TRANSPORT_NCCL;
        if (ncclCommCount(ctx->comm, &n) != ncclSuccess || ncclCommUserRank(ctx->comm, &r) != ncclSuccess)
            return HELM_ENCCL;
    }
#endif
    if (transport) *transport = t;
    if (comm_nranks) *comm_nranks = n;
    if (comm_rank) *comm_rank = r;
    return HELM_OK;
}

int helm_nccl_selftest(helm_ctx* ctx, long long nelem, int nmsg, long long* mismatches)
{
    if (!ctx || nmsg < 1 || nmsg > 4 || nelem < nmsg || !mismatches) return HELM_EINVAL;   // counts nelem - q >= 1
    z2 *sb[4] = {}, *rb[4] = {};
    size_t cnt[4];
    int peers[4];
    int rc = HELM_OK;
    std::vector<z2> h((size_t)nelem), g((size_t)nelem);
    *mismatches = 0;
    for (int a = 0; a < nmsg && !rc; a++) {
        cnt[a] = (size_t)nelem - a;   // distinct sizes per message
        peers[a] = ctx->rank;         // send-to-self: every rank of the communicator runs the same code path
        if ((rc = dalloc(ctx, &sb[a], nelem)) || (rc = dalloc(ctx, &rb[a], nelem))) break;
        for (long long e = 0; e < nelem; e++) h[e] = zmk(1000.0 * a + e, -0.5 * e);
        if (cudaMemcpyAsync(sb[a], h.data(), sizeof(z2) * nelem, cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess ||
            cudaMemsetAsync(rb[a], 0, sizeof(z2) * nelem, ctx->stream) != cudaSuccess)
            rc = set_err(ctx, HELM_ECUDA, "selftest staging");
    }
    if (!rc) rc = nccl_sendrecv(ctx, nmsg, peers, sb, cnt, rb, cnt, ctx->stream);
    for (int a = 0; a < nmsg && !rc; a++) {
        if (cudaMemcpyAsync(g.data(), rb[a], sizeof(z2) * nelem, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
            cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
            rc = set_err(ctx, HELM_ECUDA, "selftest readback");
            break;
        }
        for (long long e = 0; e < nelem; e++) {
            const z2 want = e < (long long)cnt[a] ? zmk(1000.0 * a + e, -0.5 * e) : zmk(0, 0);
            if (g[e].x != want.x || g[e].y != want.y) (*mismatches)++;
        }
    }
    for (int a = 0; a < 4; a++) {
        if (sb[a]) cudaFree(sb[a]);
        if (rb[a]) cudaFree(rb[a]);
    }
    return rc;
}

int helm_set_residual_band(helm_ctx* ctx, int on)
{
    if (!ctx || on < 0 || on > 1) return set_err(ctx, HELM_EINVAL, "helm_set_residual_band: on must be 0 or 1");
    if (on && ctx->p.pou != HELM_POU_OWNER)
        return set_err(ctx, HELM_EINVAL, "the residual band (section 3(i)) needs the owner partition of unity");
    ctx->res_band = on == 1;
    return HELM_OK;
}

int helm_comm_counters(helm_ctx* ctx, int reset, long long* out4)
{
    if (!ctx || !out4) return HELM_EINVAL;
    out4[0] = ctx->xc_sent;
    out4[1] = ctx->xc_recv;
    out4[2] = ctx->xc_msgs;
    out4[3] = ctx->xc_allreduce;
    if (reset) ctx->xc_sent = ctx->xc_recv = ctx->xc_msgs = ctx->xc_allreduce = 0;
    return HELM_OK;
}

int helm_halo_band_counts(const helm_params* params, int rank, int nranks, long long* out4)
{
    if (!params || !out4) return HELM_EINVAL;
    GridInfo G;
    char err[256];
    int rc = compute_grid(*params, rank, nranks, G, err, sizeof(err));
    if (rc) return rc;
    const std::vector<unsigned char> bx = band_flags(G, 0), by = band_flags(G, 1);
    helm_msg msgs[4];
    const int nm = halo_schedule(G, 0, msgs, 4);
    long long sf = 0, sb = 0, rf = 0, rb = 0;
    for (int q = 0; q < nm; q++) {
        const helm_msg& m = msgs[q];
        std::vector<int4> rs, rr;
        band_rects(bx, by, m.send_i0, m.send_i1, m.send_j0, m.send_j1, rs);
        band_rects(bx, by, m.recv_i0, m.recv_i1, m.recv_j0, m.recv_j1, rr);
        sf += (long long)(m.send_i1 - m.send_i0) * (m.send_j1 - m.send_j0);
        rf += (long long)(m.recv_i1 - m.recv_i0) * (m.recv_j1 - m.recv_j0);
        sb += rects_area(rs);
        rb += rects_area(rr);
    }
    out4[0] = sf;
    out4[1] = sb;
    out4[2] = rf;
    out4[3] = rb;
    return HELM_OK;
}

int helm_halo_band_rects(const helm_params* params, int rank, int nranks, int msg, int side, int* out, int cap)
{
    if (!params || msg < 0 || msg >= 4 || side < 0 || side > 1) return HELM_EINVAL;
    GridInfo G;
    char err[256];
    int rc = compute_grid(*params, rank, nranks, G, err, sizeof(err));
    if (rc) return rc;
    helm_msg msgs[4];
    const int nm = halo_schedule(G, 0, msgs, 4);
    if (msg >= nm) return HELM_EINVAL;
    const helm_msg& m = msgs[msg];
    std::vector<int4> r;
    if (side == 0) band_rects(band_flags(G, 0), band_flags(G, 1), m.send_i0, m.send_i1, m.send_j0, m.send_j1, r);
    else band_rects(band_flags(G, 0), band_flags(G, 1), m.recv_i0, m.recv_i1, m.recv_j0, m.recv_j1, r);
    for (int q = 0; q < (int)r.size() && q < cap; q++) {
        out[4 * q] = r[q].x;
        out[4 * q + 1] = r[q].y;
        out[4 * q + 2] = r[q].z;
        out[4 * q + 3] = r[q].w;
    }
    return (int)r.size();
}

int helm_get_layout(const helm_ctx* ctx, helm_layout* out)
{
    if (!ctx || !out) return HELM_EINVAL;
    const GridInfo& G = ctx->G;
    out->n_free_global = (long long)G.nf * G.nf;
    out->N_cells = G.N;
    out->n_int = G.n_int;
    out->n_ovlp = G.wo;
    out->n_pml = G.wp;
    out->owned_i0 = G.i0;
    out->owned_i1 = G.i1;
    out->owned_j0 = G.j0;
    out->owned_j1 = G.j1;
    out->n_local = ctx->n_local;
    out->n_sub = G.P[0] * G.P[1];
    out->n_sub_local = (int)ctx->subs.size();
    out->m_max = ctx->m_max;
    out->local_unknowns = ctx->local_unknowns;
    out->factor_bytes = ctx->n_dinv * 16;
    out->apply_bytes = ctx->apply_bytes;
    out->band_bytes = ctx->band_bytes + 16LL * ctx->n_local;
    // SpMV: x read + y write per row; rows off the constant interior stencil also read 7 coefficients
    const long long ncst = (long long)std::max(0, ctx->cst[1] - ctx->cst[0]) * std::max(0, ctx->cst[3] - ctx->cst[2]);
    out->spmv_bytes = 16LL * 2 * ctx->n_local + 16LL * G.ns * (ctx->n_local - ncst);
    out->stencil_slots = G.ns;
    out->overlap_interior = ctx->overlap ? ctx->n_int : 0;
    out->factor_flop = 0;
    // what helm_factor computes: one factorisation per class (D28) once the classes are known, else every subdomain
    if (!ctx->cls_rep.empty())
        for (int j : ctx->cls_rep) out->factor_flop += 8LL * ctx->subs[j].nb * ctx->subs[j].m * ctx->subs[j].m * ctx->subs[j].m;
    else
        for (const SubDesc& sd : ctx->subs) out->factor_flop += 8LL * sd.nb * sd.m * sd.m * sd.m;
    return HELM_OK;
}

int helm_rhs(helm_ctx* ctx, int nsrc, const double* xy_host, const helm_z* amp_host, double sigma, helm_z* b_dev)
{
    if (!ctx || nsrc < 0 || (nsrc > 0 && (!xy_host || !amp_host)) || !b_dev || !(sigma > 0))
        return set_err(ctx, HELM_EINVAL, "helm_rhs: bad arguments");
    const GridInfo& G = ctx->G;
    double* d_xy = nullptr;
    z2* d_amp = nullptr;
    z2* d_f = nullptr;
    const long long nfw = (long long)(G.i1 - G.i0 + 2) * (G.j1 - G.j0 + 2);
    auto body = [&]() -> int {
        int rc;
        if ((rc = dalloc(ctx, &d_xy, 2 * (size_t)std::max(nsrc, 1))) || (rc = dalloc(ctx, &d_amp, std::max(nsrc, 1))) ||
            (rc = dalloc(ctx, &d_f, nfw)))
            return rc;
        if (nsrc > 0) {
            CK(cudaMemcpyAsync(d_xy, xy_host, sizeof(double) * 2 * nsrc, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaMemcpyAsync(d_amp, amp_host, sizeof(z2) * nsrc, cudaMemcpyHostToDevice, ctx->stream));
        }
        launch_rhs(ctx->geom, nsrc, d_xy, d_amp, sigma, d_f, (z2*)b_dev, G.i0, G.i1, G.j0, G.j1, ctx->stream);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(ctx->stream));
        return HELM_OK;
    };
    const int rc = body();
    cudaFree(d_xy);   // temporaries are released on every path
    cudaFree(d_amp);
    cudaFree(d_f);
    return rc;
}

// D28: group the subdomains into classes whose assembled local operators are bitwise equal.  Candidates share every
// shape field of the descriptor (block sizes, twist, owned ranges, constant-coupling range, stencil width, impedance
// faces); k_stencil_eq then compares each candidate's whole local stencil with its class representative, bit for bit,
// and a candidate that differs anywhere starts a class of its own.  Fills cls_rep / cls_of (HELM_SHARE_FACTORS=0: one
// class per subdomain).
static int build_classes(helm_ctx* ctx)
{
    const int n = (int)ctx->subs.size();
    ctx->cls_rep.clear();
    ctx->cls_of.assign(n, -1);
    if (!ctx->share) {
        for (int j = 0; j < n; j++) {
            ctx->cls_of[j] = j;
            ctx->cls_rep.push_back(j);
        }
        return HELM_OK;
    }
    auto key = [](const SubDesc& d) {
        return std::array<int, 16>{d.m, d.nb, d.tw, d.lo, d.hi, d.olo, d.ohi, d.cx0, d.cx1, d.cy0, d.cy1, d.ns, d.imp,
                                   d.flags, d.fx1 - d.fx0, d.fy1 - d.fy0};
    };
    std::map<std::array<int, 16>, std::vector<int>> groups;
    for (int j = 0; j < n; j++) groups[key(ctx->subs[j])].push_back(j);
    std::vector<std::vector<int>> pending;
    for (auto& kv : groups) pending.push_back(kv.second);
    int2* d_pairs = nullptr;
    int* d_diff = nullptr;
    int rc = HELM_OK;
    if ((rc = dalloc(ctx, &d_pairs, n)) || (rc = dalloc(ctx, &d_diff, n))) {
        cudaFree(d_pairs);
        return rc;
    }
    std::vector<int2> pairs;
    std::vector<int> diff;
    while (!pending.empty() && rc == HELM_OK) {
        // one comparison pass over every pending group: member vs the group's first subdomain
        pairs.clear();
        for (auto& grp : pending)
            for (size_t q = 1; q < grp.size(); q++) pairs.push_back(make_int2(grp[q], grp[0]));
        diff.assign(pairs.size(), 0);
        if (!pairs.empty()) {
            if (cudaMemcpyAsync(d_pairs, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice,
                                ctx->stream) != cudaSuccess) {
                rc = set_err(ctx, HELM_ECUDA, "class detection: copy failed");
                break;
            }
            launch_stencil_eq(ctx->d_desc, ctx->d_stc, d_pairs, (int)pairs.size(), d_diff, ctx->stream);
            if (cudaMemcpyAsync(diff.data(), d_diff, sizeof(int) * diff.size(), cudaMemcpyDeviceToHost, ctx->stream) !=
                    cudaSuccess ||
                cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
                rc = set_err(ctx, HELM_ECUDA, "class detection: %s", cudaGetErrorString(cudaGetLastError()));
                break;
            }
        }
        std::vector<std::vector<int>> next;
        size_t p = 0;
        for (auto& grp : pending) {
            const int c = (int)ctx->cls_rep.size();
            ctx->cls_rep.push_back(grp[0]);
            ctx->cls_of[grp[0]] = c;
            std::vector<int> rest;
            for (size_t q = 1; q < grp.size(); q++, p++) {
                if (diff[p]) rest.push_back(grp[q]);
                else ctx->cls_of[grp[q]] = c;
            }
            if (!rest.empty()) next.push_back(rest);
        }
        pending.swap(next);
    }
    cudaFree(d_pairs);
    cudaFree(d_diff);
    return rc;
}

// The shared-factor apply (batch.cu): class factors in the batch layout, tiles of BATCH_NT members of one class
// (cost-sorted; on several ranks with the overlapped apply the interior subdomains' tiles first), launch
// configuration and per-CTA scratch.
static int setup_batch(helm_ctx* ctx)
{
    int rc;
    const int ncls = (int)ctx->cls_rep.size();
    std::vector<BatchClass> bc(ncls);
    long long off = 0;
    int mpmax = 0;
    for (int c = 0; c < ncls; c++) {
        const SubDesc& r = ctx->subs[ctx->cls_rep[c]];
        bc[c].rep = ctx->cls_rep[c];
        bc[c].mp = (r.m + 7) / 8 * 8;
        bc[c].S = bc[c].mp + 2;
        bc[c].off = off;
        off += (long long)r.nb * bc[c].mp * bc[c].S;
        mpmax = std::max(mpmax, bc[c].mp);
    }
    ctx->dinvB_len = off;
    ctx->bt_mpmax = mpmax;
    if ((rc = dalloc(ctx, &ctx->d_dinvB, off)) || (rc = dalloc(ctx, &ctx->d_bcls, ncls))) return rc;
    for (int c = 0; c < ncls; c++) {
        const SubDesc& r = ctx->subs[bc[c].rep];
        launch_relayout_batch(ctx->d_dinv, r.fac_off, r.m, r.nb, ctx->d_dinvB + bc[c].off, bc[c].mp, bc[c].S,
                              ctx->stream);
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->d_bcls, bc.data(), sizeof(BatchClass) * ncls, cudaMemcpyHostToDevice, ctx->stream));
    batch_configure(mpmax, &ctx->bt_block, &ctx->bt_smem, &ctx->bt_slot, &ctx->bt_nslots, &ctx->bt_occ);
    if (ctx->bt_occ < 1) return set_err(ctx, HELM_ECUDA, "shared-factor apply kernel does not fit (m_max %d)", mpmax);
    int nsm = 148, dev = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const int slots = nsm * ctx->bt_occ;
    // tiles: the members of each class in subdomain order, W at a time; sorted by cost, most expensive first.  Few tiles
    // per CTA slot (a rank of a large decomposition): each tile on a cluster of two CTAs running the twisted halves
    // (split, batch.cu) once 16-wide tiles would fill at most half the slots, and 8-wide tiles (one DMMA column tile)
    // once they would fill at most a sixth.  Measured at c3, apply ms per rank (scripts/batch_tile_sweep.sh), 1 / 2 / 4
    // / 8 ranks: W16 1.47 / 0.93 / 0.92 / 0.91; W16 split 1.49 / 0.76 / 0.51 / 0.50; W8 split 2.66 / 1.34 / 0.67 / 0.44.
    // A subdomain's result depends on neither choice.  HELM_BATCH_W / HELM_BATCH_SPLIT override.
    {
        std::vector<long long> cnt(ncls, 0);
        for (int k : ctx->cls_of) cnt[k]++;
        long long t16 = 0;
        for (long long c : cnt) t16 += (c + BATCH_NT - 1) / BATCH_NT;
        ctx->bt_split = 2 * t16 <= slots ? 1 : 0;
        ctx->bt_w = 6 * t16 <= slots ? 8 : BATCH_NT;
        if (const char* e = getenv("HELM_BATCH_W")) ctx->bt_w = atoi(e) == 8 ? 8 : BATCH_NT;
        if (const char* e = getenv("HELM_BATCH_SPLIT")) ctx->bt_split = e[0] == '1';
    }
    const int W = ctx->bt_w;
    std::vector<BatchTile> tiles;
    std::vector<int> members;
    auto make_tiles = [&](const std::vector<int>& set) {
        std::vector<std::vector<int>> per(ncls);
        for (int j : set) per[ctx->cls_of[j]].push_back(j);
        std::vector<BatchTile> t;
        for (int c = 0; c < ncls; c++)
            for (size_t q = 0; q < per[c].size(); q += W) {
                BatchTile bt{};
                bt.cls = c;
                bt.first = (int)members.size();
                bt.cnt = (int)std::min<size_t>(W, per[c].size() - q);
                members.insert(members.end(), per[c].begin() + q, per[c].begin() + q + bt.cnt);
                t.push_back(bt);
            }
        auto cost = [&](const BatchTile& x) {
            const SubDesc& d = ctx->subs[bc[x.cls].rep];
            return (long long)(d.nb + d.hi - d.lo) * bc[x.cls].mp * bc[x.cls].mp;
        };
        std::stable_sort(t.begin(), t.end(), [&](const BatchTile& x, const BatchTile& y) { return cost(x) > cost(y); });
        tiles.insert(tiles.end(), t.begin(), t.end());
        return (int)t.size();
    };
    const int nsub = (int)ctx->subs.size();
    if (ctx->overlap) {
        const GridInfo& G = ctx->G;
        std::vector<int> si, sb;
        for (int j = 0; j < nsub; j++) {
            const SubDesc& sd = ctx->subs[j];
            const bool inside = sd.gx0 >= G.i0 && sd.gx0 + sd.m <= G.i1 && sd.gy0 >= G.j0 && sd.gy0 + sd.nb <= G.j1;
            (inside ? si : sb).push_back(j);
        }
        ctx->bt_nint = make_tiles(si);
        make_tiles(sb);
    } else {
        std::vector<int> all(nsub);
        for (int j = 0; j < nsub; j++) all[j] = j;
        ctx->bt_nint = make_tiles(all);
    }
    ctx->bt_ntiles = (int)tiles.size();
    if ((rc = dalloc(ctx, &ctx->d_tiles, tiles.size())) || (rc = dalloc(ctx, &ctx->d_members, members.size())))
        return rc;
    CK(cudaMemcpyAsync(ctx->d_tiles, tiles.data(), sizeof(BatchTile) * tiles.size(), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_members, members.data(), sizeof(int) * members.size(), cudaMemcpyHostToDevice,
                       ctx->stream));
    auto trim = [](int n, int s) {
        s = std::max(1, std::min(s, n));
        const int per = (n + s - 1) / s;
        return (n + per - 1) / per;
    };
    // grids in tiles processed at once (a split tile occupies two CTA slots), then in CTAs
    const int nbnd = ctx->bt_ntiles - ctx->bt_nint, cpt = ctx->bt_split ? 2 : 1, tslots = std::max(1, slots / cpt);
    if (ctx->overlap && ctx->bt_nint > 0 && nbnd > 0) {
        int sb = (int)std::lround((double)tslots * nbnd / ctx->bt_ntiles);
        sb = std::max(1, std::min(tslots - 1, sb));
        ctx->bt_grid_int = cpt * trim(ctx->bt_nint, tslots - sb);
        ctx->bt_grid_bnd = cpt * trim(nbnd, sb);
    } else {
        ctx->bt_grid_int = cpt * trim(ctx->bt_ntiles, tslots);
        ctx->bt_grid_bnd = 0;
    }
    ctx->bt_grid = ctx->bt_grid_int;
    long long per = 0;
    for (int c = 0; c < ncls; c++) {
        const SubDesc& d = ctx->subs[bc[c].rep];
        per = std::max(per, (long long)(d.hi - d.lo + 1) * BATCH_NT * bc[c].mp);
    }
    ctx->bt_scr_per_cta = per;
    if ((rc = dalloc(ctx, &ctx->d_bscr, (size_t)per * (ctx->bt_grid_int + ctx->bt_grid_bnd)))) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    return HELM_OK;
}

static int factor_impl(helm_ctx* ctx)
{
    NvtxRange nv_("helm.factor");
    if (!ctx) return HELM_EINVAL;
    if (ctx->factored) return HELM_OK;
    int rc;
    // D28: factor one representative per class of bitwise-equal local operators; members alias its factors
    if (ctx->cls_rep.empty() && (rc = build_classes(ctx))) return rc;
    const int ncls = (int)ctx->cls_rep.size();
    std::vector<SubDesc> reps(ncls);
    long long fac = 0;
    for (int c = 0; c < ncls; c++) {
        reps[c] = ctx->subs[ctx->cls_rep[c]];
        reps[c].fac_off = fac;
        fac += (long long)reps[c].nb * reps[c].m * reps[c].m;
    }
    for (size_t j = 0; j < ctx->subs.size(); j++) ctx->subs[j].fac_off = reps[ctx->cls_of[j]].fac_off;
    ctx->n_dinv = fac;
    SubDesc* d_reps = nullptr;
    if ((rc = dalloc(ctx, &d_reps, ncls))) return rc;
    if (!ctx->d_dinv && (rc = dalloc(ctx, &ctx->d_dinv, ctx->n_dinv))) {
        cudaFree(d_reps);
        return rc;
    }
    CK(cudaMemcpyAsync(d_reps, reps.data(), sizeof(SubDesc) * ncls, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_desc, ctx->subs.data(), sizeof(SubDesc) * ctx->subs.size(), cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemsetAsync(ctx->d_err, 0, 4 * sizeof(int), ctx->stream));
    launch_factor(d_reps, reps.data(), ncls, ctx->m_max, ctx->d_stc, ctx->d_dinv, ctx->d_err, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    cudaFree(d_reps);
    if (ctx->sp_G > 1) {
        // cluster-split apply: relay every inverse block slab-major (one contiguous panel per CTA of a chain) --
        // once per class (members alias the representative's blocks)
        std::vector<int2> blocks;
        for (int c = 0; c < ncls; c++) {
            const int j = ctx->cls_rep[c];
            for (int i = 0; i < ctx->subs[j].nb; i++) blocks.push_back(make_int2(j, i));
        }
        int2* d_blocks = nullptr;
        z2* d_tmp = nullptr;
        const int grid = 148;
        const long long per = (long long)ctx->m_max * ctx->m_max;
        auto relay = [&]() -> int {
            int rc2;
            if ((rc2 = dalloc(ctx, &d_blocks, blocks.size())) || (rc2 = dalloc(ctx, &d_tmp, (size_t)grid * per))) return rc2;
            CK(cudaMemcpyAsync(d_blocks, blocks.data(), sizeof(int2) * blocks.size(), cudaMemcpyHostToDevice,
                               ctx->stream));
            launch_relayout(ctx->d_desc, d_blocks, (int)blocks.size(), ctx->d_dinv, d_tmp, per, grid, ctx->sp_G,
                            ctx->stream);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(ctx->stream));
            return HELM_OK;
        };
        rc = relay();
        cudaFree(d_blocks);
        cudaFree(d_tmp);
        if (rc) return rc;
    }
    int herr[4];
    CK(cudaMemcpyAsync(herr, ctx->d_err, sizeof(herr), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (herr[0])
        return set_err(ctx, HELM_EZEROPIVOT, "zero pivot (|pivot| < 1e-12 or not finite): subdomain %d, block %d, row %d",
                       herr[1] >= 0 && herr[1] < ncls ? ctx->cls_rep[herr[1]] : herr[1], herr[2], herr[3]);
    if (ctx->batched && !ctx->d_dinvB && (rc = setup_batch(ctx))) return rc;
    if ((rc = ensure_krylov(ctx, 0))) return rc;   // the solvers' work buffers belong to setup, not to a solve
    ctx->factored = true;
    return HELM_OK;
}

int helm_factor(helm_ctx* ctx)
{
    const int rc = factor_impl(ctx);
    if (rc < 0 && ctx && ctx->loop) ctx->loop->abort();   // (peers would wait for this rank in their next collective)
    return rc;
}

int helm_matvec(helm_ctx* ctx, const helm_z* x_dev, helm_z* y_dev)
{
    if (!ctx || !x_dev || !y_dev || (const void*)x_dev == (void*)y_dev)
        return set_err(ctx, HELM_EINVAL, "helm_matvec: bad arguments");
    int rc = spmv_impl(ctx, (const z2*)x_dev, (z2*)y_dev);
    if (rc) return coll(ctx, rc);
    CK(cudaGetLastError());
    return HELM_OK;
}

int helm_matvec_ext(helm_ctx* ctx, const helm_z* ext1_dev, helm_z* y_dev)
{
    if (!ctx || !ext1_dev || !y_dev) return set_err(ctx, HELM_EINVAL, "helm_matvec_ext: bad arguments");
    const GridInfo& G = ctx->G;
    const int li = G.nbr[0] >= 0, ri = G.nbr[1] >= 0, dj = G.nbr[2] >= 0;
    const StencilGeom sg = ctx->geom_for(G.i0 - li, G.j0 - dj, (long long)(G.i1 - G.i0 + li + ri));
    launch_spmv(ctx->d_A7, (const z2*)ext1_dev, (z2*)y_dev, sg, ctx->stream);
    ctx->launches++;
    CK(cudaGetLastError());
    return HELM_OK;
}

int helm_precond_apply(helm_ctx* ctx, const helm_z* r_dev, helm_z* z_dev)
{
    if (!ctx || !r_dev || !z_dev || (const void*)r_dev == (void*)z_dev)
        return set_err(ctx, HELM_EINVAL, "helm_precond_apply: bad arguments");
    return coll(ctx, apply_impl(ctx, (const z2*)r_dev, (z2*)z_dev));
}

int helm_precond_apply_ext(helm_ctx* ctx, const helm_z* ext_dev, helm_z* z_dev)
{
    if (!ctx || !ext_dev || !z_dev) return set_err(ctx, HELM_EINVAL, "helm_precond_apply_ext: bad arguments");
    const GridInfo& G = ctx->G;
    return apply_raw(ctx, (const z2*)ext_dev, G.e_i0, G.e_j0, G.e_i1 - G.e_i0, (z2*)z_dev);
}

int helm_precond_apply_host(helm_ctx* ctx, const helm_z* r_host, helm_z* z_host)
{
    if (!ctx || !r_host || !z_host) return set_err(ctx, HELM_EINVAL, "helm_precond_apply_host: bad arguments");
    int rc;
    if ((rc = ensure_krylov(ctx, 0))) return coll(ctx, rc);
    const size_t bytes = sizeof(z2) * ctx->n_local;
    CK(cudaMemcpyAsync(ctx->d_t, r_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    if ((rc = apply_impl(ctx, ctx->d_t, ctx->d_z))) return coll(ctx, rc);
    CK(cudaMemcpyAsync(z_host, ctx->d_z, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return HELM_OK;
}

int helm_gmres(helm_ctx* ctx, const helm_z* b_dev, helm_z* x_dev, int restart, double rtol, int maxit,
               helm_gmres_info* info)
{
    if (!ctx || !b_dev || !x_dev || (const void*)b_dev == (void*)x_dev)
        return set_err(ctx, HELM_EINVAL, "helm_gmres: bad arguments");
    return coll(ctx, gmres_impl(ctx, (const z2*)b_dev, (z2*)x_dev, restart, rtol, maxit, info));
}

int helm_gmres_host(helm_ctx* ctx, const helm_z* b_host, helm_z* x_host, int restart, double rtol, int maxit,
                    helm_gmres_info* info)
{
    if (!ctx || !b_host || !x_host) return set_err(ctx, HELM_EINVAL, "helm_gmres_host: bad arguments");
    int rc;
    if (!ctx->d_bb && ((rc = dalloc(ctx, &ctx->d_bb, ctx->n_local)) || (rc = dalloc(ctx, &ctx->d_xb, ctx->n_local))))
        return coll(ctx, rc);
    const size_t bytes = sizeof(z2) * ctx->n_local;
    CK(cudaMemcpyAsync(ctx->d_bb, b_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_xb, x_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
    rc = gmres_impl(ctx, ctx->d_bb, ctx->d_xb, restart, rtol, maxit, info);
    if (rc < 0) return coll(ctx, rc);
    CK(cudaMemcpyAsync(x_host, ctx->d_xb, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return rc;
}

int helm_export_stencil(helm_ctx* ctx, helm_z* out_dev)
{
    if (!ctx || !out_dev) return set_err(ctx, HELM_EINVAL, "helm_export_stencil: bad arguments");
    CK(cudaMemcpyAsync(out_dev, ctx->d_A7, sizeof(z2) * ctx->G.ns * ctx->n_local, cudaMemcpyDeviceToDevice,
                       ctx->stream));
    return HELM_OK;
}

int helm_profile_enable(helm_ctx* ctx, int on)
{
    if (!ctx) return HELM_EINVAL;
    ctx->prof = on != 0;
    return HELM_OK;
}

int helm_profile_read(helm_ctx* ctx, double* apply_ms, int* apply_launches, int* total_launches)
{
    if (!ctx) return HELM_EINVAL;
    CK(cudaStreamSynchronize(ctx->stream));
    double ms = 0.0;
    for (auto& pr : ctx->ev_used) {
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, pr.first, pr.second));
        ms += f;
        ctx->ev_free.push_back(pr.first);
        ctx->ev_free.push_back(pr.second);
    }
    if (apply_ms) *apply_ms = ms;
    if (apply_launches) *apply_launches = (int)ctx->ev_used.size();
    if (total_launches) *total_launches = ctx->launches;
    ctx->ev_used.clear();
    ctx->launches = 0;
    return HELM_OK;
}

int helm_setup(const helm_params* params, int rank, int nranks, const void* nccl_unique_id, void* cuda_stream,
               helm_ctx** out)
{
    return setup_impl(params, rank, nranks, nccl_unique_id, -1, cuda_stream, out);
}

int helm_setup_loopback(const helm_params* params, int rank, int nranks, int group, void* cuda_stream, helm_ctx** out)
{
    if (group < 0 || nranks < 2 || nranks > 16) return HELM_EINVAL;
    const int rc = setup_impl(params, rank, nranks, nullptr, group, cuda_stream, out);
    if (rc < 0) {   // the peers must not wait for this rank in their first collective: abort the group
        std::lock_guard<std::mutex> lk(g_loop_mu);
        LoopGroup*& L = g_loops[group];
        if (!L) {
            L = new LoopGroup();
            L->nranks = nranks;
            L->ctx.assign(nranks, nullptr);
            L->slot.assign(nranks, nullptr);
        }
        L->abort();
    }
    return rc;
}

const char* helm_last_error(const helm_ctx* ctx) { return ctx ? ctx->err : "null context"; }

void helm_destroy(helm_ctx* ctx)
{
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    else cudaDeviceSynchronize();
#ifdef HELM_HAVE_NCCL
    if (ctx->comm) ncclCommDestroy(ctx->comm);
#endif
    if (ctx->loop) {
        std::lock_guard<std::mutex> lk(g_loop_mu);
        ctx->loop->ctx[ctx->rank] = nullptr;
        if (--ctx->loop->members == 0) {
            delete ctx->loop;
            g_loops.erase(ctx->loop_id);
        }
        ctx->loop = nullptr;
    }
    if (ctx->d_loop_tmp) cudaFree(ctx->d_loop_tmp);
    for (void* b : {(void*)ctx->d_dinvB, (void*)ctx->d_tiles, (void*)ctx->d_bcls, (void*)ctx->d_members,
                    (void*)ctx->d_bscr})
        if (b) cudaFree(b);
    void* bufs[] = {ctx->d_desc, ctx->d_order, ctx->d_A7, ctx->d_stc, ctx->d_dinv, ctx->d_scratch, ctx->d_err,
                    ctx->d_V, ctx->d_w, ctx->d_z, ctx->d_t, ctx->d_r, ctx->d_xb, ctx->d_bb, ctx->d_h1, ctx->d_h2,
                    ctx->d_Hcol, ctx->d_y, ctx->d_norm, ctx->d_zpart, ctx->d_dpart, ctx->d_ext, ctx->d_sq,
                    ctx->d_pou, ctx->d_candx, ctx->d_candy, ctx->d_cext, ctx->d_H, ctx->d_dots, ctx->d_ca,
                    ctx->d_ce, ctx->d_hout, ctx->d_sc, ctx->d_Z};
    for (void* b : bufs)
        if (b) cudaFree(b);
    for (int q = 0; q < 4; q++) {
        if (ctx->d_sendbuf[q]) cudaFree(ctx->d_sendbuf[q]);
        if (ctx->d_recvbuf[q]) cudaFree(ctx->d_recvbuf[q]);
        for (auto* bm : {&ctx->band_send[q], &ctx->band_recv[q]}) {
            if (bm->d_rects) cudaFree(bm->d_rects);
            if (bm->d_off) cudaFree(bm->d_off);
        }
    }
    if (ctx->d_bandx) cudaFree(ctx->d_bandx);
    if (ctx->d_bandy) cudaFree(ctx->d_bandy);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    if (ctx->phases)
        fprintf(stderr, "HELM_GMRES_PHASES ms: apply %.1f spmv %.1f multidot2 %.1f reduce+coef %.1f update %.1f "
                        "norm+record %.1f gap(host) %.1f\n", ctx->ph_ms[0], ctx->ph_ms[1], ctx->ph_ms[2], ctx->ph_ms[3],
                ctx->ph_ms[4], ctx->ph_ms[5], ctx->ph_ms[7]);
    for (auto e : ctx->ev_ph)
        if (e) cudaEventDestroy(e);
    if (ctx->h_hc) cudaFreeHost(ctx->h_hc);
    if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
    for (auto e : ctx->ev_ov)
        if (e) cudaEventDestroy(e);
    if (ctx->d_order_ov) cudaFree(ctx->d_order_ov);
    for (auto e : ctx->ev_hc)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->ev_free) cudaEventDestroy(e);
    for (auto& pr : ctx->ev_used) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    delete ctx;
}

}  // extern "C"
