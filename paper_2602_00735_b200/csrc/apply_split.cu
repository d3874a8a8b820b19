// apply_split.cu -- K4s: the fused RAS-PML apply for FEW, LARGE subdomains (the paper's own regime,
// 4-64 subdomains of ~320-360 nodes per block row).
//
// k_apply streams every subdomain through one CTA, so a problem with fewer subdomains than SMs leaves most of HBM
// idle.  Here one thread-block cluster of 2G CTAs owns one subdomain:
//   group 0 (CTAs 0..G-1)   the bottom chain  B: y_i = P_i^-1 (b_i - L_i y_{i-1}), i = 0..tw-1,  then the twist,
//                           then the down sweep D: x_i = y_i - P_i^-1 U_i x_{i+1}, i = tw-1..lo
//   group 1 (CTAs G..2G-1)  the top chain     T: z_i = Q_i^-1 (b_i - U_i z_{i+1}), i = nb-1..tw+1, the twist,
//                           then the up sweep U: x_i = z_i - Q_i^-1 L_i x_{i-1}, i = tw+1..hi
// CTA g of a group owns the row slab [r0, r1) of every block it visits and streams exactly that slab: after the
// factorisation the inverse blocks are relaid "slab-major" (slab g of a block is one contiguous, column-major
// R x m panel), so each CTA's share is one bulk-copy stream (cp.async.bulk into an mbarrier ring, as in k_apply).
// Every step, each CTA computes its R entries of the new carried vector and pushes them into the vector buffer of
// every CTA of its group through distributed shared memory with st.async, each store completing 16 bytes of
// transaction count on the receiver's exchange mbarrier (which expects m x 16 bytes per step): no fences, no
// polling of remote state; the next step waits on its own barrier.  At the twist the two groups swap
// y_{tw-1} / z_{tw+1} the same way; both groups form x_tw (group 0 alone writes it).  The producer also
// bulk-copies each step's input row b_i and coupling vectors into a double-buffered "aux" slot one step ahead, so
// the per-step right-hand side is formed from shared memory only.  Per row the arithmetic is k_apply's up to the
// split of the GEMV into two partial sums.
#include <stdlib.h>

#include <mutex>

#include "internal.cuh"

namespace {

constexpr int NSMAX = 16;           // ring slots (runtime count nss <= NSMAX: sized from the smem left per CTA)
// target bytes per ring slot; swept on the paper workloads (apply ms t300 / t600 / t1200): 16384 -> 2.26 / 3.76 / 13.87,
// 32000 -> 1.58 / 3.27 / 13.85, 48000 -> 1.47 / 3.24 / 11.92, 80000 -> 1.29 / 3.22 / 12.13 (scripts/split_ring_sweep.sh;
// HELM_SPLIT_SLOTB / HELM_SPLIT_SLOTS override)
constexpr int SLOT_T = 48000;
constexpr int NAUX = 2;             // aux slots: [b, cd, clo, chi] x mcap each; the twist step takes two

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok = 0;
    const uint32_t a = s_u32(bar);
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s_u32(dst)),
                 "l"(src), "r"(bytes), "r"(s_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, int rank)   // this CTA's smem address -> peer's
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(s_u32(p)), "r"(rank));
    return r;
}
// 16-byte store into a peer CTA's shared memory that completes 16 bytes of transaction count on its mbarrier
__device__ __forceinline__ void st_async(uint32_t addr, z2 v, uint32_t bar_addr)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(v.x), "d"(v.y), "r"(bar_addr)
                 : "memory");
}
__device__ __forceinline__ void cluster_barrier()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cta_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}
__device__ __forceinline__ void cbar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

enum { PH_T = 0, PH_B = 1, PH_Z = 2, PH_D = 3, PH_U = 4 };
struct Step { int ph, i; };

// the step sequence of a group: group 0 B..., Z, D...; group 1 T..., Z, U...
__device__ __forceinline__ int pre_steps(const SubDesc& d, int grp) { return grp == 0 ? d.tw : d.nb - 1 - d.tw; }
__device__ __forceinline__ int group_steps(const SubDesc& d, int grp)
{
    return pre_steps(d, grp) + 1 + (grp == 0 ? d.tw - d.lo : d.hi - d.tw);
}
__device__ __forceinline__ Step gstep(const SubDesc& d, int grp, int s)
{
    const int n1 = pre_steps(d, grp);
    if (s < n1) return grp == 0 ? Step{PH_B, s} : Step{PH_T, d.nb - 1 - s};
    if (s == n1) return Step{PH_Z, d.tw};
    s -= n1 + 1;
    return grp == 0 ? Step{PH_D, d.tw - 1 - s} : Step{PH_U, d.tw + 1 + s};
}

// r (+/-)= C v with C the coupling row of node q (d, lo -> v[q-1], hi -> v[q+1]); same order as k_apply
__device__ __forceinline__ void cpl(z2& r, z2 cd, z2 clo, z2 chi, const z2* v, int q, int m, bool minus)
{
    const double s = minus ? -1.0 : 1.0;
    zfma(r, zmk(s * cd.x, s * cd.y), v[q]);
    if (q > 0) zfma(r, zmk(s * clo.x, s * clo.y), v[q - 1]);
    if (q + 1 < m) zfma(r, zmk(s * chi.x, s * chi.y), v[q + 1]);
}

// aux vectors a step needs: bit 0 b_i, bit 1 L_i set, bit 2 U_i set
__device__ __forceinline__ int aux_need(const SubDesc& d, Step st)
{
    switch (st.ph) {
    case PH_T: return 1 | (st.i < d.nb - 1 ? 4 : 0);
    case PH_B: return 1 | (st.i > 0 ? 2 : 0);
    case PH_Z: return 1 | (st.i > 0 ? 2 : 0) | (st.i < d.nb - 1 ? 4 : 0);
    case PH_D: return 4;
    default: return 2;
    }
}

__device__ __forceinline__ void split_body(const ApplyArgs& a, int G, int ncw, int slot_bytes, int mcap, int NSS)
{
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    z2* aux = reinterpret_cast<z2*>(smem + (size_t)NSS * slot_bytes);   // [NAUX][4][mcap]
    uint64_t* full = reinterpret_cast<uint64_t*>(aux + (size_t)NAUX * 4 * mcap);
    uint64_t* empty = full + NSS;
    uint64_t* afull = empty + NSS;       // [NAUX]
    uint64_t* aempty = afull + NAUX;     // [NAUX]
    uint64_t* ex = aempty + NAUX;        // [2] group exchange (G arrivals per phase)
    uint64_t* twb = ex + 2;              // twist exchange (G arrivals, once)
    z2* V = reinterpret_cast<z2*>(twb + 2);   // [2][mcap] carried vector, double-buffered by step parity
    z2* W = V + 2 * mcap;                // [mcap] the other chain's vector at the twist
    z2* rhs = W + mcap;                  // [mcap]
    z2* red = rhs + mcap;                // [4][R] partial sums of the column residues (P > 1)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = cta_rank(), grp = crank / G, gr = crank - grp * G;
    const int sub = a.order[blockIdx.x / (2 * G)];
    const SubDesc d = a.desc[sub];
    const int m = d.m;
    const int r0 = (int)(((long long)m * gr) / G), r1 = (int)(((long long)m * (gr + 1)) / G), R = r1 - r0;
    const int kc = max(4, slot_bytes / (R * (int)sizeof(z2)) / 4 * 4);   // whole groups of 4 columns
    const int S = group_steps(d, grp);
    const int n1 = pre_steps(d, grp);

    if (tid == 0) {
        for (int q = 0; q < NSS; q++) {
            mb_init(&full[q], 1);
            mb_init(&empty[q], ncw);
        }
        for (int q = 0; q < NAUX; q++) {
            mb_init(&afull[q], 1);
            mb_init(&aempty[q], 1);
        }
        // exchange barriers: one local arrive per phase (with the expected m x 16 bytes), the bytes from st.async
        mb_init(&ex[0], 1);
        mb_init(&ex[1], 1);
        mb_init(&twb[0], 1);
        mb_expect_tx(&ex[0], (uint32_t)(m * sizeof(z2)));       // step 0's all-gather
        // the twist vector of the other chain (nothing if that chain has no steps before the twist)
        mb_expect_tx(&twb[0], pre_steps(d, 1 - grp) > 0 ? (uint32_t)(m * sizeof(z2)) : 0u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_barrier();   // every barrier of the cluster initialised before any remote transaction

    if (warp == ncw) {
        // ---------------------------------------------------------------- producer
        if (lane == 0) {
            const uint32_t vb = (uint32_t)(m * sizeof(z2));
            uint32_t ka = 0;   // aux slot uses
            auto issue_aux = [&](int s) {
                const Step st = gstep(d, grp, s);
                const int need = aux_need(d, st);
                const z2* srow = a.stencil + d.stc_off + (long long)st.i * a.ns * m;
                // the twist needs both coupling sets: two slots (L in the first, U in the second)
                const int parts = st.ph == PH_Z ? 2 : 1;
                for (int part = 0; part < parts; part++, ka++) {
                    const uint32_t slot = ka % NAUX, ph = (ka / NAUX) & 1;
                    mb_wait(&aempty[slot], ph ^ 1);
                    const bool want_b = (need & 1) && part == 0;
                    const bool low = st.ph == PH_Z ? part == 0 && (need & 2) : (need & 2) != 0;
                    const bool up = st.ph == PH_Z ? part == 1 && (need & 4) : (need & 4) != 0;
                    const int nv = (want_b ? 1 : 0) + ((low || up) ? (a.ns == 9 ? 3 : 2) : 0);
                    mb_expect_tx(&afull[slot], nv * vb);
                    z2* dst = aux + (size_t)slot * 4 * mcap;
                    if (want_b) {
                        const long long gi = d.gx0 - a.in_i0, gj = d.gy0 + st.i - a.in_j0;
                        bulk_load(dst, a.in + gi + a.in_stride * gj, vb, &afull[slot]);
                    }
                    if (low || up) {
                        const int sd = low ? SL_S : SL_N, slo = low ? SL_SW : SL_NW, shi = low ? SL_SE : SL_NE;
                        bulk_load(dst + mcap, srow + (long long)sd * m, vb, &afull[slot]);
                        if (a.ns == 9 || !low) bulk_load(dst + 3 * mcap, srow + (long long)shi * m, vb, &afull[slot]);
                        if (a.ns == 9 || low) bulk_load(dst + 2 * mcap, srow + (long long)slo * m, vb, &afull[slot]);
                    }
                }
            };
            uint32_t k = 0;
            issue_aux(0);
            for (int s = 0; s < S; s++) {
                if (s + 1 < S) issue_aux(s + 1);
                const Step st = gstep(d, grp, s);
                const z2* slab = a.dinv + d.fac_off + (long long)st.i * m * m + (long long)r0 * m;
                for (int c0 = 0; c0 < m; c0 += kc, k++) {
                    const int nc = min(kc, m - c0);
                    const uint32_t slot = k % NSS, ph = (k / NSS) & 1;
                    mb_wait(&empty[slot], ph ^ 1);
                    const uint32_t bytes = (uint32_t)(nc * R * sizeof(z2));
                    mb_expect_tx(&full[slot], bytes);
                    bulk_load(ring + (size_t)slot * slot_bytes, slab + (long long)c0 * R, bytes, &full[slot]);
                }
            }
        }
    } else {
        // ---------------------------------------------------------------- consumers
        const int nct = ncw * 32;
        // GEMV mapping: thread -> (row tr of the slab, column phase cp).  Canonical order shared with k_apply: four
        // partial sums over the columns c = 0..3 (mod 4), each in increasing c, combined as (s0+s1)+(s2+s3); the
        // P in {1, 2, 4} phases each own the residues q with q mod P = cp, so the result does not depend on P or G
        const int P = nct / R >= 4 ? 4 : (nct / R >= 2 ? 2 : 1);
        const int tr = tid % R, cp = tid / R;
        const bool act = cp < P;
        const bool own = cp == 0;
        const int t = tid;
        z2* scr = a.scratch + (long long)blockIdx.x * a.scratch_per_cta;
        const int og = 1 - grp;
        const bool p1 = a.ns != 9;
        uint32_t k = 0, ka = 0;
        for (int s = 0; s < S; s++) {
            const Step st = gstep(d, grp, s);
            const z2* Vc = V + (s & 1) * mcap;
            if (st.ph == PH_Z) mb_wait(&twb[0], 0);
            const int need = aux_need(d, st);
            // ---- right-hand side of this step, all m rows (redundant across the group), from the aux slot(s)
            const uint32_t sa = ka % NAUX;
            mb_wait(&afull[sa], (ka / NAUX) & 1);
            const z2* X = aux + (size_t)sa * 4 * mcap;
            const z2* X2 = X;
            if (st.ph == PH_Z) {
                const uint32_t sb = (ka + 1) % NAUX;
                mb_wait(&afull[sb], ((ka + 1) / NAUX) & 1);
                X2 = aux + (size_t)sb * 4 * mcap;
            }
            for (int q = t; q < m; q += nct) {
                z2 r = (need & 1) ? X[q] : zmk(0, 0);
                const z2 zero = zmk(0, 0);
                switch (st.ph) {
                case PH_T:
                    if (need & 4) cpl(r, X[mcap + q], p1 ? zero : X[2 * mcap + q], X[3 * mcap + q], Vc, q, m, true);
                    break;
                case PH_B:
                    if (need & 2) cpl(r, X[mcap + q], X[2 * mcap + q], p1 ? zero : X[3 * mcap + q], Vc, q, m, true);
                    break;
                case PH_Z: {
                    const z2* yv = grp == 0 ? Vc : W;   // y_{tw-1}
                    const z2* zv = grp == 0 ? W : Vc;   // z_{tw+1}
                    if (need & 2) cpl(r, X[mcap + q], X[2 * mcap + q], p1 ? zero : X[3 * mcap + q], yv, q, m, true);
                    if (need & 4) cpl(r, X2[mcap + q], p1 ? zero : X2[2 * mcap + q], X2[3 * mcap + q], zv, q, m, true);
                    break;
                }
                case PH_D:
                    cpl(r, X[mcap + q], p1 ? zero : X[2 * mcap + q], X[3 * mcap + q], Vc, q, m, false);
                    break;
                default:
                    cpl(r, X[mcap + q], X[2 * mcap + q], p1 ? zero : X[3 * mcap + q], Vc, q, m, false);
                    break;
                }
                rhs[q] = r;
            }
            cbar(nct);
            if (t == 0) {
                mb_arrive(&aempty[sa]);
                if (st.ph == PH_Z) mb_arrive(&aempty[(ka + 1) % NAUX]);
                // post the next step's all-gather (its barrier's previous phase, step s - 1, has completed)
                if (s + 1 < S) mb_expect_tx(&ex[(s + 1) & 1], (uint32_t)(m * sizeof(z2)));
            }
            ka += st.ph == PH_Z ? 2 : 1;
            // ---- slab GEMV: acc = Dinv_i[r0 + tr, :] rhs
            z2 sp[4] = {zmk(0, 0), zmk(0, 0), zmk(0, 0), zmk(0, 0)};
            for (int c0 = 0; c0 < m; c0 += kc, k++) {
                const int nc = min(kc, m - c0);
                const uint32_t slot = k % NSS, ph = (k / NSS) & 1;
                mb_wait(&full[slot], ph);
                const z2* col = reinterpret_cast<const z2*>(ring + (size_t)slot * slot_bytes);
                if (act) {
                    // P = 4: sp[0] = residue cp.  P = 2: sp[0], sp[1] = residues cp, cp + 2.  P = 1: sp[q] = residue q.
                    if (P == 4) {
#pragma unroll 4
                        for (int c = cp; c < nc; c += 4) zfma(sp[0], col[(size_t)c * R + tr], rhs[c0 + c]);
                    } else if (P == 2) {
                        int c = cp;
#pragma unroll 2
                        for (; c + 2 < nc; c += 4) {
                            zfma(sp[0], col[(size_t)c * R + tr], rhs[c0 + c]);
                            zfma(sp[1], col[(size_t)(c + 2) * R + tr], rhs[c0 + c + 2]);
                        }
                        if (c < nc) zfma(sp[0], col[(size_t)c * R + tr], rhs[c0 + c]);
                    } else {
                        int c = 0;
#pragma unroll 2
                        for (; c + 3 < nc; c += 4) {
                            zfma(sp[0], col[(size_t)c * R + tr], rhs[c0 + c]);
                            zfma(sp[1], col[(size_t)(c + 1) * R + tr], rhs[c0 + c + 1]);
                            zfma(sp[2], col[(size_t)(c + 2) * R + tr], rhs[c0 + c + 2]);
                            zfma(sp[3], col[(size_t)(c + 3) * R + tr], rhs[c0 + c + 3]);
                        }
                        if (c < nc) zfma(sp[0], col[(size_t)c * R + tr], rhs[c0 + c]);
                        if (c + 1 < nc) zfma(sp[1], col[(size_t)(c + 1) * R + tr], rhs[c0 + c + 1]);
                        if (c + 2 < nc) zfma(sp[2], col[(size_t)(c + 2) * R + tr], rhs[c0 + c + 2]);
                    }
                }
                __syncwarp();
                if (lane == 0) mb_arrive(&empty[slot]);
            }
            // ---- reduce the column phases, finish own rows, scratch, owner write; all-gather into the group
            const bool to_twist = s == n1 - 1;
            if (P > 1) {
                if (act) {
                    red[cp * R + tr] = sp[0];
                    if (P == 2) red[(cp + 2) * R + tr] = sp[1];
                }
                cbar(nct);
            }
            if (own) {
                const int row = r0 + tr;
                z2 acc;
                if (P > 1)
                    acc = zadd(zadd(red[tr], red[R + tr]), zadd(red[2 * R + tr], red[3 * R + tr]));
                else
                    acc = zadd(zadd(sp[0], sp[1]), zadd(sp[2], sp[3]));
                z2 x = acc;
                if (st.ph == PH_T || st.ph == PH_B) {
                    if (st.i >= d.lo && st.i <= d.hi) scr[(long long)(st.i - d.lo) * R + tr] = acc;
                } else {
                    if (st.ph != PH_Z) x = zsub(scr[(long long)(st.i - d.lo) * R + tr], acc);
                    const bool writer = st.ph != PH_Z || grp == 0;
                    if (writer && st.i >= d.lo && st.i <= d.hi && row >= d.olo && row <= d.ohi) {
                        if (a.pou_buf) {
                            const double w = chi_ramp(d.gx0 + row, d.s0x, d.s1x, a.delta, d.flags & 1, d.flags & 2) *
                                             chi_ramp(d.gy0 + st.i, d.s0y, d.s1y, a.delta, d.flags & 4, d.flags & 8);
                            a.pou_buf[d.pou_off + (row - d.olo) + (long long)(d.ohi - d.olo + 1) * (st.i - d.lo)] =
                                zscale(x, w);
                        } else {
                            const long long gi = d.gx0 + row - a.out_i0, gj = d.gy0 + st.i - a.out_j0;
                            a.out[gi + a.out_stride * gj] = x;
                        }
                    }
                }
                z2* Vn = V + ((s + 1) & 1) * mcap;
                for (int q = 0; q < G; q++)
                    st_async(map_rank(Vn + row, grp * G + q), x, map_rank(&ex[s & 1], grp * G + q));
                if (to_twist)
                    for (int q = 0; q < G; q++) st_async(map_rank(W + row, og * G + q), x, map_rank(&twb[0], og * G + q));
            }
            mb_wait(&ex[s & 1], (s >> 1) & 1);
        }
    }
    __syncwarp();
    cluster_barrier();   // no CTA leaves while a peer may still address its shared memory
}

// two register budgets: <= 288 threads with two CTAs per SM (113 registers), <= 512 threads with one
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_apply_split(ApplyArgs a, int G, int ncw, int slot_bytes, int mcap, int nss)
{
    split_body(a, G, ncw, slot_bytes, mcap, nss);
}

const void* split_fn(int block) { return block <= 288 ? (const void*)k_apply_split<288, 2> : (const void*)k_apply_split<512, 1>; }

// the dynamic-smem limit is a per-function attribute shared by every context in the process: only ever raise it
void ensure_split_smem(int block, int smem) { raise_smem_attr(split_fn(block), smem, true); }

// slab-major relayout of every inverse block (column-major m x m -> G contiguous column-major R_g x m panels)
__global__ void k_relayout(const SubDesc* __restrict__ desc, const int2* __restrict__ blocks, int nblocks, z2* dinv,
                           z2* tmp, long long tmp_per_cta, int G)
{
    z2* buf = tmp + (long long)blockIdx.x * tmp_per_cta;
    for (int b = blockIdx.x; b < nblocks; b += gridDim.x) {
        const int2 bi = blocks[b];
        const SubDesc d = desc[bi.x];
        const int m = d.m;
        z2* A = dinv + d.fac_off + (long long)bi.y * m * m;
        for (long long e = threadIdx.x; e < (long long)m * m; e += blockDim.x) buf[e] = A[e];
        __syncthreads();
        for (int g = 0; g < G; g++) {
            const int r0 = (int)(((long long)m * g) / G), r1 = (int)(((long long)m * (g + 1)) / G), R = r1 - r0;
            z2* P = A + (long long)r0 * m;
            for (long long e = threadIdx.x; e < (long long)R * m; e += blockDim.x) {
                const int c = (int)(e / R), r = (int)(e - (long long)c * R);
                P[e] = buf[(long long)c * m + r0 + r];
            }
        }
        __syncthreads();
    }
}

}  // namespace

int split_slot_bytes(int m_max, int G)
{
    const int R = (m_max + G - 1) / G;
    static const int target = [] { const char* e = getenv("HELM_SPLIT_SLOTB"); return e ? atoi(e) : SLOT_T; }();
    int kc = target / (R * (int)sizeof(z2)) / 4 * 4;
    if (kc < 4) kc = 4;
    return kc * R * (int)sizeof(z2);
}

// ctas_per_sm: how many CTAs of this kernel must share an SM; the ring takes what shared memory is left
int split_configure(int m_max, int G, int ctas_per_sm, int* block_threads, int* smem_bytes, int* slot_bytes,
                    int* ncw_out, int* nslots)
{
    const int R = (m_max + G - 1) / G;
    // consumer warps: enough for 4 column phases per row when the CTA stays <= 16 warps, else 2, else 1
    int ncw = (4 * R + 31) / 32;
    if (ncw > 15) ncw = (2 * R + 31) / 32;
    if (ncw > 15) ncw = (R + 31) / 32;
    ncw = std::max(4, ncw);
    *ncw_out = ncw;
    *block_threads = 32 * (ncw + 1);
    *slot_bytes = split_slot_bytes(m_max, G);
    const int fixed = NAUX * 4 * m_max * (int)sizeof(z2) + (2 * NSMAX + 2 * NAUX + 4) * 8 + 4 * m_max * (int)sizeof(z2) +
                      std::max(32 * ncw, 4 * R) * (int)sizeof(z2);
    const int budget = 227 * 1024 / std::max(1, ctas_per_sm) - 1024 - fixed;
    static const int cap = [] { const char* e = getenv("HELM_SPLIT_SLOTS"); return e ? atoi(e) : NSMAX; }();
    const int nss = std::min(std::min(NSMAX, cap), budget / *slot_bytes);
    if (nss < 2 || *block_threads > 512) return -1;
    *nslots = nss;
    *smem_bytes = nss * *slot_bytes + fixed;
    ensure_split_smem(*block_threads, *smem_bytes);
    return 0;
}

int launch_apply_split(const ApplyArgs& a, int nsub, int G, int block, int smem, int slot_bytes, int ncw, int m_max,
                       int nslots, cudaStream_t s)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(nsub * 2 * G);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ensure_split_smem(block, smem);
    if (block <= 288) return (int)cudaLaunchKernelEx(&cfg, k_apply_split<288, 2>, a, G, ncw, slot_bytes, m_max, nslots);
    return (int)cudaLaunchKernelEx(&cfg, k_apply_split<512, 1>, a, G, ncw, slot_bytes, m_max, nslots);
}

int max_split_clusters(int G, int block, int smem)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2 * G;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(2 * G);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, split_fn(block), &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void launch_relayout(const SubDesc* desc, const int2* blocks, int nblocks, z2* dinv, z2* tmp, long long tmp_per_cta,
                     int grid, int G, cudaStream_t s)
{
    k_relayout<<<grid, 512, 0, s>>>(desc, blocks, nblocks, dinv, tmp, tmp_per_cta, G);
}
