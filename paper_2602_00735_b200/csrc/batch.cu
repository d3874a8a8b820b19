// batch.cu -- the RAS-PML preconditioner application (z = sum_j R~_j^T A_j^-1 R_j r) for subdomains that
// share their local operator, on the FP64 tensor cores.
//
// With a constant wave speed (c = 1) the local operator A_j (the shifted global problem with the
// local PML g_j on the full box) depends only on the subdomain's shape and on where the global PML reaches it: the
// thousands of interior subdomains of the BJ configs are translates of one another and their assembled stencils are
// bitwise equal (D28).  Setup groups the subdomains into classes of bitwise-equal local operators (k_stencil_eq
// proves the equality; nothing is assumed), factors one representative per class, and this kernel applies each
// class's explicit Schur-complement inverses to NT = 16 subdomains at a time: every block step of the twisted
// substitution (ring.cuh) becomes one complex GEMM
//     Y_i (m x 16) = F_i (m x m) R_i (m x 16),     R_i = b_i - L_i Y_{i-1}  (or the U / D / Z forms)
// on mma.sync.m8n8k4.f64 (DMMA; three real products per complex k-step, the 3M form), with F_i streamed by TMA bulk
// copies into a shared-memory ring (read once per 16 subdomains instead of once per subdomain), the step's coupling
// rows bulk-copied beside it, and R_i, the two chain carries and the accumulator epilogue in shared memory.  Two CTAs
// per SM; on ranks with few tiles per SM, 8-wide tiles and a cluster of two CTAs per tile (one per twisted half).
// The result of every subdomain is computed exactly as in the per-subdomain solve, up to the order of the
// floating-point additions of the GEMV (column n of a DMMA product depends on column n of R only, so a subdomain's
// result does not depend on which other subdomains share its tile, on the tile width, on the split, or on the rank).
//
// Layout of the class factors ("batch layout"): block i of class c at off_c + i * mp * S, column k (mp of them, m
// padded to a multiple of 8, zero beyond m) at k * S, rows contiguous with S = mp + 2 (== 2 mod 8 z2: the A-fragment
// loads of a quarter warp -- rows g, g+1, columns t..t+3 -- hit eight distinct 16-byte bank groups).
#include <cooperative_groups.h>
#include <stdio.h>
#include <stdlib.h>

#include "internal.cuh"
#include "ring.cuh"

using namespace ring;

namespace {

constexpr int NT = BATCH_NT;   // subdomains per tile: two 8-wide DMMA column tiles
constexpr int KC = 8;          // factor columns per ring slot (two k-steps of 4)

// FP64 tensor cores: d += a b for one 8 x 8 x 4 real tile per warp.  Fragments: a = A[g][t], b = B[t][g],
// c = (C[g][2t], C[g][2t+1]) with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Split tiles (few tiles per SM, e.g. one rank of a large decomposition): a cluster of two CTAs shares a tile -- rank 0
// runs the top chain then the upward expansion (T, then U), rank 1 the bottom chain, the twist and the downward
// expansion (B, Z, D) -- so the serial chain of a tile is half as long.  At the twist the two swap carries through
// distributed shared memory: rank 0 sends z_{tw+1}, rank 1 computes x_tw and sends it back (two cluster barriers).
// role 0: the whole solve in one CTA (ring.cuh's order); 1 / 2: the two halves.
__device__ __forceinline__ int nsteps_role(const SubDesc& d, int role)
{
    if (role == 0) return nsteps(d);
    return role == 1 ? (d.nb - 1 - d.tw) + (d.hi - d.tw) : d.tw + 1 + (d.tw - d.lo);
}
__device__ __forceinline__ Step step_role(const SubDesc& d, int role, int s)
{
    if (role == 0) return step_of(d, s);
    if (role == 1) {
        const int nT = d.nb - 1 - d.tw;
        return s < nT ? Step{PH_T, d.nb - 1 - s} : Step{PH_U, d.tw + 1 + (s - nT)};
    }
    return s < d.tw ? Step{PH_B, s} : (s == d.tw ? Step{PH_Z, d.tw} : Step{PH_D, d.tw - 1 - (s - d.tw - 1)});
}
// the carry exchanges of a split tile happen before step x1 (rank 0: both barriers; rank 1: the first) and x2 (rank 1)
__device__ __forceinline__ int xchg1(const SubDesc& d, int role) { return role == 1 ? d.nb - 1 - d.tw : d.tw; }

#ifdef HELM_BATCH_PROF
// development aid (-DHELM_BATCH_PROF): clock64 cycles per phase of every block step as thread 0 of CTA 0 sees them
// (waits included), printed at the end: right-hand sides, barrier after them, ring waits, DMMA loop, epilogue, barrier
#define BPROF(k) do { if (tid == 0 && blockIdx.x == 0) { const long long t_ = clock64(); bpr[k] += t_ - bt0; bt0 = t_; } } while (0)
#else
#define BPROF(k) do { } while (0)
#endif

__device__ __forceinline__ void batch_body(const BatchArgs& a, int ncw, int mpmax, int slot_bytes, int NSL, int split)
{
    namespace cg = cooperative_groups;
    const int role = split ? (int)cg::this_cluster().block_rank() + 1 : 0;
    const int cid = split ? blockIdx.x >> 1 : blockIdx.x, ncl = split ? gridDim.x >> 1 : gridDim.x;
#ifdef HELM_BATCH_PROF
    long long bpr[7] = {0, 0, 0, 0, 0, 0, 0}, bt0 = clock64();
#endif
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_gx[NT], s_gy[NT], s_sub[NT];
    __shared__ SubDesc s_d;      // the tile's class representative (shape, couplings, owned ranges)
    __shared__ BatchClass s_c;
    unsigned char* ringb = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSL * slot_bytes);
    uint64_t* empty = full + NSL;
    const int SR = mpmax + 4;                                // R row stride (== 4 mod 8: conflict-free B fragments)
    z2* R = reinterpret_cast<z2*>(empty + NSL + 2);          // [NT][SR]: right-hand sides of the current step
    const int SV = mpmax + 1;                                // carry row stride (odd: conflict-free epilogue stores)
    z2* vb = R + NT * SR;                                    // [NT][SV]: bottom chain / down-expansion carry
    z2* vt = vb + NT * SV;                                   // [NT][SV]: top chain / up-expansion carry
    // the coupling rows of the current block step, bulk-copied by the producer: U_i (N, NE, NW) then L_i (S, SW, SE)
    z2* cpb = vt + NT * SV;                                  // [6][mpmax]
    uint64_t* cfull = empty + NSL;                           // coupling rows landed
    uint64_t* cempty = cfull + 1;                            // every consumer warp has built its right-hand sides
    const int nct = ncw * 32;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;

    if (tid == 0) {
        for (int s = 0; s < NSL; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], ncw);
        }
        mbar_init(cfull, 1);
        mbar_init(cempty, ncw);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int e = tid; e < 6 * mpmax; e += blockDim.x) cpb[e] = zmk(0, 0);   // NW / SE stay 0 for P1
    __syncthreads();

    if (warp == ncw) {
        // ---------------------------------------------------------------- producer: stream the class factors
        // (lane 0 issues; with split tiles the whole warp stays for the cluster barriers)
        if (lane != 0 && !split) return;
        uint32_t slot = 0, ph = 0, cph = 0;
        const int ns = a.cc.ns, nv = ns == 9 ? 3 : 2;
        const int sl_u[3] = {SL_N, SL_NE, SL_NW}, sl_l[3] = {SL_S, SL_SW, SL_SE};
        for (int w = cid; w < a.ntiles; w += ncl) {
            const BatchClass C = a.cls[a.tiles[w].cls];
            const SubDesc d = a.desc[C.rep];
            const int S = nsteps_role(d, role);
            const uint32_t bytes = (uint32_t)(KC * C.S * sizeof(z2));
            const uint32_t vbytes = (uint32_t)(d.m * sizeof(z2));
            for (int s = 0; s <= S; s++) {
                if (role && s == xchg1(d, role)) {
                    cg::this_cluster().sync();
                    if (role == 1) cg::this_cluster().sync();
                }
                if (role == 2 && s == d.tw + 1) cg::this_cluster().sync();
                if (s == S) break;
                const int i = step_role(d, role, s).i;
                if (lane == 0) {
                // coupling rows of step s (once the previous step's right-hand sides are built), then its factor block
                mbar_wait(cempty, cph ^ 1);
                mbar_arrive_expect_tx(cfull, 2 * nv * vbytes);
                const z2* row = a.stencil + d.stc_off + (long long)i * ns * d.m;
                for (int q = 0; q < nv; q++) {
                    bulk_g2s(cpb + q * mpmax, row + sl_u[q] * d.m, vbytes, cfull);
                    bulk_g2s(cpb + (3 + q) * mpmax, row + sl_l[q] * d.m, vbytes, cfull);
                }
                cph ^= 1;
                const z2* blk = a.dinvB + C.off + (long long)i * C.mp * C.S;
                for (int c0 = 0; c0 < C.mp; c0 += KC) {
                    mbar_wait(&empty[slot], ph ^ 1);
                    mbar_arrive_expect_tx(&full[slot], bytes);
                    bulk_g2s(ringb + (size_t)slot * slot_bytes, blk + (long long)c0 * C.S, bytes, &full[slot]);
                    if (++slot == (uint32_t)NSL) {
                        slot = 0;
                        ph ^= 1;
                    }
                }
                }
                if (split) __syncwarp();
            }
        }
        return;
    }

    // ------------------------------------------------------------------------ consumers
    uint32_t slot = 0, ph = 0, cph = 0;
    z2* scr = a.scratch + (long long)blockIdx.x * a.scratch_per_cta;   // [hi-lo+1][NT][mp]
    for (int w = cid; w < a.ntiles; w += ncl) {
        const BatchTile T = a.tiles[w];
        if (tid == 0) {
            s_c = a.cls[T.cls];
            s_d = a.desc[s_c.rep];
        }
        const int cnt = T.cnt;
        if (tid < NT) {
            const int j = tid < cnt ? a.members[T.first + tid] : -1;
            s_sub[tid] = j;
            s_gx[tid] = j >= 0 ? a.desc[j].gx0 : 0;
            s_gy[tid] = j >= 0 ? a.desc[j].gy0 : 0;
        }
        consumer_bar(nct);
        const SubDesc& d = s_d;
        const BatchClass& C = s_c;
        const int m = d.m, mp = C.mp;
        const int S = nsteps_role(d, role);
        const bool mw = warp * 8 < mp;   // this warp owns factor rows [8 warp, 8 warp + 8)
        // Phase-A mapping: thread tid owns row tr of the subdomain columns q = tq + k P (P = nct / mp >= 4 rows of mp
        // threads per pass, k < 4), so its coupling coefficients are read once per step for all its columns.  The
        // restricted inputs b_i (the gather R_j r) are loaded one step ahead, in flight under the DMMAs.
        const int P = nct / mp, tq = tid / mp, tr = tid - tq * mp;
        const bool ract = tq < P;
        auto load_b = [&](int s2, z2(&pb)[4]) {
            if (s2 >= S || !ract) return;
            const Step sn = step_role(d, role, s2);
            if (sn.ph > PH_Z) return;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int q = tq + k * P;
                pb[k] = (q < cnt && tr < m)
                            ? __ldg(a.in + (s_gx[q] + tr - a.in_i0) + a.in_stride * (long long)(s_gy[q] + sn.i - a.in_j0))
                            : zmk(0, 0);
            }
        };
        z2 pb[4];
        load_b(0, pb);
        for (int s = 0; s <= S; s++) {
            if (role) {
                // split tile: the carry exchanges at the twist (z_{tw+1} to rank 1, x_tw back to rank 0), each
                // copied into the peer's top-chain carry through distributed shared memory
                auto send = [&](const z2* src) {
                    z2* dst = cg::this_cluster().map_shared_rank(vt, 2 - role);
                    for (int e = tid; e < NT * SV; e += nct) dst[e] = src[e];
                };
                if (s == xchg1(d, role)) {
                    if (role == 1) send(vt);
                    cg::this_cluster().sync();
                    if (role == 1) cg::this_cluster().sync();
                }
                if (role == 2 && s == d.tw + 1) {
                    send(vb);
                    cg::this_cluster().sync();
                }
            }
            if (s == S) break;
            BPROF(5);
            const Step st = step_role(d, role, s);
            const z2 cb[4] = {pb[0], pb[1], pb[2], pb[3]};
            if (mw && st.ph >= PH_D)   // the epilogue's y_i / z_i entries: on their way to L1 under phase A and the DMMAs
#pragma unroll
                for (int ct = 0; ct < 2; ct++) {
                    const int q = 8 * ct + 2 * t4;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(scr + ((long long)(st.i - d.lo) * NT + q) * mp + 8 * warp + g));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(scr + ((long long)(st.i - d.lo) * NT + q + 1) * mp + 8 * warp + g));
                }
            mbar_wait(cfull, cph);
            BPROF(6);
            // ---- right-hand sides R[q][tr] of this block step: r = [b_i] - C1 v1 [- C2 v2] (T: U_i z_{i+1}; B: L_i
            // y_{i-1}; Z: both) or r = C1 v1 (D: U_i x_{i+1}; U: L_i x_{i-1}); the step's form is uniform, so it is
            // resolved once and the thread's four columns run as independent chains
            if (ract) {
                const Cp up = {cpb[tr], cpb[2 * mpmax + tr], cpb[mpmax + tr]};                  // d = N, lo = NW, hi = NE
                const Cp dn = {cpb[3 * mpmax + tr], cpb[4 * mpmax + tr], cpb[5 * mpmax + tr]};  // S, SW, SE
                const bool hb = st.ph <= PH_Z;                                   // restricted input present
                const bool lower = st.ph == PH_B || st.ph == PH_U || st.ph == PH_Z;
                const bool use1 = st.ph == PH_T ? st.i < d.nb - 1 : (st.ph == PH_B || st.ph == PH_Z) ? st.i > 0 : true;
                const bool use2 = st.ph == PH_Z && st.i < d.nb - 1;              // the twist's U_tw z_{tw+1}
                const double sg = hb ? -1.0 : 1.0;
                const Cp c0 = lower ? dn : up;
                const Cp c1 = {zscale(c0.d, sg), zscale(c0.lo, sg), zscale(c0.hi, sg)};
                const Cp c2 = {zscale(up.d, -1.0), zscale(up.lo, -1.0), zscale(up.hi, -1.0)};
                const z2* v1 = (st.ph == PH_B || st.ph == PH_Z || st.ph == PH_D) ? vb : vt;
                const bool lo_ok = tr > 0, hi_ok = tr + 1 < m;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const int q = tq + k * P;
                    if (q < NT) {
                        z2 r = zmk(0, 0);
                        if (q < cnt && tr < m) {
                            if (hb) r = cb[k];
                            if (use1) {
                                const z2* v = v1 + q * SV + tr;
                                zfma(r, c1.d, v[0]);
                                if (lo_ok) zfma(r, c1.lo, v[-1]);
                                if (hi_ok) zfma(r, c1.hi, v[1]);
                            }
                            if (use2) {
                                const z2* v = vt + q * SV + tr;
                                zfma(r, c2.d, v[0]);
                                if (lo_ok) zfma(r, c2.lo, v[-1]);
                                if (hi_ok) zfma(r, c2.hi, v[1]);
                            }
                        }
                        R[q * SR + tr] = r;
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(cempty);
            cph ^= 1;
            BPROF(0);
            consumer_bar(nct);
            BPROF(1);
            load_b(s + 1, pb);
            // ---- Y = F_i R on the tensor cores, three real products per complex k-step and column tile (3M:
            // p1 = Fr Rr, p2 = Fi Ri, p3 = (Fr + Fi)(Rr + Ri); re = p1 - p2, im = p3 - p1 - p2), each in its own
            // accumulator; the operand sums run on the FP64 pipe beside the tensor pipe
            double p1[2][2] = {}, p2[2][2] = {}, p3[2][2] = {};
            for (int c0 = 0; c0 < mp; c0 += KC) {
                BPROF(3);
                mbar_wait(&full[slot], ph);
                BPROF(2);
                if (mw) {
                    const z2* F = reinterpret_cast<const z2*>(ringb + (size_t)slot * slot_bytes);
#pragma unroll
                    for (int ks = 0; ks < KC / 4; ks++) {
                        const z2 av = F[(4 * ks + t4) * C.S + 8 * warp + g];
                        const double as = av.x + av.y;
                        const int kk = c0 + 4 * ks + t4;
#pragma unroll
                        for (int ct = 0; ct < 2; ct++) {
                            if (ct == 1 && cnt <= 8) break;   // 8-wide tile: one column tile
                            const z2 bv = R[(8 * ct + g) * SR + kk];
                            dmma(p1[ct][0], p1[ct][1], av.x, bv.x);
                            dmma(p2[ct][0], p2[ct][1], av.y, bv.y);
                            dmma(p3[ct][0], p3[ct][1], as, bv.x + bv.y);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == (uint32_t)NSL) {
                    slot = 0;
                    ph ^= 1;
                }
            }
            BPROF(3);
            // ---- finish the step: carries, y / z scratch, owner write
            if (mw) {
                const int t = 8 * warp + g;
#pragma unroll
                for (int ct = 0; ct < 2; ct++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int q = 8 * ct + 2 * t4 + e;
                        if (q >= cnt || t >= m) continue;
                        const z2 acc = zmk(p1[ct][e] - p2[ct][e], (p3[ct][e] - p1[ct][e]) - p2[ct][e]);
                        z2* sc = scr + ((long long)(st.i - d.lo) * NT + q) * mp + t;
                        if (st.ph == PH_T) {
                            vt[q * SV + t] = acc;
                            if (st.i <= d.hi) *sc = acc;
                        } else if (st.ph == PH_B) {
                            vb[q * SV + t] = acc;
                            if (st.i >= d.lo) *sc = acc;
                        } else {
                            z2 x;
                            if (st.ph == PH_Z) {
                                x = acc;
                                vb[q * SV + t] = x;
                                vt[q * SV + t] = x;
                            } else {
                                x = zsub(*sc, acc);
                                (st.ph == PH_D ? vb : vt)[q * SV + t] = x;
                            }
                            if (t >= d.olo && t <= d.ohi) {
                                const int gx = s_gx[q] + t, gy = s_gy[q] + st.i;
                                if (a.pou_buf) {
                                    // linear-ramp PoU: chi_j-weighted solution into the subdomain's slot
                                    const SubDesc& dj = a.desc[s_sub[q]];
                                    const double wgt = chi_ramp(gx, dj.s0x, dj.s1x, a.delta, dj.flags & 1, dj.flags & 2) *
                                                       chi_ramp(gy, dj.s0y, dj.s1y, a.delta, dj.flags & 4, dj.flags & 8);
                                    a.pou_buf[dj.pou_off + (t - d.olo) + (long long)(d.ohi - d.olo + 1) * (st.i - d.lo)] =
                                        zscale(x, wgt);
                                } else {
                                    a.out[(gx - a.out_i0) + a.out_stride * (long long)(gy - a.out_j0)] = x;
                                }
                            }
                        }
                    }
            }
            BPROF(4);
            consumer_bar(nct);
        }
    }
#ifdef HELM_BATCH_PROF
    if (tid == 0 && blockIdx.x == 0)
        printf("BPROF cpl_wait %lld rhs %lld bar_rhs %lld ring_wait %lld dmma %lld epilogue %lld bar_end %lld\n", bpr[6],
               bpr[0], bpr[1], bpr[2], bpr[3], bpr[4], bpr[5]);
#endif
}

// one instance per CTA size (consumer warps = mp_max / 8, plus the producer warp), two CTAs per SM up to mp_max = 88
// (one CTA's serial phases -- right-hand sides, epilogue, barriers -- then run under the other's DMMAs)
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_apply_batch(BatchArgs a, int ncw, int mpmax, int slot_bytes, int nslots,
                                                            int split)
{
    batch_body(a, ncw, mpmax, slot_bytes, nslots, split);
}

const void* batch_fn(int block)
{
    if (block <= 288) return (const void*)k_apply_batch<288, 2>;
    if (block <= 384) return (const void*)k_apply_batch<384, 2>;
    return (const void*)k_apply_batch<544, 1>;
}

int batch_smem(int mpmax, int nslots, int slot_bytes)
{
    return nslots * slot_bytes + 2 * nslots * 8 + 16 + NT * (mpmax + 4) * (int)sizeof(z2) +
           2 * NT * (mpmax + 1) * (int)sizeof(z2) + 6 * mpmax * (int)sizeof(z2);
}

// class factors: standard layout (m x m column-major blocks at fac_off) -> batch layout
__global__ void k_relayout_batch(const z2* __restrict__ dinv, long long fac_off, int m, int nb, z2* __restrict__ dst,
                                 int mp, int S)
{
    const long long n = (long long)nb * mp * S;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e % S);
        const long long ck = e / S;
        const int k = (int)(ck % mp), i = (int)(ck / mp);
        dst[e] = (r < m && k < m) ? dinv[fac_off + (long long)i * m * m + (long long)k * m + r] : zmk(0, 0);
    }
}

// diff[p] = 1 iff the local stencils of pairs[p].x and pairs[p].y differ in any bit (same m, nb, ns by construction)
__global__ void k_stencil_eq(const SubDesc* __restrict__ desc, const z2* __restrict__ stc, const int2* __restrict__ pairs,
                             int npairs, int* __restrict__ diff)
{
    for (int p = blockIdx.x; p < npairs; p += gridDim.x) {
        const SubDesc x = desc[pairs[p].x], y = desc[pairs[p].y];
        const long long n = 2LL * x.nb * x.ns * x.m;
        const unsigned long long* u = reinterpret_cast<const unsigned long long*>(stc + x.stc_off);
        const unsigned long long* v = reinterpret_cast<const unsigned long long*>(stc + y.stc_off);
        int bad = 0;
        for (long long e = threadIdx.x; e < n; e += blockDim.x) bad |= (__ldg(u + e) != __ldg(v + e));
        bad = __syncthreads_or(bad);
        if (threadIdx.x == 0) diff[p] = bad;
    }
}

}  // namespace

int batch_configure(int mpmax, int* block, int* smem, int* slot_bytes, int* nslots, int* ctas_per_sm)
{
    const int ncw = mpmax / 8;
    *block = 32 * (ncw + 1);
    *slot_bytes = KC * (mpmax + 2) * (int)sizeof(z2);
    const void* fn = batch_fn(*block);
    // the deepest ring (<= 6 slots) that keeps two CTAs per SM, else the deepest that fits one (measured at c3:
    // two CTAs of 4 slots 1.63 ms; one CTA of 6 slots 2.19 ms; one CTA running the two chains in lockstep, 1.93 ms)
    const char* env = getenv("HELM_BATCH_SLOTS");   // tuning override: ring depth (the CTAs per SM follow)
    const int force = env ? atoi(env) : 0;
    for (int want = 2; want >= 1; want--)
        for (int ns = 6; ns >= 2; ns--) {
            if (force > 0 && ns != force) continue;
            const int sm = batch_smem(mpmax, ns, *slot_bytes);
            raise_smem_attr(fn, sm);
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, *block, sm) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            if (occ >= want || (force > 0 && occ >= 1)) {
                *smem = sm;
                *nslots = ns;
                *ctas_per_sm = occ;
                return ncw;
            }
        }
    *ctas_per_sm = 0;
    return ncw;
}

int launch_apply_batch(const BatchArgs& a, int grid, int block, int smem, int slot_bytes, int nslots, int mpmax,
                       int split, cudaStream_t s)
{
    const void* fn = batch_fn(block);
    raise_smem_attr(fn, smem);
    const int ncw = block / 32 - 1;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = split ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (block <= 288) e = cudaLaunchKernelEx(&cfg, k_apply_batch<288, 2>, a, ncw, mpmax, slot_bytes, nslots, split);
    else if (block <= 384) e = cudaLaunchKernelEx(&cfg, k_apply_batch<384, 2>, a, ncw, mpmax, slot_bytes, nslots, split);
    else e = cudaLaunchKernelEx(&cfg, k_apply_batch<544, 1>, a, ncw, mpmax, slot_bytes, nslots, split);
    return (int)e;
}

void launch_relayout_batch(const z2* dinv, long long fac_off, int m, int nb, z2* dst, int mp, int S, cudaStream_t s)
{
    k_relayout_batch<<<148, 256, 0, s>>>(dinv, fac_off, m, nb, dst, mp, S);
}

void launch_stencil_eq(const SubDesc* desc, const z2* stc, const int2* pairs, int npairs, int* diff, cudaStream_t s)
{
    if (npairs > 0) k_stencil_eq<<<std::min(npairs, 148 * 8), 256, 0, s>>>(desc, stc, pairs, npairs, diff);
}
