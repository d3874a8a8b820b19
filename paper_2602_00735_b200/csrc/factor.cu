// factor.cu -- K3: setup factorisation of every local operator A_j (exact local solves, P:143-147 A_j^-1).
//
// A_j is block tridiagonal in its local x-fastest numbering (7-point SW->NE stencil, D1): block row i
// holds T_i (tridiagonal: C, E, W), L_i = A_{i,i-1} (S on the diagonal, SW below it) and
// U_i = A_{i,i+1} (N on the diagonal, NE above it).  We use a TWISTED block LU:
//   bottom chain  P_0 = T_0,        P_i = T_i - L_i P_{i-1}^-1 U_{i-1},        i = 1 .. tw-1
//   top chain     Q_{nb-1} = T_{nb-1}, Q_i = T_i - U_i Q_{i+1}^-1 L_{i+1},      i = nb-2 .. tw+1
//   twist         Z = T_tw - L_tw P_{tw-1}^-1 U_{tw-1} - U_tw Q_{tw+1}^-1 L_{tw+1}
// and store the explicit inverse of each block (P_i^-1, Z^-1, Q_i^-1) in block slot i, column-major.
// Each inverse is formed by blocked Gauss-Jordan elimination WITHOUT pivoting (D12: the oracle's band LU is
// unpivoted too) with 8-column panels: the 8 x 8 pivot block inverted in one warp's registers (the serial part),
// the row panel / trailing update / column panel on the FP64 tensor cores (DMMA), the next pivot block formed and
// inverted by warp 0 while the other warps finish the trailing update (gj_panels8); a zero, non-finite or tiny pivot (|pivot| < 1e-12, against O(1) stencil entries) raises
// HELM_EZEROPIVOT naming subdomain, block and row.
// The two chains run in separate CTAs; a second launch forms the twist blocks.  Blocks wider than M_SMEM use
// thread-block clusters and blocked Gauss-Jordan in global memory (k_factor_big).  The 9-point Q1 stencil (D18)
// adds a third diagonal to L_i (SE) and U_i (NW).
#include <stdio.h>

#include <stdlib.h>

#include "internal.cuh"

namespace {

constexpr int FT = 512;  // threads per factor CTA
constexpr int GB = 32;   // Gauss-Jordan panel width
constexpr int DLD = GB + 1;

// acc -= a * b
__device__ __forceinline__ void zfms(z2& acc, z2 a, z2 b)
{
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(-a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

// FP64 tensor cores (DMMA, mma.sync m8n8k4): d += a b for one 8 x 8 x 4 real tile per warp.  Fragments: a = A[g][t],
// b = B[t][g], c = (C[g][2t], C[g][2t+1]) with g = lane / 4, t = lane % 4.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Complex 8 x 8 tile update C -= A B over k in [0, kw) on the tensor cores, with A(r, q) = la(r, q), B(q, c) = lb(q, c)
// supplied as accessors returning complex values (zero outside the matrix): Cr += (-Ar) Br + Ai Bi,
// Ci += (-Ar) Bi + (-Ai) Br -- four real DMMAs per k-step of 4.
// The four real products accumulate into four independent fragments (C_r += -A_r B_r, R2 += A_i B_i, C_i += -A_r B_i,
// I2 += -A_i B_r), summed at the end: the dependent DMMA chain per tile is half as long (the factorisation's trailing
// tiles are latency-bound on it: ncu "wait" stalls on the NOPs between dependent DMMAs).
template <class LA, class LB>
__device__ __forceinline__ void ztile_fms(z2& c0, z2& c1, int kw, LA la, LB lb)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    double r20 = 0.0, r21 = 0.0, i20 = 0.0, i21 = 0.0;
    for (int k = 0; k < kw; k += 4) {
        const z2 a = k + t < kw ? la(g, k + t) : zmk(0, 0);
        const z2 b = k + t < kw ? lb(k + t, g) : zmk(0, 0);
        dmma(c0.x, c1.x, -a.x, b.x);
        dmma(r20, r21, a.y, b.y);
        dmma(c0.y, c1.y, -a.x, b.y);
        dmma(i20, i21, -a.y, b.x);
    }
    c0.x += r20;
    c1.x += r21;
    c0.y += i20;
    c1.y += i21;
}

// D (kw x kw, row-major, stride DLD, kw <= 32) <- D^-1 by unpivoted in-place Gauss-Jordan, executed by the first
// GJW warps of the CTA (lane c owns column c, warp w the rows r = w, w + GJW, ...; named barrier 2 over those warps
// only).  A zero pivot is recorded as row kb + p.
// Shared-memory layout of the block S being inverted: row stride ld = round_up(m, 8) + 4 16-B words (== 4 mod 8) and
// the column swizzle c ^ (r & 3).  An LDS.128 is served 8 lanes at a time; with this layout the DMMA fragment loads of
// both operands -- A (lanes: rows g in {2h, 2h+1}, columns t in 0..3) and B (rows t, columns g) -- AND the loads and
// stores of the accumulator tile C (rows g in {2h, 2h+1}, columns 2t or 2t + 1) hit 8 distinct 16-B bank groups per
// quarter warp.  (ld == 1 mod 8 left A and B 2-way conflicted: 5.3e9 excess wavefronts at c3; the swizzle c ^ (r & 2)
// fixed those but left C 2-way conflicted: 3.9e9 excess shared-load wavefronts, ncu.)
__host__ __device__ __forceinline__ int lds_of(int m) { return ((m + 7) / 8) * 8 + 4; }
__device__ __forceinline__ int sx(int r, int c, int ld) { return r * ld + (c ^ (r & 3)); }

constexpr int GJW = 8;
// |pivot| < 1e-12 is reported as singular: the stencil entries of A_j are O(1e-3 .. 10) (P1/Q1 stiffness is
// scale-free in 2D; |gamma|^-2 >= 1e-3 in every PML used here), so such a pivot means cond > 1e12
constexpr double PIV_TINY2 = 1e-24;

__device__ __forceinline__ void gj_bar() { asm volatile("bar.sync 2, %0;" ::"r"(GJW * 32) : "memory"); }

__device__ void warp_gj(z2* D, int kw, int kb, int* bad)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int p = 0; p < kw; p++) {
        const z2 pv = D[p * DLD + p];
        const bool zero = !(pv.x * pv.x + pv.y * pv.y >= PIV_TINY2);   // zero, tiny or not finite
        if (zero && threadIdx.x == 0 && *bad < 0) *bad = kb + p;
        const z2 inv = zero ? zmk(0, 0) : zinv(pv);
        z2 rp = lane < kw ? D[p * DLD + lane] : zmk(0, 0);
        if (lane != p) rp = zmul(rp, inv);                         // row p scaled (pivot column excluded)
        gj_bar();                                                   // everyone has read row p before it changes
        if (lane < kw && lane != p) {
#pragma unroll 4
            for (int r = w; r < kw; r += GJW)
                if (r != p) zfms(D[r * DLD + lane], D[r * DLD + p], rp);   // column p is read, never written here
        }
        gj_bar();
        if (w == 0 && lane < kw) {
            if (lane != p) {
                const z2 f = D[lane * DLD + p];
                z2 v = zmk(0, 0);
                zfms(v, f, inv);
                D[lane * DLD + p] = v;                               // column p: -D[r][p] / pivot
                D[p * DLD + lane] = rp;
            } else {
                D[p * DLD + p] = inv;
            }
        }
        gj_bar();
    }
}

// The same inverse with the matrix in REGISTERS of the GJW = 8 warps: warp w holds rows w, w + 8, w + 16, w + 24 (lane
// c = column c), so the pivot column reaches every row by a shuffle and only the scaled pivot row goes through shared
// memory (a two-slot buffer, so one named barrier per pivot instead of three).  Per entry the arithmetic is
// warp_gj's, in the same order:
//   D[p][c] <- D[p][c] / D[p][p];  D[r][c] <- D[r][c] - D[r][p] D[p][c];  D[r][p] <- -D[r][p] / D[p][p];
//   D[p][p] <- 1 / D[p][p]          (r != p, c != p).  A zero pivot is recorded as row kb + p.
__device__ __forceinline__ z2 shfl_z(z2 v, int src)
{
    return zmk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

__device__ void warp_gj8(z2* D, z2* rowbuf /* 2 x 32 */, int kw, int kb, int* bad)
{
    static_assert(GB == 4 * GJW, "four rows per warp");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    z2 row[4];
#pragma unroll
    for (int s4 = 0; s4 < 4; s4++) {
        const int r = w + GJW * s4;
        row[s4] = (r < kw && lane < kw) ? D[r * DLD + lane] : zmk(0, 0);
    }
#pragma unroll
    for (int p = 0; p < GB; p++) {
        if (p >= kw) break;
        z2* rb = rowbuf + (p & 1) * GB;
        if (w == p % GJW) {   // owner of row p: scale it, publish it
            const z2 pv = shfl_z(row[p / GJW], p);
            const bool zero = !(pv.x * pv.x + pv.y * pv.y >= PIV_TINY2);   // zero, tiny or not finite
            if (zero && lane == 0 && *bad < 0) *bad = kb + p;
            const double rd = zero ? 0.0 : 1.0 / (pv.x * pv.x + pv.y * pv.y);   // one division per pivot
            const z2 inv = zmk(pv.x * rd, -pv.y * rd);
            const z2 v = lane == p ? inv : zmul(row[p / GJW], inv);
            row[p / GJW] = v;
            rb[lane] = v;
        }
        gj_bar();
        const z2 b = rb[lane], inv = rb[p];
#pragma unroll
        for (int s4 = 0; s4 < 4; s4++) {
            if (w + GJW * s4 == p) continue;
            const z2 f = shfl_z(row[s4], p);   // D[r][p]
            if (lane != p) {
                zfms(row[s4], f, b);
            } else {
                z2 v = zmk(0, 0);
                zfms(v, f, inv);
                row[s4] = v;
            }
        }
    }
#pragma unroll
    for (int s4 = 0; s4 < 4; s4++) {
        const int r = w + GJW * s4;
        if (r < kw && lane < kw) D[r * DLD + lane] = row[s4];
    }
}

// 8 x 8 inverse in the registers of ONE warp, in the DMMA accumulator layout (lane l holds row g = l / 4, columns
// 2 (l % 4) and 2 (l % 4) + 1): unpivoted Gauss-Jordan (D12), the pivot and the pivot row reach the other lanes by
// shuffles -- no shared memory, no barrier.  Rows / columns >= w8 must hold the identity.  A zero / tiny pivot is
// recorded as row kbase + p.
__device__ __forceinline__ void inv8_regs(z2& x0, z2& x1, int w8, int kbase, int* bad)
{
    const int lane = threadIdx.x & 31, r = lane >> 2, t = lane & 3, c0 = 2 * t, c1 = 2 * t + 1;
#pragma unroll
    for (int p = 0; p < 8; p++) {
        const z2 mine = (p & 1) ? x1 : x0;
        const z2 pv = shfl_z(mine, 4 * p + (p >> 1));          // D[p][p]
        const z2 f = shfl_z(mine, (lane & ~3) + (p >> 1));     // D[r][p] of my row, before the update
        const bool zero = !(pv.x * pv.x + pv.y * pv.y >= PIV_TINY2);
        if (zero && p < w8 && lane == 0 && *bad < 0) *bad = kbase + p;
        const double rd = zero ? 0.0 : 1.0 / (pv.x * pv.x + pv.y * pv.y);
        const z2 inv = zmk(pv.x * rd, -pv.y * rd);
        const z2 s0 = c0 == p ? inv : zmul(x0, inv), s1 = c1 == p ? inv : zmul(x1, inv);   // pivot row scaled
        const z2 y0 = shfl_z(s0, 4 * p + t), y1 = shfl_z(s1, 4 * p + t);
        if (r == p) {
            x0 = s0;
            x1 = s1;
        } else {
            const z2 b0 = c0 == p ? inv : y0, b1 = c1 == p ? inv : y1;
            if (c0 == p) x0 = zmk(0, 0);                       // -D[r][p] / pivot
            if (c1 == p) x1 = zmk(0, 0);
            zfms(x0, f, b0);                                   // D[r][c] - D[r][p] D[p][c]
            zfms(x1, f, b1);
        }
    }
}

// Couplings of block row i as m x m matrices (7-point P1: two diagonals; 9-point Q1: three):
//   L_i[a][a] = S_i(a), L_i[a][a-1] = SW_i(a), L_i[a][a+1] = SE_i(a)          (A_{i,i-1})
//   U_i[a][a] = N_i(a), U_i[a][a+1] = NE_i(a), U_i[a][a-1] = NW_i(a)          (A_{i,i+1})
// Wl(c, d) reads W = the inverse stored column-major in global memory.
struct Cpl { const z2 *d, *lo, *hi; };   // diagonal, sub-diagonal (entry [a][a-1]) and super ([a][a+1]) vectors

// (L_i W U_{i-1})(a,b) = sum_c L[a][c] sum_d W[c][d] U[d][b];  U[d][b]: d = b N(b), d = b-1 NE(b-1), d = b+1 NW(b+1).
// Branch-free: the three coefficients of each factor and the nine W entries (indices clamped into the block, their
// coefficient zero when clamped) are loaded together, so the L2 round trips of one entry overlap instead of chaining
// through data-dependent tests (ncu at c3: long-scoreboard stalls on these loads were 12 % of the kernel's samples).
__device__ __forceinline__ z2 cpl3(const z2* __restrict__ W, int m, int a, int b, z2 l0, z2 l1, z2 l2, z2 u0, z2 u1,
                                   z2 u2)
{
    const int cm = a > 0 ? a - 1 : a, cp = a + 1 < m ? a + 1 : a;
    const int dm = b > 0 ? b - 1 : b, dp = b + 1 < m ? b + 1 : b;
    const z2* w0 = W + (long long)dm * m;
    const z2* w1 = W + (long long)b * m;
    const z2* w2 = W + (long long)dp * m;
    const z2 x00 = w0[cm], x01 = w1[cm], x02 = w2[cm];
    const z2 x10 = w0[a], x11 = w1[a], x12 = w2[a];
    const z2 x20 = w0[cp], x21 = w1[cp], x22 = w2[cp];
    const z2 r0 = zadd(zadd(zmul(x00, u0), zmul(x01, u1)), zmul(x02, u2));
    const z2 r1 = zadd(zadd(zmul(x10, u0), zmul(x11, u1)), zmul(x12, u2));
    const z2 r2 = zadd(zadd(zmul(x20, u0), zmul(x21, u1)), zmul(x22, u2));
    return zadd(zadd(zmul(l0, r0), zmul(l1, r1)), zmul(l2, r2));
}

__device__ __forceinline__ z2 term_below(const z2* __restrict__ W, int m, int a, int b, Cpl L, Cpl U)
{
    const z2 zero = zmk(0, 0);
    const z2 l0 = a > 0 ? L.lo[a] : zero, l1 = L.d[a], l2 = (L.hi && a + 1 < m) ? L.hi[a] : zero;
    const z2 u0 = b > 0 ? U.hi[b - 1] : zero, u1 = U.d[b], u2 = (U.lo && b + 1 < m) ? U.lo[b + 1] : zero;
    return cpl3(W, m, a, b, l0, l1, l2, u0, u1, u2);
}

// (U_i W L_{i+1})(a,b) = sum_c U[a][c] sum_d W[c][d] L[d][b];  L[d][b]: d = b S(b), d = b+1 SW(b+1), d = b-1 SE(b-1)
__device__ __forceinline__ z2 term_above(const z2* __restrict__ W, int m, int a, int b, Cpl U, Cpl L)
{
    const z2 zero = zmk(0, 0);
    const z2 c0 = (U.lo && a > 0) ? U.lo[a] : zero, c1 = U.d[a], c2 = a + 1 < m ? U.hi[a] : zero;
    const z2 d0 = (L.hi && b > 0) ? L.hi[b - 1] : zero, d1 = L.d[b], d2 = b + 1 < m ? L.lo[b + 1] : zero;
    return cpl3(W, m, a, b, c0, c1, c2, d0, d1, d2);
}

__device__ __forceinline__ Cpl lower_of(const z2* row, int m, int ns)   // L of a block row
{
    return Cpl{row + SL_S * m, row + SL_SW * m, ns == 9 ? row + SL_SE * m : nullptr};
}
__device__ __forceinline__ Cpl upper_of(const z2* row, int m, int ns)   // U of a block row
{
    return Cpl{row + SL_N * m, ns == 9 ? row + SL_NW * m : nullptr, row + SL_NE * m};
}

// Schur complement entry (a, b) of block row i: mode 0 bottom chain (P_i), 1 top chain (Q_i), 2 twist (Z)
__device__ __forceinline__ z2 schur_entry(const SubDesc& d, int i, int mode, const z2* __restrict__ stc,
                                          const z2* __restrict__ dinv, int a, int b)
{
    const int m = d.m, ns = d.ns;
    const z2* rowi = stc + d.stc_off + (long long)i * ns * m;
    z2 v = zmk(0, 0);
    if (b == a) v = rowi[SL_C * m + a];
    else if (b == a + 1) v = rowi[SL_E * m + a];
    else if (b == a - 1) v = rowi[SL_W * m + a];
    if ((mode == 0 || mode == 2) && i > 0) {
        const z2* Wb = dinv + d.fac_off + (long long)(i - 1) * m * m;
        const z2* rowm = stc + d.stc_off + (long long)(i - 1) * ns * m;
        v = zsub(v, term_below(Wb, m, a, b, lower_of(rowi, m, ns), upper_of(rowm, m, ns)));
    }
    if ((mode == 1 || mode == 2) && i < d.nb - 1) {
        const z2* Wa = dinv + d.fac_off + (long long)(i + 1) * m * m;
        const z2* rowp = stc + d.stc_off + (long long)(i + 1) * ns * m;
        v = zsub(v, term_above(Wa, m, a, b, upper_of(rowi, m, ns), lower_of(rowp, m, ns)));
    }
    return v;
}

struct FactorSmem {
    z2* S;       // [m][lds] row-major, swizzled (sx)
    z2* Dk[2];   // pivot-block inverses: [GB][DLD] (32-wide path) / the current and the next 8 x 8 (8-wide path)
    z2* rowbuf;  // [2][GB] warp_gj8's pivot-row buffer
};

// mode: 0 bottom chain block, 1 top chain block, 2 twist block
__device__ void build_block(const SubDesc& d, int i, int mode, const z2* __restrict__ stc, const z2* __restrict__ dinv,
                            FactorSmem sm)
{
    const int m = d.m, ld = lds_of(m);
    // consecutive threads take consecutive ROWS a: the column-major W entries W[d m + c], c = a - 1 .. a + 1, and the
    // coupling vectors L.*[a] / U.*[a] are then coalesced (with b fastest every W load of a warp touched 32 lines --
    // the build took a third of the factorisation)
#pragma unroll 2
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int b = e / m, a = e - b * m;
        sm.S[sx(a, b, ld)] = schur_entry(d, i, mode, stc, dinv, a, b);
    }
    __syncthreads();
}

// In-place inversion of S (m x m, row-major, stride ld, shared memory) by blocked, unpivoted Gauss-Jordan with panels K
// of GB columns (unpivoted, D12; on the bottom chain the pivots are the oracle's no-pivot band-LU pivots):
//   Dk = S[K,K]^-1 (8 warps);  S[K,j] = Dk S[K,j] (j not in K);  S[i,j] -= S[i,K] S[K,j] (i, j not in K);
//   S[i,K] = -S[i,K] Dk (i not in K);  S[K,K] = Dk.
// All three products (row panel, trailing update, column panel -- complex GEMMs, 32 deep) run on the FP64 tensor cores
// (DMMA), one warp per 8 x 8 tile; a panel warp loads its whole operand strip before writing, so they work in place.

// one warp: S[K,j] = Dk S[K,j] for the 8-column strip j0.. (B fragments loaded before the row tiles are written)
__device__ __forceinline__ void row_strip(z2* S, int ld, int m, int kb, int kw, const z2* Dk, int j0)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, col = j0 + g;
    z2 bf[GB / 4];
#pragma unroll
    for (int s4 = 0; s4 < GB / 4; s4++) {
        const int q = 4 * s4 + t;
        bf[s4] = (q < kw && col < m) ? S[sx(kb + q, col, ld)] : zmk(0, 0);
    }
#pragma unroll
    for (int rt = 0; rt < GB / 8; rt++) {
        if (8 * rt >= kw) break;
        z2 c0 = zmk(0, 0), c1 = zmk(0, 0);
#pragma unroll
        for (int s4 = 0; s4 < GB / 4; s4++) {
            if (4 * s4 >= kw) break;
            const int r = 8 * rt + g, q = 4 * s4 + t;
            const z2 a = (r < kw && q < kw) ? Dk[r * DLD + q] : zmk(0, 0);
            dmma(c0.x, c1.x, a.x, bf[s4].x);    // C += A B
            dmma(c0.x, c1.x, -a.y, bf[s4].y);
            dmma(c0.y, c1.y, a.x, bf[s4].y);
            dmma(c0.y, c1.y, a.y, bf[s4].x);
        }
        const int r = 8 * rt + g, cA = j0 + 2 * t;
        if (r < kw && cA < m) S[sx(kb + r, cA, ld)] = c0;
        if (r < kw && cA + 1 < m) S[sx(kb + r, cA + 1, ld)] = c1;
    }
}

// one warp: trailing tile S[i0.., j0..] -= S[i0.., K] S[K, j0..]
__device__ __forceinline__ void trail_tile(z2* S, int ld, int m, int kb, int kw, int i0, int j0)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int r = i0 + g, cA = j0 + 2 * t, cB = cA + 1;
    z2 c0 = (r < m && cA < m) ? S[sx(r, cA, ld)] : zmk(0, 0);
    z2 c1 = (r < m && cB < m) ? S[sx(r, cB, ld)] : zmk(0, 0);
    ztile_fms(
        c0, c1, kw, [&](int rr, int q) { return i0 + rr < m ? S[sx(i0 + rr, kb + q, ld)] : zmk(0, 0); },
        [&](int q, int cc) { return j0 + cc < m ? S[sx(kb + q, j0 + cc, ld)] : zmk(0, 0); });
    if (r < m && cA < m) S[sx(r, cA, ld)] = c0;
    if (r < m && cB < m) S[sx(r, cB, ld)] = c1;
}

// one warp: S[i, K] = -S[i, K] Dk for the 8-row strip i0.. (A fragments loaded before it writes)
__device__ __forceinline__ void col_strip(z2* S, int ld, int m, int kb, int kw, const z2* Dk, int i0)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, row = i0 + g;
    z2 af[GB / 4];
#pragma unroll
    for (int s4 = 0; s4 < GB / 4; s4++) {
        const int q = 4 * s4 + t;
        af[s4] = (q < kw && row < m) ? S[sx(row, kb + q, ld)] : zmk(0, 0);
    }
#pragma unroll
    for (int ct = 0; ct < GB / 8; ct++) {
        if (8 * ct >= kw) break;
        z2 c0 = zmk(0, 0), c1 = zmk(0, 0);
#pragma unroll
        for (int s4 = 0; s4 < GB / 4; s4++) {
            if (4 * s4 >= kw) break;
            const int q = 4 * s4 + t, c = 8 * ct + g;
            const z2 b = (q < kw && c < kw) ? Dk[q * DLD + c] : zmk(0, 0);
            dmma(c0.x, c1.x, -af[s4].x, b.x);   // C -= A B
            dmma(c0.x, c1.x, af[s4].y, b.y);
            dmma(c0.y, c1.y, -af[s4].x, b.y);
            dmma(c0.y, c1.y, -af[s4].y, b.x);
        }
        const int cA = 8 * ct + 2 * t;
        if (row < m && cA < kw) S[sx(row, kb + cA, ld)] = c0;
        if (row < m && cA + 1 < kw) S[sx(row, kb + cA + 1, ld)] = c1;
    }
}

// warps 0 .. GJW-1: Dk = S[K,K]^-1 (K = kb .. kb + kw - 1)
__device__ __forceinline__ void pivot_inverse(const z2* S, int ld, z2* Dk, z2* rowbuf, int kb, int kw, int* bad_row)
{
    const int tid = threadIdx.x;
    for (int e = tid; e < kw * kw; e += GJW * 32) {
        const int r = e / kw, c = e - r * kw;
        Dk[r * DLD + c] = S[sx(kb + r, kb + c, ld)];
    }
    gj_bar();
    warp_gj8(Dk, rowbuf, kw, kb, bad_row);
}

#ifdef HELM_FACTOR_PROF
#define CPROF(k) do { if (cpr) { const long long t_ = clock64(); cpr[k] += t_ - *ctp; *ctp = t_; } } while (0)
#define CPROF_ARGS , long long* cpr, long long* ctp
#define CPROF_PASS , cpr, ctp
#else
#define CPROF(k) do { } while (0)
#define CPROF_ARGS
#define CPROF_PASS
#endif

// Panels of 32 columns (the former default; HELM_FACTOR_PANEL=32 keeps it for A/B): the pivot inverse is warp_gj8,
// one 256-thread barrier per pivot.
__device__ void gj_blocked(int m, FactorSmem sm, int* bad_row CPROF_ARGS)
{
    const int ld = lds_of(m);
    z2* S = sm.S;
    const int tid = threadIdx.x, nw = blockDim.x >> 5, w = tid >> 5, mt = (m + 7) / 8;
    const z2* Dk = sm.Dk[0];
    for (int kb = 0; kb < m; kb += GB) {
        const int kw = min(GB, m - kb);
        if (tid < GJW * 32) pivot_inverse(S, ld, sm.Dk[0], sm.rowbuf, kb, kw, bad_row);
        __syncthreads();
        CPROF(1);
        // ---- row panel: S[K, j] = Dk S[K, j] (j not in K), one warp per 8-column strip
        for (int strip = w; strip < mt; strip += nw) {
            const int j0 = strip * 8;
            if (j0 >= kb && j0 < kb + kw) continue;
            row_strip(S, ld, m, kb, kw, Dk, j0);
        }
        __syncthreads();
        CPROF(2);
        // ---- trailing update S[i,j] -= S[i,K] S[K,j]: tiles aligned to the 32-column panels, so the panel's rows
        //      and columns are skipped as whole tiles
        for (int tile = w; tile < mt * mt; tile += nw) {
            const int i0 = (tile / mt) * 8, j0 = (tile % mt) * 8;
            if ((i0 >= kb && i0 < kb + kw) || (j0 >= kb && j0 < kb + kw)) continue;
            trail_tile(S, ld, m, kb, kw, i0, j0);
        }
        __syncthreads();
        CPROF(4);
        // ---- column panel: S[i, K] = -S[i, K] Dk (i not in K), one warp per 8-row strip; S[K, K] = Dk
        for (int strip = w; strip < mt; strip += nw) {
            const int i0 = strip * 8;
            if (i0 >= kb && i0 < kb + kw) continue;
            col_strip(S, ld, m, kb, kw, Dk, i0);
        }
        for (int e = tid; e < kw * kw; e += blockDim.x) {
            const int r = e / kw, c = e - r * kw;
            S[sx(kb + r, kb + c, ld)] = Dk[r * DLD + c];
        }
        __syncthreads();
        CPROF(5);
    }
}

// Panels of 8 columns (P8): the same blocked Gauss-Jordan with GB = 8.  The pivot inverse is the serial part of any
// blocked Gauss-Jordan (m pivots per block); with 8-wide panels it runs in ONE warp's registers (inv8_regs: no
// barrier per pivot), and warp 0 forms the NEXT panel's pivot tile (its trailing update, in the accumulator layout
// inv8_regs takes) and inverts it while warps 1.. finish the trailing update: three CTA barriers per 8 pivots instead
// of one 256-thread barrier per pivot.  The DMMA work (row panel, trailing update, column panel) is the same m^3.
// Full 8-wide panels (kw = 8) with S zero-padded to a multiple of 8 rows (padded rows / columns stay 0 through the
// elimination): no bounds tests, swizzle bits hoisted -- ncu at c3 counted 31 integer / control instructions per DMMA in
// the generic tile code (IMAD 26 %, ISETP 11 %, DMMA 3 % of the warp instructions), which left the kernel issue-bound.
// Row r's swizzle is c ^ (r & 3); rows kb + t and kb + 4 + t (kb a multiple of 8) both swizzle by t.
#ifndef HELM_TRAIL_SPLIT
#define HELM_TRAIL_SPLIT 0
#endif
constexpr bool TRAIL_SPLIT = HELM_TRAIL_SPLIT;   // split real / imaginary accumulators in the trailing tiles
template <bool STORE>
__device__ __forceinline__ void trail8(z2* S, int ld, int kb, int i0, int j0, z2& c0, z2& c1)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int r = i0 + g, sw = r & 3, tb = t;      // rows kb + t and kb + 4 + t swizzle by t
    z2* Sr = S + r * ld;
    const int cA = j0 + ((2 * t) ^ sw), cB = j0 + ((2 * t + 1) ^ sw);
    if (STORE) {
        c0 = Sr[cA];
        c1 = Sr[cB];
    }
    const z2 a0 = Sr[kb + (t ^ sw)], a1 = Sr[kb + ((4 + t) ^ sw)];
    const z2 b0 = S[(kb + t) * ld + ((j0 + g) ^ tb)], b1 = S[(kb + 4 + t) * ld + ((j0 + g) ^ tb)];
    if (TRAIL_SPLIT) {
        double r20 = 0.0, r21 = 0.0, i20 = 0.0, i21 = 0.0;
        dmma(c0.x, c1.x, -a0.x, b0.x);
        dmma(r20, r21, a0.y, b0.y);
        dmma(c0.y, c1.y, -a0.x, b0.y);
        dmma(i20, i21, -a0.y, b0.x);
        dmma(c0.x, c1.x, -a1.x, b1.x);
        dmma(r20, r21, a1.y, b1.y);
        dmma(c0.y, c1.y, -a1.x, b1.y);
        dmma(i20, i21, -a1.y, b1.x);
        c0.x += r20;
        c1.x += r21;
        c0.y += i20;
        c1.y += i21;
    } else {
        dmma(c0.x, c1.x, -a0.x, b0.x);
        dmma(c0.y, c1.y, -a0.x, b0.y);
        dmma(c0.x, c1.x, a0.y, b0.y);
        dmma(c0.y, c1.y, -a0.y, b0.x);
        dmma(c0.x, c1.x, -a1.x, b1.x);
        dmma(c0.y, c1.y, -a1.x, b1.y);
        dmma(c0.x, c1.x, a1.y, b1.y);
        dmma(c0.y, c1.y, -a1.y, b1.x);
    }
    if (STORE) {
        Sr[cA] = c0;
        Sr[cB] = c1;
    }
}

// S[K, j0..j0+7] = Dk S[K, j0..j0+7] (kw = 8): B fragments loaded before the tile is written
__device__ __forceinline__ void row8(z2* S, int ld, int kb, const z2* Dk, int j0)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, tb = t;
    const z2 b0 = S[(kb + t) * ld + ((j0 + g) ^ tb)], b1 = S[(kb + 4 + t) * ld + ((j0 + g) ^ tb)];
    const z2 a0 = Dk[g * DLD + t], a1 = Dk[g * DLD + 4 + t];
    double cr0 = 0.0, cr1 = 0.0, r20 = 0.0, r21 = 0.0, ci0 = 0.0, ci1 = 0.0, i20 = 0.0, i21 = 0.0;
    dmma(cr0, cr1, a0.x, b0.x);
    dmma(r20, r21, -a0.y, b0.y);
    dmma(ci0, ci1, a0.x, b0.y);
    dmma(i20, i21, a0.y, b0.x);
    dmma(cr0, cr1, a1.x, b1.x);
    dmma(r20, r21, -a1.y, b1.y);
    dmma(ci0, ci1, a1.x, b1.y);
    dmma(i20, i21, a1.y, b1.x);
    const int r = kb + g;
    z2* Sr = S + r * ld;
    Sr[j0 + ((2 * t) ^ (r & 3))] = zmk(cr0 + r20, ci0 + i20);
    Sr[j0 + ((2 * t + 1) ^ (r & 3))] = zmk(cr1 + r21, ci1 + i21);
}

// S[i0..i0+7, K] = -S[i0..i0+7, K] Dk (kw = 8): A fragments loaded before the tile is written
__device__ __forceinline__ void col8(z2* S, int ld, int kb, const z2* Dk, int i0)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int r = i0 + g, sw = r & 3;
    z2* Sr = S + r * ld;
    const z2 a0 = Sr[kb + (t ^ sw)], a1 = Sr[kb + ((4 + t) ^ sw)];
    const z2 b0 = Dk[t * DLD + g], b1 = Dk[(4 + t) * DLD + g];
    double cr0 = 0.0, cr1 = 0.0, r20 = 0.0, r21 = 0.0, ci0 = 0.0, ci1 = 0.0, i20 = 0.0, i21 = 0.0;
    dmma(cr0, cr1, -a0.x, b0.x);
    dmma(r20, r21, a0.y, b0.y);
    dmma(ci0, ci1, -a0.x, b0.y);
    dmma(i20, i21, -a0.y, b0.x);
    dmma(cr0, cr1, -a1.x, b1.x);
    dmma(r20, r21, a1.y, b1.y);
    dmma(ci0, ci1, -a1.x, b1.y);
    dmma(i20, i21, -a1.y, b1.x);
    Sr[kb + ((2 * t) ^ sw)] = zmk(cr0 + r20, ci0 + i20);
    Sr[kb + ((2 * t + 1) ^ sw)] = zmk(cr1 + r21, ci1 + i21);
}

__device__ void gj_panels8(int m, FactorSmem sm, int* bad_row CPROF_ARGS)
{
    const int ld = lds_of(m);
    z2* S = sm.S;
    const int tid = threadIdx.x, nw = blockDim.x >> 5, w = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int mt = (m + 7) / 8;
    int cur = 0;
    if (w == 0) {   // P_0 = S[0:8, 0:8]^-1
        const int w8 = min(8, m);
        z2 x0 = (g < w8 && 2 * t < w8) ? S[sx(g, 2 * t, ld)] : zmk(g == 2 * t ? 1.0 : 0.0, 0.0);
        z2 x1 = (g < w8 && 2 * t + 1 < w8) ? S[sx(g, 2 * t + 1, ld)] : zmk(g == 2 * t + 1 ? 1.0 : 0.0, 0.0);
        inv8_regs(x0, x1, w8, 0, bad_row);
        sm.Dk[0][g * DLD + 2 * t] = x0;
        sm.Dk[0][g * DLD + 2 * t + 1] = x1;
    }
    __syncthreads();
    CPROF(1);
    for (int kb = 0; kb < m; kb += 8) {
        const int kw = min(8, m - kb);
        const z2* Dk = cur ? sm.Dk[1] : sm.Dk[0];
        // ---- row panel: S[K, j] = Dk S[K, j] (j not in K), one 8 x 8 tile per warp
        const bool full = kw == 8;
        for (int strip = w; strip < mt; strip += nw)
            if (strip * 8 != kb) {
                if (full) row8(S, ld, kb, Dk, strip * 8);
                else row_strip(S, ld, m, kb, kw, Dk, strip * 8);
            }
        __syncthreads();
        CPROF(2);
        // ---- trailing update; warp 0 first forms and inverts the next pivot tile
        const int nk = kb + 8;
        if (w == 0 && nk < m) {
            const int w8 = min(8, m - nk);
            // (a next panel exists, so this one is full: kw = 8)
            z2 c0 = S[sx(nk + g, nk + 2 * t, ld)], c1 = S[sx(nk + g, nk + 2 * t + 1, ld)];
            trail8<false>(S, ld, kb, nk, nk, c0, c1);
            if (!(g < w8 && 2 * t < w8)) c0 = zmk(g == 2 * t ? 1.0 : 0.0, 0.0);          // identity padding
            if (!(g < w8 && 2 * t + 1 < w8)) c1 = zmk(g == 2 * t + 1 ? 1.0 : 0.0, 0.0);
            inv8_regs(c0, c1, w8, nk, bad_row);
            z2* Dn = cur ? sm.Dk[0] : sm.Dk[1];
            Dn[g * DLD + 2 * t] = c0;
            Dn[g * DLD + 2 * t + 1] = c1;
        }
        {
            const int w0 = nk < m ? 1 : 0;   // warp 0 is busy with the next pivot
            const int stp = nw - w0, sq = stp / mt, sr = stp - sq * mt;
            int it = (w - w0) / mt, jt = (w - w0) - it * mt;   // tile (it, jt) = the warp's linear index, stepped
            for (int tile = w - w0; tile < mt * mt; tile += stp) {   // without a division per tile
                if (tile < 0) break;                                  // (warp 0 when it forms the next pivot)
                const int i0 = it * 8, j0 = jt * 8;
                if (!(i0 == kb || j0 == kb || (i0 == nk && j0 == nk))) {
                    if (full) {
                        z2 c0, c1;
                        trail8<true>(S, ld, kb, i0, j0, c0, c1);
                    } else {
                        trail_tile(S, ld, m, kb, kw, i0, j0);
                    }
                }
                it += sq;
                jt += sr;
                if (jt >= mt) {
                    jt -= mt;
                    it++;
                }
            }
        }
        __syncthreads();
        CPROF(4);
        // ---- column panel: S[i, K] = -S[i, K] Dk (i not in K); S[K, K] = Dk
        for (int strip = w; strip < mt; strip += nw)
            if (strip * 8 != kb) {
                if (full) col8(S, ld, kb, Dk, strip * 8);
                else col_strip(S, ld, m, kb, kw, Dk, strip * 8);
            }
        if (tid < 64) {
            const int r = tid >> 3, c = tid & 7;
            if (r < kw && c < kw) S[sx(kb + r, kb + c, ld)] = Dk[r * DLD + c];
        }
        __syncthreads();
        CPROF(5);
        cur ^= 1;
    }
}

__device__ void store_block(const SubDesc& d, int i, FactorSmem sm, z2* __restrict__ dinv)
{
    const int m = d.m, ld = lds_of(m);
    z2* out = dinv + d.fac_off + (long long)i * m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int c = e / m, r = e % m;   // column-major: coalesced stores
        out[e] = sm.S[sx(r, c, ld)];
    }
    __syncthreads();
}

// S, then Dk[0] (GB x DLD: the 32-wide path's pivot inverse; the 8-wide path uses its first 8 rows), Dk[1] (8 x DLD:
// the 8-wide path's next pivot inverse), the pivot-row buffer (2 x GB)
__device__ FactorSmem carve(unsigned char* base, int m)
{
    FactorSmem sm;
    sm.S = reinterpret_cast<z2*>(base);
    sm.Dk[0] = sm.S + (size_t)((m + 7) / 8 * 8) * lds_of(m);   // S has m rounded up to a multiple of 8 rows
    sm.Dk[1] = sm.Dk[0] + GB * DLD;
    sm.rowbuf = sm.Dk[1] + 8 * DLD;
    return sm;
}

__device__ void report(int* err, int bad_row, int sub, int block)
{
    if (threadIdx.x == 0 && bad_row >= 0 && atomicCAS(err, 0, 1) == 0) {
        err[1] = sub;
        err[2] = block;
        err[3] = bad_row;
    }
}

// blockIdx.x = 2 * sub + chain (0 bottom: i = 0 .. tw-1, 1 top: i = nb-1 .. tw+1)
template <bool P8>
__global__ void __launch_bounds__(FT) k_factor_chains(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                      z2* __restrict__ dinv, int* err)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int sub = blockIdx.x >> 1, chain = blockIdx.x & 1;
    const SubDesc d = desc[sub];
    FactorSmem sm = carve(smem, d.m);
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    // zero S once: the rows / columns padding m up to a multiple of 8 stay zero through every elimination
    for (int e = threadIdx.x; e < (d.m + 7) / 8 * 8 * lds_of(d.m); e += blockDim.x) sm.S[e] = zmk(0, 0);
    __syncthreads();
#ifdef HELM_FACTOR_PROF
    // development aid (-DHELM_FACTOR_PROF): clock64 cycles per phase as thread 0 sees them (waits included), printed
    // by CTA 0: build, pivot inverse (alone), row panel, -, trailing (+ the 8-wide path's next pivot inverse), column
    // panel, store
    long long prl[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tnow = clock64();
    long long* cpr = threadIdx.x == 0 ? prl : nullptr;
    long long* ctp = &tnow;
#endif
    const int i0 = chain == 0 ? 0 : d.nb - 1, i1 = chain == 0 ? d.tw : d.tw, step = chain == 0 ? 1 : -1;
    for (int i = i0; i != i1; i += step) {
        build_block(d, i, chain, stc, dinv, sm);
        CPROF(0);
        if (P8)
            gj_panels8(d.m, sm, &bad CPROF_PASS);
        else
            gj_blocked(d.m, sm, &bad CPROF_PASS);
        store_block(d, i, sm, dinv);
        CPROF(6);
        report(err, bad, sub, i);
    }
#ifdef HELM_FACTOR_PROF
    // CTA 0 (a corner subdomain) and the bottom chain of the middle subdomain (an interior one)
    if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == 2 * (gridDim.x / 4 + 32)))
        printf("CPROF cta %d m %d blocks %d build %lld pinv %lld row %lld nextpiv %lld trail %lld col %lld store %lld\n",
               blockIdx.x, d.m, d.tw, prl[0], prl[1], prl[2], prl[3], prl[4], prl[5], prl[6]);
#endif
}

template <bool P8>
__global__ void __launch_bounds__(FT) k_factor_twist(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                     z2* __restrict__ dinv, int* err)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int sub = blockIdx.x;
    const SubDesc d = desc[sub];
    FactorSmem sm = carve(smem, d.m);
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    // zero S once: the rows / columns padding m up to a multiple of 8 stay zero through every elimination
    for (int e = threadIdx.x; e < (d.m + 7) / 8 * 8 * lds_of(d.m); e += blockDim.x) sm.S[e] = zmk(0, 0);
    __syncthreads();
    build_block(d, d.tw, 2, stc, dinv, sm);
#ifdef HELM_FACTOR_PROF
    long long* cpr = nullptr;
    long long* ctp = nullptr;
#endif
    if (P8)
        gj_panels8(d.m, sm, &bad CPROF_PASS);
    else
        gj_blocked(d.m, sm, &bad CPROF_PASS);
    store_block(d, d.tw, sm, dinv);
    report(err, bad, sub, d.tw);
}

// ------------------------------------------------------------------------------------------------------------------
// Large blocks (m > M_SMEM: the paper's ~300-node-wide subdomains, D21).  The Schur complement no longer fits in
// shared memory.  One thread-block cluster of BC CTAs owns a chain; each block is formed and inverted IN PLACE in
// its factor slot (column-major, L2-resident) by blocked, unpivoted Gauss-Jordan with panels K of GB columns:
//   Dk = A[K,K]^-1                   every CTA, redundantly, in shared memory
//   A[K,j] = Dk A[K,j] (j not in K), A[K,K] = Dk          columns split over the CTAs
//   -- cluster barrier --
//   A[i,j] -= A[i,K] A[K,j] (i, j not in K);  A[i,K] = -A[i,K] Dk (i not in K)   row slabs per CTA, A[i,K] staged
//   -- cluster barrier --
// Unpivoted (D12): on the bottom chain the elimination order is the oracle's no-pivot band LU (O7), so the pivots are
// the oracle's; a zero pivot is reported like the shared-memory path.
// ------------------------------------------------------------------------------------------------------------------
constexpr int BCMAX = 16;  // CTAs per cluster (one cluster per chain): 8, or 16 when there are few chains
constexpr int BT = 256;    // threads per CTA
constexpr int CW = 128;    // columns of the row panel staged per chunk of the trailing update

__host__ __device__ __forceinline__ int big_rows(int m, int bc) { return (m + bc - 1) / bc; }

// 16-byte asynchronous global -> shared copy (LDGSTS): the staging loops issue all their loads before waiting
__device__ __forceinline__ void cp_async16(z2* dst, const z2* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void cluster_sync_all()
{
    __threadfence();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ int cluster_rank()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}

#ifdef HELM_FACTOR_PROF
// development aid (-DHELM_FACTOR_PROF via HELM_NVCC_EXTRA): clock64 cycles per phase of big_block, printed by the
// first CTA of the first cluster
#define FPROF_N 8
#define FPROF_T(k) do { const long long t_ = clock64(); if (prof) prof[k] += t_ - tprev; tprev = t_; } while (0)
#else
#define FPROF_T(k) do { } while (0)
#endif

// one block of a chain, formed then inverted in place (column-major in its factor slot)
__device__ void big_block(const SubDesc& d, int i, int mode, const z2* __restrict__ stc, z2* __restrict__ dinv, int rk,
                          int bc, z2* Dk, z2* Aik, z2* AK, int* bad
#ifdef HELM_FACTOR_PROF
                          , long long* prof
#endif
                          )
{
#ifdef HELM_FACTOR_PROF
    long long tprev = clock64();
#endif
    const int m = d.m, tid = threadIdx.x;
    z2* A = dinv + d.fac_off + (long long)i * m * m;
    const int c0 = (int)(((long long)m * rk) / bc), c1 = (int)(((long long)m * (rk + 1)) / bc);
    // Schur complement, columns split over the cluster
    for (long long e = (long long)c0 * m + tid; e < (long long)c1 * m; e += BT) {
        const int b = (int)(e / m), a = (int)(e - (long long)b * m);
        A[e] = schur_entry(d, i, mode, stc, dinv, a, b);
    }
    FPROF_T(0);
    cluster_sync_all();
    FPROF_T(1);
    const int R = big_rows(m, bc), r0 = rk * R, r1 = min(m, r0 + R), nr = max(0, r1 - r0);
    for (int kb = 0; kb < m; kb += GB) {
        const int kw = min(GB, m - kb);
        // ---- Dk = A[K,K]^-1 (every CTA, one warp)
        for (int e = tid; e < kw * kw; e += BT) {
            const int c = e / kw, r = e - c * kw;
            Dk[r * DLD + c] = A[(long long)(kb + c) * m + kb + r];
        }
        __syncthreads();
        FPROF_T(2);
        if (tid < GJW * 32) warp_gj8(Dk, Dk + GB * DLD, kw, kb, bad);
        __syncthreads();
        FPROF_T(3);
        // ---- row panel: A[K,j] = Dk A[K,j] for this CTA's columns on the tensor cores; one warp per 8-column strip
        //      loads the strip's old 32 x 8 block as B fragments first, then writes its four row tiles (in place)
        {
            const int lane = tid & 31, g = lane >> 2, t = lane & 3;
            for (int j0 = c0 + (tid >> 5) * 8; j0 < c1; j0 += (BT >> 5) * 8) {
                const int col = j0 + g;
                z2 bf[GB / 4];
#pragma unroll
                for (int s4 = 0; s4 < GB / 4; s4++) {
                    const int q = 4 * s4 + t;
                    bf[s4] = (q < kw && col < c1) ? A[(long long)col * m + kb + q] : zmk(0, 0);
                }
#pragma unroll
                for (int rt = 0; rt < GB / 8; rt++) {
                    if (8 * rt >= kw) break;
                    z2 v0 = zmk(0, 0), v1 = zmk(0, 0);
#pragma unroll
                    for (int s4 = 0; s4 < GB / 4; s4++) {
                        if (4 * s4 >= kw) break;
                        const int r = 8 * rt + g, q = 4 * s4 + t;
                        const z2 a = (r < kw && q < kw) ? Dk[r * DLD + q] : zmk(0, 0);
                        dmma(v0.x, v1.x, a.x, bf[s4].x);   // C += A B
                        dmma(v0.x, v1.x, -a.y, bf[s4].y);
                        dmma(v0.y, v1.y, a.x, bf[s4].y);
                        dmma(v0.y, v1.y, a.y, bf[s4].x);
                    }
                    // outputs: row 8 rt + g of K, columns j0 + 2t, j0 + 2t + 1
                    const int r = 8 * rt + g;
                    for (int u = 0; u < 2; u++) {
                        const int cc = j0 + 2 * t + u;
                        if (r >= kw || cc >= c1) continue;
                        const bool kcol = cc >= kb && cc < kb + kw;
                        A[(long long)cc * m + kb + r] = kcol ? Dk[r * DLD + (cc - kb)] : (u ? v1 : v0);
                    }
                }
            }
        }
        FPROF_T(4);
        cluster_sync_all();
        FPROF_T(1);
        // ---- trailing update of this CTA's row slab [r0, r1): A[i,K] staged in Aik (once), the row panel A[K, :] in
        //      chunks of CW columns in AK (the K columns stage Dk: A[i,K] = -A[i,K] Dk is the same product with C = 0).
        //      A warp owns 8 slab rows x 32 columns: its A fragments are loaded once and feed four independent 8 x 8
        //      accumulators (four DMMA chains in flight).
        for (int e = tid; e < nr * kw; e += BT) {
            const int q = e / nr, ii = e - q * nr;
            cp_async16(&Aik[ii * DLD + q], &A[(long long)(kb + q) * m + r0 + ii]);
        }
        const int nrt = (nr + 7) / 8, lane = tid & 31, g = lane >> 2, t = lane & 3;
        for (int cs = 0; cs < m; cs += CW) {
            const int cw = min(CW, m - cs), ncg = (cw + 31) / 32;
            for (int e = tid; e < cw * kw; e += BT) {
                const int jj = e / kw, q = e - jj * kw, j = cs + jj;
                if (j >= kb && j < kb + kw) AK[q * CW + jj] = Dk[q * DLD + (j - kb)];
                else cp_async16(&AK[q * CW + jj], &A[(long long)j * m + kb + q]);
            }
            cp_async_wait_all();
            __syncthreads();
            FPROF_T(5);
            for (int u = tid >> 5; u < nrt * ncg; u += BT >> 5) {
                const int i0 = (u / ncg) * 8, jg = (u % ncg) * 32;
                const int r = i0 + g, row = r0 + r;
                const bool rok = r < nr && !(row >= kb && row < kb + kw);   // rows of the panel are final already
                z2 af[GB / 4];
#pragma unroll
                for (int s4 = 0; s4 < GB / 4; s4++) {
                    const int q = 4 * s4 + t;
                    af[s4] = (r < nr && q < kw) ? Aik[r * DLD + q] : zmk(0, 0);
                }
                z2 c0[4], c1[4];
#pragma unroll
                for (int ct = 0; ct < 4; ct++) {
                    const int jA = jg + 8 * ct + 2 * t, jB = jA + 1;   // chunk-relative output columns
                    const int gA = cs + jA, gB = cs + jB;
                    const bool kA = gA >= kb && gA < kb + kw, kB = gB >= kb && gB < kb + kw;
                    c0[ct] = (rok && jA < cw && !kA) ? A[(long long)gA * m + row] : zmk(0, 0);
                    c1[ct] = (rok && jB < cw && !kB) ? A[(long long)gB * m + row] : zmk(0, 0);
                }
#pragma unroll
                for (int s4 = 0; s4 < GB / 4; s4++) {
                    if (4 * s4 >= kw) break;
                    const z2 a = af[s4];
                    const int q = 4 * s4 + t;
#pragma unroll
                    for (int ct = 0; ct < 4; ct++) {
                        const int jj = jg + 8 * ct + g;
                        const z2 b = (q < kw && jj < cw) ? AK[q * CW + jj] : zmk(0, 0);
                        dmma(c0[ct].x, c1[ct].x, -a.x, b.x);   // C -= A B
                        dmma(c0[ct].x, c1[ct].x, a.y, b.y);
                        dmma(c0[ct].y, c1[ct].y, -a.x, b.y);
                        dmma(c0[ct].y, c1[ct].y, -a.y, b.x);
                    }
                }
                if (rok) {
#pragma unroll
                    for (int ct = 0; ct < 4; ct++) {
                        const int jA = jg + 8 * ct + 2 * t, jB = jA + 1;
                        if (jA < cw) A[(long long)(cs + jA) * m + row] = c0[ct];
                        if (jB < cw) A[(long long)(cs + jB) * m + row] = c1[ct];
                    }
                }
            }
            __syncthreads();
            FPROF_T(6);
        }
        cluster_sync_all();
        FPROF_T(1);
    }
}

// blockIdx.x / bc = chain: mode 0 -> 2 * sub + (0 bottom | 1 top), mode 2 -> sub (twist block)
__global__ void __launch_bounds__(BT, 2) k_factor_big(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                   z2* __restrict__ dinv, int* err, int mode, int bc)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int rk = cluster_rank(), chain = blockIdx.x / bc;
    const int sub = mode == 0 ? chain >> 1 : chain;
    const SubDesc d = desc[sub];
    z2* Dk = reinterpret_cast<z2*>(smem);
    z2* AK = Dk + GB * DLD;
    z2* Aik = AK + GB * CW;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    __syncthreads();
#ifdef HELM_FACTOR_PROF
    long long pr[FPROF_N] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long* prof = threadIdx.x == 0 ? pr : nullptr;
#define PROFARG , prof
#else
#define PROFARG
#endif
    if (mode == 2) {
        big_block(d, d.tw, 2, stc, dinv, rk, bc, Dk, Aik, AK, &bad PROFARG);
        report(err, bad, sub, d.tw);
    } else if ((chain & 1) == 0) {
        for (int i = 0; i < d.tw; i++) {
            big_block(d, i, 0, stc, dinv, rk, bc, Dk, Aik, AK, &bad PROFARG);
            report(err, bad, sub, i);
        }
    } else {
        for (int i = d.nb - 1; i > d.tw; i--) {
            big_block(d, i, 1, stc, dinv, rk, bc, Dk, Aik, AK, &bad PROFARG);
            report(err, bad, sub, i);
        }
    }
#ifdef HELM_FACTOR_PROF
    if (threadIdx.x == 0 && blockIdx.x == 0 && mode == 0)
        printf("FPROF schur %lld clusterbar %lld dkload %lld gj %lld rowpanel %lld akstage %lld tiles %lld\n", pr[0], pr[1],
               pr[2], pr[3], pr[4], pr[5], pr[6]);
#endif
}

// Dk, AK (its first 2 x GB entries double as warp_gj8's pivot-row buffer: not live at the same time), Aik
int big_smem_bytes(int m_max, int bc) { return (int)sizeof(z2) * (GB * DLD + GB * CW + big_rows(m_max, bc) * DLD); }

}  // namespace

int factor_smem_bytes(int m_max)
{
    return (int)(sizeof(z2) * ((size_t)((m_max + 7) / 8 * 8) * lds_of(m_max) + GB * DLD + 8 * DLD + 2 * GB));
}

// 8-wide panels with the register-resident pivot inverse (gj_panels8) unless HELM_FACTOR_PANEL=32
bool factor_panels8()
{
    const char* e = getenv("HELM_FACTOR_PANEL");
    return !(e && atoi(e) == 32);
}

void launch_factor(const SubDesc* d_desc, const SubDesc* /*h_desc*/, int nsub, int m_max, const z2* stencil, z2* dinv,
                   int* d_err, cudaStream_t s)
{
    if (m_max > M_SMEM) {
        // clusters of bc CTAs: all chains, then all twist blocks; 16-CTA clusters when 8-CTA ones leave SMs idle.
        // Otherwise 6 or 8 CTAs per chain, whichever the model (waves of resident CTAs) x (per-block cost ~ 29 + m/bc
        // rows) says is shorter -- calibrated at k = 1200 (128 chains: bc 6 0.77 s, 8 0.86 s) and k = 600 (32 chains:
        // bc 8 0.21 s, 6 0.23 s).  HELM_FACTOR_BC overrides.
        int nsm = 148, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int bc = 2 * nsub * 8 < nsm ? BCMAX : 8;
        if (bc == 8) {
            double best = 1e300;
            for (int cand : {8, 6}) {
                const int sm = big_smem_bytes(m_max, cand);
                raise_smem_attr((const void*)k_factor_big, sm);
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_factor_big, BT, sm);
                if (occ < 1) continue;
                const long long slots = (long long)nsm * occ, ctas = 2LL * nsub * cand;
                const double est = (double)((ctas + slots - 1) / slots) * (29.0 + (double)m_max / cand);
                if (est < best) {
                    best = est;
                    bc = cand;
                }
            }
            cudaGetLastError();
        }
        if (const char* e = getenv("HELM_FACTOR_BC")) bc = atoi(e);
        const int smem = big_smem_bytes(m_max, bc);
        raise_smem_attr((const void*)k_factor_big, smem, bc > 8);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = bc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(BT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(2 * nsub * bc);
        cudaLaunchKernelEx(&cfg, k_factor_big, d_desc, stencil, dinv, d_err, 0, bc);
        cfg.gridDim = dim3(nsub * bc);
        cudaLaunchKernelEx(&cfg, k_factor_big, d_desc, stencil, dinv, d_err, 2, bc);
        return;
    }
    const int smem = factor_smem_bytes(m_max);
    auto go = [&](auto kc, auto kt) {
        raise_smem_attr((const void*)kc, smem);
        raise_smem_attr((const void*)kt, smem);
        kc<<<2 * nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
        kt<<<nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
    };
    if (factor_panels8())
        go(k_factor_chains<true>, k_factor_twist<true>);
    else
        go(k_factor_chains<false>, k_factor_twist<false>);
}

// ------------------------------------------------------------------------------------------------------------------
// Measurement aid: FP64 peak of this GPU (the factorisation's roofline denominator; MEASURED_PEAKS.json holds only
// HBM and bf16).  mode 0: DMMA (mma.sync m8n8k4 f64, 8 independent accumulator tiles per warp); mode 1: DFMA
// (8 independent FMA chains per thread).  Grid = SMs x 4 CTAs of 256 threads, `iters` loop trips, timed with events.
// ------------------------------------------------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) k_fp64_probe(int mode, int iters, double* sink)
{
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * blockIdx.x;
    double c[16];
#pragma unroll
    for (int q = 0; q < 16; q++) c[q] = 1e-3 * q;
    if (mode == 0) {
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int q = 0; q < 8; q++) dmma(c[2 * q], c[2 * q + 1], a, b);
        }
    } else {
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int q = 0; q < 16; q++) c[q] = fma(a, c[q], b);
        }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 16; q++) s += c[q];
    if (s == 1234.5678) *sink = s;   // keeps the chains live
}
}  // namespace

extern "C" int helm_probe_fp64_tflops(int mode, double* tflops)
{
    if (!tflops || mode < 0 || mode > 1) return HELM_EINVAL;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return HELM_ENOMEM;
    }
    const int grid = 4 * nsm, block = 256, iters = mode == 0 ? 4096 : 8192;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64_probe<<<grid, block>>>(mode, iters / 8, sink);   // warm-up
    cudaEventRecord(e0);
    k_fp64_probe<<<grid, block>>>(mode, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return HELM_ECUDA;
    // DMMA: 8 tiles x 8x8x4 MACs per warp per trip; DFMA: 16 FMAs per thread per trip
    const double flops = mode == 0 ? 2.0 * 8 * 256 * (double)iters * (grid * block / 32)
                                   : 2.0 * 16 * (double)iters * grid * block;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return HELM_OK;
}
