// factor.cu -- K3: setup factorisation of every local operator A_j (exact local solves, P:143-147 A_j^-1).
//
// A_j is block tridiagonal in its local x-fastest numbering (7-point SW->NE stencil, D1): block row i
// holds T_i (tridiagonal: C, E, W), L_i = A_{i,i-1} (S on the diagonal, SW below it) and
// U_i = A_{i,i+1} (N on the diagonal, NE above it).  We use a TWISTED block LU:
//   bottom chain  P_0 = T_0,        P_i = T_i - L_i P_{i-1}^-1 U_{i-1},        i = 1 .. tw-1
//   top chain     Q_{nb-1} = T_{nb-1}, Q_i = T_i - U_i Q_{i+1}^-1 L_{i+1},      i = nb-2 .. tw+1
//   twist         Z = T_tw - L_tw P_{tw-1}^-1 U_{tw-1} - U_tw Q_{tw+1}^-1 L_{tw+1}
// and store the explicit inverse of each block (P_i^-1, Z^-1, Q_i^-1) in block slot i, column-major.
// Each inverse is formed by Gauss-Jordan elimination with partial (row) pivoting in shared memory.
// The two chains run in separate CTAs; a second launch forms the twist blocks.  Blocks wider than M_SMEM use
// thread-block clusters and blocked Gauss-Jordan in global memory (k_factor_big).  The 9-point Q1 stencil (D18)
// adds a third diagonal to L_i (SE) and U_i (NW).
#include <stdio.h>

#include "internal.cuh"

namespace {

constexpr int FT = 512;  // threads per factor CTA

__host__ __device__ __forceinline__ int lds_of(int m) { return ((m + 7) / 8) * 8 + 1; }  // 16B-words, = 1 mod 8

// Couplings of block row i as m x m matrices (7-point P1: two diagonals; 9-point Q1: three):
//   L_i[a][a] = S_i(a), L_i[a][a-1] = SW_i(a), L_i[a][a+1] = SE_i(a)          (A_{i,i-1})
//   U_i[a][a] = N_i(a), U_i[a][a+1] = NE_i(a), U_i[a][a-1] = NW_i(a)          (A_{i,i+1})
// Wl(c, d) reads W = the inverse stored column-major in global memory.
struct Cpl { const z2 *d, *lo, *hi; };   // diagonal, sub-diagonal (entry [a][a-1]) and super ([a][a+1]) vectors

// (L_i W U_{i-1})(a,b) = sum_c L[a][c] sum_d W[c][d] U[d][b];  U[d][b]: d = b N(b), d = b-1 NE(b-1), d = b+1 NW(b+1)
__device__ __forceinline__ z2 term_below(const z2* __restrict__ W, int m, int a, int b, Cpl L, Cpl U)
{
    z2 ud[3];          // U[b-1][b], U[b][b], U[b+1][b]
    ud[0] = (b > 0) ? U.hi[b - 1] : zmk(0, 0);
    ud[1] = U.d[b];
    ud[2] = (U.lo && b + 1 < m) ? U.lo[b + 1] : zmk(0, 0);
    z2 acc = zmk(0, 0);
    for (int dc = -1; dc <= 1; dc++) {
        const int c = a + dc;
        if (c < 0 || c >= m) continue;
        const z2 l = dc == 0 ? L.d[a] : (dc < 0 ? L.lo[a] : (L.hi ? L.hi[a] : zmk(0, 0)));
        if (l.x == 0.0 && l.y == 0.0) continue;
        z2 r = zmk(0, 0);
        for (int dd = -1; dd <= 1; dd++) {
            const int d = b + dd;
            if (d < 0 || d >= m) continue;
            r = zadd(r, zmul(W[(long long)d * m + c], ud[dd + 1]));
        }
        acc = zadd(acc, zmul(l, r));
    }
    return acc;
}

// (U_i W L_{i+1})(a,b) = sum_c U[a][c] sum_d W[c][d] L[d][b];  L[d][b]: d = b S(b), d = b+1 SW(b+1), d = b-1 SE(b-1)
__device__ __forceinline__ z2 term_above(const z2* __restrict__ W, int m, int a, int b, Cpl U, Cpl L)
{
    z2 ld[3];          // L[b-1][b], L[b][b], L[b+1][b]
    ld[0] = (L.hi && b > 0) ? L.hi[b - 1] : zmk(0, 0);
    ld[1] = L.d[b];
    ld[2] = (b + 1 < m) ? L.lo[b + 1] : zmk(0, 0);
    z2 acc = zmk(0, 0);
    for (int dc = -1; dc <= 1; dc++) {
        const int c = a + dc;
        if (c < 0 || c >= m) continue;
        const z2 u = dc == 0 ? U.d[a] : (dc > 0 ? U.hi[a] : (U.lo ? U.lo[a] : zmk(0, 0)));
        if (u.x == 0.0 && u.y == 0.0) continue;
        z2 r = zmk(0, 0);
        for (int dd = -1; dd <= 1; dd++) {
            const int d = b + dd;
            if (d < 0 || d >= m) continue;
            r = zadd(r, zmul(W[(long long)d * m + c], ld[dd + 1]));
        }
        acc = zadd(acc, zmul(u, r));
    }
    return acc;
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
    z2* S;      // [m][lds] row-major
    z2* fcol;   // [m]
    int* perm;  // [m]
    int* piv;   // [1]
};

// mode: 0 bottom chain block, 1 top chain block, 2 twist block
__device__ void build_block(const SubDesc& d, int i, int mode, const z2* __restrict__ stc, const z2* __restrict__ dinv,
                            FactorSmem sm)
{
    const int m = d.m, ld = lds_of(m);
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int a = e / m, b = e % m;
        sm.S[a * ld + b] = schur_entry(d, i, mode, stc, dinv, a, b);
    }
    __syncthreads();
}

// In-place Gauss-Jordan inversion with partial row pivoting of S (m x m, row-major, stride ld).
// Returns (through *err) the first zero pivot row.
__device__ void gj_invert(int m, FactorSmem sm, int* bad_row)
{
    const int ld = lds_of(m);
    z2* S = sm.S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int k = 0; k < m; k++) {
        if (warp == 0) {
            double best = -1.0;
            int bi = k;
            for (int r = k + lane; r < m; r += 32) {
                const double v = zabs2(S[r * ld + k]);
                if (v > best) { best = v; bi = r; }
            }
            for (int off = 16; off; off >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (lane == 0) {
                *sm.piv = bi;
                sm.perm[k] = bi;
                if (best == 0.0 && *bad_row < 0) *bad_row = k;
            }
        }
        __syncthreads();
        const int p = *sm.piv;
        if (p != k)
            for (int c = tid; c < m; c += blockDim.x) {
                const z2 t = S[k * ld + c];
                S[k * ld + c] = S[p * ld + c];
                S[p * ld + c] = t;
            }
        __syncthreads();
        const z2 pv = S[k * ld + k];
        const z2 inv = (zabs2(pv) > 0.0) ? zinv(pv) : zmk(0, 0);
        // save column k (multipliers) and zero it; scale row k; pivot entry -> 1/pivot
        for (int r = tid; r < m; r += blockDim.x) {
            if (r != k) {
                sm.fcol[r] = S[r * ld + k];
                S[r * ld + k] = zmk(0, 0);
            }
        }
        for (int c = tid; c < m; c += blockDim.x)
            if (c != k) S[k * ld + c] = zmul(S[k * ld + c], inv);
        __syncthreads();
        if (tid == 0) S[k * ld + k] = inv;
        __syncthreads();
        // rank-1 update of every row but k
        for (int e = tid; e < m * m; e += blockDim.x) {
            const int r = e / m, c = e % m;
            if (r == k) continue;
            const z2 f = sm.fcol[r];
            const z2 s = S[k * ld + c];
            z2 v = S[r * ld + c];
            v.x = fma(-f.x, s.x, v.x);
            v.x = fma(f.y, s.y, v.x);
            v.y = fma(-f.x, s.y, v.y);
            v.y = fma(-f.y, s.x, v.y);
            S[r * ld + c] = v;
        }
        __syncthreads();
    }
    // undo the row interchanges as column interchanges, last first
    for (int k = m - 1; k >= 0; k--) {
        const int p = sm.perm[k];
        if (p != k)
            for (int r = tid; r < m; r += blockDim.x) {
                const z2 t = S[r * ld + k];
                S[r * ld + k] = S[r * ld + p];
                S[r * ld + p] = t;
            }
        __syncthreads();
    }
}

__device__ void store_block(const SubDesc& d, int i, FactorSmem sm, z2* __restrict__ dinv)
{
    const int m = d.m, ld = lds_of(m);
    z2* out = dinv + d.fac_off + (long long)i * m * m;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int c = e / m, r = e % m;   // column-major: coalesced stores
        out[e] = sm.S[r * ld + c];
    }
    __syncthreads();
}

__device__ FactorSmem carve(unsigned char* base, int m)
{
    FactorSmem sm;
    sm.S = reinterpret_cast<z2*>(base);
    sm.fcol = sm.S + (size_t)m * lds_of(m);
    sm.perm = reinterpret_cast<int*>(sm.fcol + m);
    sm.piv = sm.perm + m;
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
__global__ void __launch_bounds__(FT) k_factor_chains(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                      z2* __restrict__ dinv, int* err)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int sub = blockIdx.x >> 1, chain = blockIdx.x & 1;
    const SubDesc d = desc[sub];
    FactorSmem sm = carve(smem, d.m);
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    __syncthreads();
    if (chain == 0) {
        for (int i = 0; i < d.tw; i++) {
            build_block(d, i, 0, stc, dinv, sm);
            gj_invert(d.m, sm, &bad);
            store_block(d, i, sm, dinv);
            report(err, bad, sub, i);
        }
    } else {
        for (int i = d.nb - 1; i > d.tw; i--) {
            build_block(d, i, 1, stc, dinv, sm);
            gj_invert(d.m, sm, &bad);
            store_block(d, i, sm, dinv);
            report(err, bad, sub, i);
        }
    }
}

__global__ void __launch_bounds__(FT) k_factor_twist(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                     z2* __restrict__ dinv, int* err)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int sub = blockIdx.x;
    const SubDesc d = desc[sub];
    FactorSmem sm = carve(smem, d.m);
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    __syncthreads();
    build_block(d, d.tw, 2, stc, dinv, sm);
    gj_invert(d.m, sm, &bad);
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
// Unpivoted elimination in natural order meets exactly the pivots of the oracle's no-pivot band LU (O7, D12), so it
// breaks down only where the oracle does; a zero pivot is reported like the shared-memory path.
// ------------------------------------------------------------------------------------------------------------------
constexpr int BC = 8;      // CTAs per cluster (one cluster per chain)
constexpr int BT = 256;    // threads per CTA
constexpr int GB = 32;     // panel width
constexpr int JT = 32;     // column tile of the trailing update
constexpr int DLD = GB + 1;

__host__ __device__ __forceinline__ int big_rows(int m) { return (m + BC - 1) / BC; }

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

// acc -= a * b
__device__ __forceinline__ void zfms(z2& acc, z2 a, z2 b)
{
    acc.x = fma(-a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(-a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

// Dk (kw x kw, row-major, stride DLD) <- Dk^-1 by unpivoted in-place Gauss-Jordan
__device__ void small_gj(z2* Dk, int kw, int kb, int* bad)
{
    const int tid = threadIdx.x;
    for (int p = 0; p < kw; p++) {
        const z2 pv = Dk[p * DLD + p];
        const bool zero = pv.x == 0.0 && pv.y == 0.0;
        if (zero && tid == 0 && *bad < 0) *bad = kb + p;
        const z2 inv = zero ? zmk(0, 0) : zinv(pv);
        if (tid < kw && tid != p) Dk[p * DLD + tid] = zmul(Dk[p * DLD + tid], inv);   // scale row p
        __syncthreads();
        for (int e = tid; e < kw * kw; e += blockDim.x) {                          // rank-1 update off row / col p
            const int r = e / kw, c = e - r * kw;
            if (r == p || c == p) continue;
            zfms(Dk[r * DLD + c], Dk[r * DLD + p], Dk[p * DLD + c]);
        }
        __syncthreads();
        if (tid < kw && tid != p) {                                                 // column p
            const z2 f = Dk[tid * DLD + p];
            Dk[tid * DLD + p] = zmk(0, 0);
            zfms(Dk[tid * DLD + p], f, inv);
        }
        if (tid == 0) Dk[p * DLD + p] = inv;
        __syncthreads();
    }
}

// one block of a chain, formed then inverted in place
__device__ void big_block(const SubDesc& d, int i, int mode, const z2* __restrict__ stc, z2* __restrict__ dinv, int rk,
                          z2* Dk, z2* Aik, z2* AKj, int* bad)
{
    const int m = d.m, tid = threadIdx.x;
    z2* A = dinv + d.fac_off + (long long)i * m * m;
    {   // Schur complement, columns split over the cluster
        const int c0 = (int)(((long long)m * rk) / BC), c1 = (int)(((long long)m * (rk + 1)) / BC);
        for (long long e = (long long)c0 * m + tid; e < (long long)c1 * m; e += BT) {
            const int b = (int)(e / m), a = (int)(e - (long long)b * m);
            A[e] = schur_entry(d, i, mode, stc, dinv, a, b);
        }
    }
    cluster_sync_all();
    const int R = big_rows(m), r0 = rk * R, r1 = min(m, r0 + R), nr = max(0, r1 - r0);
    for (int kb = 0; kb < m; kb += GB) {
        const int kw = min(GB, m - kb);
        // ---- Dk = A[K,K]^-1
        for (int e = tid; e < kw * kw; e += BT) {
            const int c = e / kw, r = e - c * kw;
            Dk[r * DLD + c] = A[(long long)(kb + c) * m + kb + r];
        }
        __syncthreads();
        small_gj(Dk, kw, kb, bad);
        // ---- row panel: A[K,j] = Dk A[K,j] for this CTA's columns (tiles of BT / GB columns)
        {
            const int c0 = (int)(((long long)m * rk) / BC), c1 = (int)(((long long)m * (rk + 1)) / BC);
            const int per = BT / GB;
            for (int jt = c0; jt < c1; jt += per) {
                const int jj = tid / GB, r = tid - jj * GB, j = jt + jj;
                const bool act = j < c1 && r < kw;
                if (act) AKj[jj * GB + r] = A[(long long)j * m + kb + r];
                __syncthreads();
                if (act) {
                    z2 v;
                    if (j >= kb && j < kb + kw) {
                        v = Dk[r * DLD + (j - kb)];
                    } else {
                        v = zmk(0, 0);
                        for (int q = 0; q < kw; q++) zfma(v, Dk[r * DLD + q], AKj[jj * GB + q]);
                    }
                    A[(long long)j * m + kb + r] = v;
                }
                __syncthreads();
            }
        }
        cluster_sync_all();
        // ---- trailing update of this CTA's row slab [r0, r1)
        for (int e = tid; e < nr * kw; e += BT) {
            const int q = e / nr, ii = e - q * nr;
            Aik[ii * DLD + q] = A[(long long)(kb + q) * m + r0 + ii];
        }
        __syncthreads();
        for (int jt = 0; jt < m; jt += JT) {
            const int jw = min(JT, m - jt);
            for (int e = tid; e < jw * kw; e += BT) {
                const int jj = e / kw, q = e - jj * kw;
                AKj[q * JT + jj] = A[(long long)(jt + jj) * m + kb + q];
            }
            __syncthreads();
            for (int e = tid; e < nr * jw; e += BT) {
                const int jj = e / nr, ii = e - jj * nr;
                const int row = r0 + ii, j = jt + jj;
                if (row >= kb && row < kb + kw) continue;
                z2* dst = A + (long long)j * m + row;
                z2 v;
                if (j >= kb && j < kb + kw) {
                    v = zmk(0, 0);
                    for (int q = 0; q < kw; q++) zfms(v, Aik[ii * DLD + q], Dk[q * DLD + (j - kb)]);
                } else {
                    v = *dst;
                    for (int q = 0; q < kw; q++) zfms(v, Aik[ii * DLD + q], AKj[q * JT + jj]);
                }
                *dst = v;
            }
            __syncthreads();
        }
        cluster_sync_all();
    }
}

// blockIdx.x / BC = chain: mode 0 -> 2 * sub + (0 bottom | 1 top), mode 2 -> sub (twist block)
__global__ void __launch_bounds__(BT) k_factor_big(const SubDesc* __restrict__ desc, const z2* __restrict__ stc,
                                                   z2* __restrict__ dinv, int* err, int mode)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const int rk = cluster_rank(), chain = blockIdx.x / BC;
    const int sub = mode == 0 ? chain >> 1 : chain;
    const SubDesc d = desc[sub];
    z2* Dk = reinterpret_cast<z2*>(smem);
    z2* AKj = Dk + GB * DLD;
    z2* Aik = AKj + GB * JT;
    __shared__ int bad;
    if (threadIdx.x == 0) bad = -1;
    __syncthreads();
    if (mode == 2) {
        big_block(d, d.tw, 2, stc, dinv, rk, Dk, Aik, AKj, &bad);
        report(err, bad, sub, d.tw);
    } else if ((chain & 1) == 0) {
        for (int i = 0; i < d.tw; i++) {
            big_block(d, i, 0, stc, dinv, rk, Dk, Aik, AKj, &bad);
            report(err, bad, sub, i);
        }
    } else {
        for (int i = d.nb - 1; i > d.tw; i--) {
            big_block(d, i, 1, stc, dinv, rk, Dk, Aik, AKj, &bad);
            report(err, bad, sub, i);
        }
    }
}

int big_smem_bytes(int m_max) { return (int)sizeof(z2) * (GB * DLD + GB * JT + big_rows(m_max) * DLD); }

}  // namespace

int factor_smem_bytes(int m_max)
{
    return (int)(sizeof(z2) * ((size_t)m_max * lds_of(m_max) + m_max) + sizeof(int) * (m_max + 4));
}

void launch_factor(const SubDesc* d_desc, const SubDesc* /*h_desc*/, int nsub, int m_max, const z2* stencil, z2* dinv,
                   int* d_err, cudaStream_t s)
{
    if (m_max > M_SMEM) {
        // clusters of BC CTAs: all chains, then all twist blocks
        const int smem = big_smem_bytes(m_max);
        cudaFuncSetAttribute(k_factor_big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = BC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(BT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(2 * nsub * BC);
        cudaLaunchKernelEx(&cfg, k_factor_big, d_desc, stencil, dinv, d_err, 0);
        cfg.gridDim = dim3(nsub * BC);
        cudaLaunchKernelEx(&cfg, k_factor_big, d_desc, stencil, dinv, d_err, 2);
        return;
    }
    const int smem = factor_smem_bytes(m_max);
    cudaFuncSetAttribute(k_factor_chains, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_factor_twist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_factor_chains<<<2 * nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
    k_factor_twist<<<nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
}
