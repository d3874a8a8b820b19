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
// The two chains run in separate CTAs; a second launch forms the twist blocks.
#include <stdio.h>

#include "internal.cuh"

namespace {

constexpr int FT = 512;  // threads per factor CTA

__host__ __device__ __forceinline__ int lds_of(int m) { return ((m + 7) / 8) * 8 + 1; }  // 16B-words, = 1 mod 8

// -(L_i W U_{i-1})(a,b) with W = P_{i-1}^-1 (column-major in global memory)
__device__ __forceinline__ z2 term_below(const z2* __restrict__ W, int m, int a, int b, const z2* Lrow_S,
                                         const z2* Lrow_SW, const z2* Urow_N, const z2* Urow_NE)
{
    // (L W U)[a][b] = sum_{c in {a, a-1}} sum_{d in {b, b-1}} L[a][c] W[c][d] U[d][b]
    // L[a][a] = S_i(a), L[a][a-1] = SW_i(a); U[b][b] = N_{i-1}(b), U[b-1][b] = NE_{i-1}(b-1)
    const z2 un = Urow_N[b];
    const z2 une = b > 0 ? Urow_NE[b - 1] : zmk(0, 0);
    z2 r0 = zmul(W[(long long)b * m + a], un);
    if (b > 0) r0 = zadd(r0, zmul(W[(long long)(b - 1) * m + a], une));
    z2 acc = zmul(Lrow_S[a], r0);
    if (a > 0) {
        z2 r1 = zmul(W[(long long)b * m + a - 1], un);
        if (b > 0) r1 = zadd(r1, zmul(W[(long long)(b - 1) * m + a - 1], une));
        acc = zadd(acc, zmul(Lrow_SW[a], r1));
    }
    return acc;
}

// (U_i W L_{i+1})(a,b) with W = Q_{i+1}^-1
__device__ __forceinline__ z2 term_above(const z2* __restrict__ W, int m, int a, int b, const z2* Urow_N,
                                         const z2* Urow_NE, const z2* Lrow_S, const z2* Lrow_SW)
{
    // U[a][a] = N_i(a), U[a][a+1] = NE_i(a); L[b][b] = S_{i+1}(b), L[b+1][b] = SW_{i+1}(b+1)
    const z2 ls = Lrow_S[b];
    const z2 lsw = b + 1 < m ? Lrow_SW[b + 1] : zmk(0, 0);
    z2 r0 = zmul(W[(long long)b * m + a], ls);
    if (b + 1 < m) r0 = zadd(r0, zmul(W[(long long)(b + 1) * m + a], lsw));
    z2 acc = zmul(Urow_N[a], r0);
    if (a + 1 < m) {
        z2 r1 = zmul(W[(long long)b * m + a + 1], ls);
        if (b + 1 < m) r1 = zadd(r1, zmul(W[(long long)(b + 1) * m + a + 1], lsw));
        acc = zadd(acc, zmul(Urow_NE[a], r1));
    }
    return acc;
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
    const z2* rowi = stc + d.stc_off + (long long)i * 7 * m;
    const z2* C = rowi + SL_C * m;
    const z2* E = rowi + SL_E * m;
    const z2* Wc = rowi + SL_W * m;
    const bool below = (mode == 0 || mode == 2) && i > 0;
    const bool above = (mode == 1 || mode == 2) && i < d.nb - 1;
    const z2* Wb = below ? dinv + d.fac_off + (long long)(i - 1) * m * m : nullptr;
    const z2* Wa = above ? dinv + d.fac_off + (long long)(i + 1) * m * m : nullptr;
    const z2* rowm = below ? stc + d.stc_off + (long long)(i - 1) * 7 * m : nullptr;
    const z2* rowp = above ? stc + d.stc_off + (long long)(i + 1) * 7 * m : nullptr;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int a = e / m, b = e % m;
        z2 v = zmk(0, 0);
        if (b == a) v = C[a];
        else if (b == a + 1) v = E[a];
        else if (b == a - 1) v = Wc[a];
        if (below) v = zsub(v, term_below(Wb, m, a, b, rowi + SL_S * m, rowi + SL_SW * m, rowm + SL_N * m, rowm + SL_NE * m));
        if (above) v = zsub(v, term_above(Wa, m, a, b, rowi + SL_N * m, rowi + SL_NE * m, rowp + SL_S * m, rowp + SL_SW * m));
        sm.S[a * ld + b] = v;
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

}  // namespace

int factor_smem_bytes(int m_max)
{
    return (int)(sizeof(z2) * ((size_t)m_max * lds_of(m_max) + m_max) + sizeof(int) * (m_max + 4));
}

void launch_factor(const SubDesc* d_desc, const SubDesc* /*h_desc*/, int nsub, int m_max, const z2* stencil, z2* dinv,
                   int* d_err, cudaStream_t s)
{
    const int smem = factor_smem_bytes(m_max);
    cudaFuncSetAttribute(k_factor_chains, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_factor_twist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_factor_chains<<<2 * nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
    k_factor_twist<<<nsub, FT, smem, s>>>(d_desc, stencil, dinv, d_err);
}
