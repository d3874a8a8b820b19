// krylov.cu -- K5 SpMV (7-point P1 / 9-point Q1 stencil) and the GMRES vector kernels (K6-K8): multi-dot, multi-axpy
// with fused norm, normalisation, basis combination.  All reductions are deterministic: a fixed row
// partition per CTA, warp-shuffle trees inside a CTA, and a single-CTA pass over the CTA partials in
// index order (D15).  No floating-point atomics.
#include <algorithm>

#include "internal.cuh"

namespace {

constexpr int KT = 256;          // threads per CTA
constexpr int NVMAX = 64;        // max vectors in one multi-dot / multi-axpy (restart + 1 <= 64)

__device__ __forceinline__ z2 warp_sum(z2 v)
{
    for (int off = 16; off; off >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
    }
    return v;
}
__device__ __forceinline__ double warp_sum(double v)
{
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

__device__ __forceinline__ void chunk_of(long long n, long long& r0, long long& r1)
{
    const long long per = ((n + gridDim.x - 1) / gridDim.x + 31) / 32 * 32;
    r0 = (long long)blockIdx.x * per;
    r1 = r0 + per < n ? r0 + per : n;
}

// CTA-wide deterministic sum of a per-thread double -> thread 0
__device__ double block_sum(double v, double* sh)
{
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += sh[w];
    __syncthreads();
    return s;
}

__constant__ int c_dx[9] = { 0, 1, -1, 0, 0, 1, -1, -1, 1 };
__constant__ int c_dy[9] = { 0, 0, 0, 1, -1, 1, -1, 1, -1 };

// Row r of the owned rectangle (x-fastest): y = sum_s A[s][r] x(neighbour_s), NS = 7 (P1) or 9 (Q1) slots; x is
// read from a buffer covering the owned rectangle plus whatever ghost frame the caller provides (origin xi0,
// xj0; stride).
template <int NS>
__device__ __forceinline__ z2 stencil_row(const z2* __restrict__ A7, const z2* __restrict__ x, long long r,
                                          const StencilGeom& G)
{
    const long long n = (long long)G.nx * G.ny;
    // rows of one rank fit in 32 bits (< 2^31 nodes): 32-bit division
    const unsigned ru = (unsigned)r;
    const int lj = (int)(ru / (unsigned)G.nx);
    const int i = G.i0 + (int)(ru - (unsigned)lj * (unsigned)G.nx), j = G.j0 + lj;
    z2 acc = zmk(0, 0);
    if (i >= G.ci0 && i < G.ci1 && j >= G.cj0 && j < G.cj1) {   // constant interior stencil (all neighbours free)
        const z2* xc = x + (i - G.xi0) + G.xstride * (j - G.xj0);
#pragma unroll
        for (int s = 0; s < NS; s++) zfma(acc, G.c7[s], __ldg(xc + c_dx[s] + G.xstride * c_dy[s]));
        return acc;
    }
#pragma unroll
    for (int s = 0; s < NS; s++) {
        const int qi = i + c_dx[s], qj = j + c_dy[s];
        if (qi >= 1 && qi <= G.nf && qj >= 1 && qj <= G.nf)
            zfma(acc, __ldg(A7 + s * n + r), __ldg(x + (qi - G.xi0) + G.xstride * (qj - G.xj0)));
    }
    return acc;
}

// 2-D launch: blockIdx.y strides over rows j, x-threads over i (no 64-bit division per row)
template <int NS>
__global__ void __launch_bounds__(KT) k_spmv(const z2* __restrict__ A7, const z2* __restrict__ x, z2* __restrict__ y,
                                             StencilGeom G, int a0, int a1, int b0, int b1)
{
    // rows li in [a0, nx - a1), lj in [b0, ny - b1) of the owned rectangle (all of it: a0 = a1 = b0 = b1 = 0)
    const int li = a0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (li >= G.nx - a1) return;
    for (int lj = b0 + blockIdx.y; lj < G.ny - b1; lj += gridDim.y) {
        const long long r = li + (long long)G.nx * lj;
        y[r] = stencil_row<NS>(A7, x, r, G);
    }
}

// the complement: the frame of width a0 / a1 / b0 / b1 around that interior (the rows whose stencil reads ghost nodes)
template <int NS>
__global__ void __launch_bounds__(KT) k_spmv_frame(const z2* __restrict__ A7, const z2* __restrict__ x,
                                                   z2* __restrict__ y, StencilGeom G, int a0, int a1, int b0, int b1)
{
    const long long nrow = (long long)(b0 + b1) * G.nx;            // bottom and top rows, full width
    const int hin = G.ny - b0 - b1;                                   // rows of the side columns
    const long long n = nrow + (long long)(a0 + a1) * max(hin, 0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        int li, lj;
        if (e < nrow) {
            const int q = (int)(e / G.nx);
            li = (int)(e - (long long)q * G.nx);
            lj = q < b0 ? q : G.ny - b1 + (q - b0);
        } else {
            const long long f = e - nrow;
            const int c = (int)(f / hin);
            lj = b0 + (int)(f - (long long)c * hin);
            li = c < a0 ? c : G.nx - a1 + (c - a0);
        }
        const long long r = li + (long long)G.nx * lj;
        y[r] = stencil_row<NS>(A7, x, r, G);
    }
}

// r = b - A x, partial[blk] = ||r||^2 over the CTA's rows
template <int NS>
__global__ void __launch_bounds__(KT) k_residual(const z2* __restrict__ A7, const z2* __restrict__ x,
                                                 const z2* __restrict__ b, z2* __restrict__ r, StencilGeom G,
                                                 double* __restrict__ partial)
{
    __shared__ double sh[KT / 32];
    const long long n = (long long)G.nx * G.ny;
    long long r0, r1;
    chunk_of(n, r0, r1);
    double s = 0.0;
    for (long long e = r0 + threadIdx.x; e < r1; e += blockDim.x) {
        const z2 v = zsub(__ldg(b + e), stencil_row<NS>(A7, x, e, G));
        r[e] = v;
        s += zabs2(v);
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// dst(rect) = src(rect): strided 2-D copy between vectors with different origins / strides (halo pack,
// unpack, owned -> ghost-framed buffer)
// add: dst(rect) += src(rect) (unpack of the additive reverse exchange of the ramp PoU)
__global__ void __launch_bounds__(KT) k_copy_rect(const z2* __restrict__ src, int si0, int sj0, long long sstride,
                                                  z2* __restrict__ dst, int di0, int dj0, long long dstride,
                                                  int i0, int i1, int j0, int j1, int add)
{
    const int w = i1 - i0;
    const long long n = (long long)w * (j1 - j0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int i = i0 + (int)(e % w), j = j0 + (int)(e / w);
        z2* d = dst + (i - di0) + dstride * (j - dj0);
        const z2 v = src[(i - si0) + sstride * (j - sj0)];
        *d = add ? zadd(*d, v) : v;
    }
}

// Section 3(i): the interface band.  bx[i] / by[j] flag the node indices whose stencil crosses a block
// boundary along that axis (i = s_p - 1, s_p).  k_band_mask zeroes every entry of the owned vector outside the band;
// k_pack_rects moves the band part of a ghost-framed buffer through a contiguous message buffer, rectangle by
// rectangle (a canonical decomposition of the message rectangle into band sub-rectangles, offsets = prefix areas).
__global__ void __launch_bounds__(KT) k_band_mask(z2* __restrict__ v, int i0, int i1, int j0, int j1,
                                                 const unsigned char* __restrict__ bx, const unsigned char* __restrict__ by)
{
    const int w = i1 - i0;
    const long long n = (long long)w * (j1 - j0);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int i = i0 + (int)(e % w), j = j0 + (int)(e / w);
        if (!bx[i] && !by[j]) v[e] = zmk(0, 0);
    }
}

__global__ void __launch_bounds__(KT) k_pack_rects(z2* __restrict__ ext, int e_i0, int e_j0, long long stride,
                                                  const int4* __restrict__ rects, const long long* __restrict__ off,
                                                  z2* __restrict__ buf, int unpack)
{
    const int4 r = rects[blockIdx.y];
    const int w = r.y - r.x;
    const long long n = (long long)w * (r.w - r.z);
    z2* b = buf + off[blockIdx.y];
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int i = r.x + (int)(e % w), j = r.z + (int)(e / w);
        z2* x = ext + (i - e_i0) + stride * (j - e_j0);
        if (unpack)
            *x = b[e];
        else
            b[e] = *x;
    }
}

// sum of squares (no sqrt) -> *sq; used before a cross-rank allreduce
__global__ void k_reduce_sq(const double* __restrict__ partial, int nblk, double* sq)
{
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[b];
    s = warp_sum(s);
    if (lane == 0) *sq = s;
}

__global__ void k_finish_norm(const double* sq, z2* out_slot, double* out_norm)
{
    const double nrm = sqrt(*sq);
    if (out_slot) *out_slot = zmk(nrm, 0.0);
    if (out_norm) *out_norm = nrm;
}

// out[v] = a[v] + b[v]
__global__ void k_zadd(const z2* __restrict__ a, const z2* __restrict__ b, z2* __restrict__ out, int nv)
{
    for (int v = threadIdx.x; v < nv; v += blockDim.x) out[v] = zadd(a[v], b[v]);
}

// partial[blk][v] = sum_{e in blk} conj(V_v[e]) w[e],  v < nv
template <int R>
__global__ void __launch_bounds__(KT) k_multidot(const z2* __restrict__ V, long long ldv, int nv,
                                                 const z2* __restrict__ w, long long n, z2* __restrict__ partial)
{
    __shared__ z2 acc[KT / 32][NVMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int v = lane; v < NVMAX; v += 32) acc[warp][v] = zmk(0, 0);
    __syncwarp();
    long long r0, r1;
    chunk_of(n, r0, r1);
    for (long long base = r0; base < r1; base += (long long)KT * R) {
        z2 wv[R];
        long long e[R];
#pragma unroll
        for (int q = 0; q < R; q++) {
            e[q] = base + q * KT + threadIdx.x;
            wv[q] = e[q] < r1 ? __ldg(w + e[q]) : zmk(0, 0);
        }
        for (int v = 0; v < nv; v++) {
            const z2* Vv = V + v * ldv;
            z2 s = zmk(0, 0);
#pragma unroll
            for (int q = 0; q < R; q++)
                if (e[q] < r1) zfma_conj(s, __ldg(Vv + e[q]), wv[q]);
            s = warp_sum(s);
            if (lane == 0) acc[warp][v] = zadd(acc[warp][v], s);
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        z2 s = zmk(0, 0);
        for (int q = 0; q < KT / 32; q++) s = zadd(s, acc[q][v]);
        partial[(long long)blockIdx.x * NVMAX + v] = s;
    }
}

// Fused second CGS pass: w -= sum_v h[v] V_v and partial[blk][v] = sum_e conj(V_v[e]) w_new[e] in one sweep
// (V is read from HBM once; the second touch of each tile hits L1/L2).
template <int R>
__global__ void __launch_bounds__(KT) k_axpy_dot(const z2* __restrict__ V, long long ldv, int nv,
                                                 const z2* __restrict__ h, z2* __restrict__ w, long long n,
                                                 z2* __restrict__ partial)
{
    __shared__ z2 hs[NVMAX];
    __shared__ z2 acc[KT / 32][NVMAX];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int v = threadIdx.x; v < nv; v += blockDim.x) hs[v] = h[v];
    for (int v = lane; v < NVMAX; v += 32) acc[warp][v] = zmk(0, 0);
    __syncthreads();
    long long r0, r1;
    chunk_of(n, r0, r1);
    for (long long base = r0; base < r1; base += (long long)KT * R) {
        z2 wv[R];
        long long e[R];
#pragma unroll
        for (int q = 0; q < R; q++) {
            e[q] = base + q * KT + threadIdx.x;
            wv[q] = e[q] < r1 ? w[e[q]] : zmk(0, 0);
        }
        for (int v = 0; v < nv; v++) {
            const z2 hv = zmk(-hs[v].x, -hs[v].y);
            const z2* Vv = V + v * ldv;
#pragma unroll
            for (int q = 0; q < R; q++)
                if (e[q] < r1) zfma(wv[q], hv, __ldg(Vv + e[q]));
        }
#pragma unroll
        for (int q = 0; q < R; q++)
            if (e[q] < r1) w[e[q]] = wv[q];
        for (int v = 0; v < nv; v++) {
            const z2* Vv = V + v * ldv;
            z2 s = zmk(0, 0);
#pragma unroll
            for (int q = 0; q < R; q++)
                if (e[q] < r1) zfma_conj(s, __ldg(Vv + e[q]), wv[q]);
            s = warp_sum(s);
            if (lane == 0) acc[warp][v] = zadd(acc[warp][v], s);
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nv; v += blockDim.x) {
        z2 s = zmk(0, 0);
        for (int q = 0; q < KT / 32; q++) s = zadd(s, acc[q][v]);
        partial[(long long)blockIdx.x * NVMAX + v] = s;
    }
}

// w -= sum_v h[v] V_v ; partial[blk] = ||w_new||^2
__global__ void __launch_bounds__(KT) k_multiaxpy(const z2* __restrict__ V, long long ldv, int nv,
                                                  const z2* __restrict__ h, z2* __restrict__ w, long long n,
                                                  double* __restrict__ partial)
{
    __shared__ z2 hs[NVMAX];
    __shared__ double sh[KT / 32];
    for (int v = threadIdx.x; v < nv; v += blockDim.x) hs[v] = h[v];
    __syncthreads();
    long long r0, r1;
    chunk_of(n, r0, r1);
    double s = 0.0;
    for (long long e = r0 + threadIdx.x; e < r1; e += blockDim.x) {
        z2 acc = w[e];
        for (int v = 0; v < nv; v++) {
            const z2 hv = hs[v];
            zfma(acc, zmk(-hv.x, -hv.y), __ldg(V + v * ldv + e));
        }
        w[e] = acc;
        s += zabs2(acc);
    }
    if (partial) {
        s = block_sum(s, sh);
        if (threadIdx.x == 0) partial[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------------------------------------------------
// DCGS2: CGS2 with the re-orthogonalisation of v_j delayed into the projection sweep of step j + 1.
// Step j holds V_j = [v_0 .. v_{j-1}] (final), the candidate u_j (V slot j, projected once) and w_j = A B^-1 u_j.
//   sweep 1  (k_multidot2)  a = V_j^H u_j, alpha = u_j^H u_j, b = V_j^H w_j, c = u_j^H w_j          (reads V once)
//   coeffs   (k_dcgs2_coef) nu = sqrt(alpha - |a|^2); column j-1 of H += a, H(j, j-1) = nu (final);
//                           p = H(0:j, 0:j) a, q = nu a_{j-1}; column j of H (pending): h = (b - p) / nu,
//                           h_jj = ((c - a^H b) / nu - q) / nu
//   sweep 2  (k_dcgs2_update) v_j = (u_j - V_j a) / nu;  u_{j+1} = w_j / nu - (sigma / nu) u_j - V_j e,
//                           sigma = q / nu + h_jj, e = p / nu + h - a sigma / nu                   (reads V once)
// which is CGS2's v_j and u_{j+1} = A B^-1 v_j - V_{j+1} h in exact arithmetic (A B^-1 V_j = V_{j+1} H(0:j+1, 0:j)).

// partial[blk][q] = sum_e conj(V_q[e]) u[e] (q < nv), partial[blk][NVMAX + q] = sum_e conj(V_q[e]) w[e], with a
// transposing warp reduction: per batch of 8 basis vectors each lane holds 32 partial values
// (8 vectors x {u, w} x {re, im}); five exchange-and-add levels (16 + 8 + 4 + 2 + 1 = 31 shuffles, instead of 5 per
// value) leave lane L with the warp's sum of value L.  Fixed order: deterministic.
template <int R>
__global__ void __launch_bounds__(KT) k_multidot2(const z2* __restrict__ V, long long ldv, int nv,
                                                   const z2* __restrict__ u, const z2* __restrict__ w, long long n,
                                                   z2* __restrict__ partial)
{
    constexpr int VB = 8;
    __shared__ double acc[KT / 32][2 * NVMAX * 2];   // [warp][(v | NVMAX for w) * 2 + re/im]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int q = lane; q < 4 * NVMAX; q += 32) acc[warp][q] = 0.0;
    __syncwarp();
    long long r0, r1;
    chunk_of(n, r0, r1);
    for (long long base = r0; base < r1; base += (long long)KT * R) {
        z2 uv[R], wv[R];
        long long e[R];
#pragma unroll
        for (int q = 0; q < R; q++) {
            e[q] = base + q * KT + threadIdx.x;
            uv[q] = e[q] < r1 ? __ldg(u + e[q]) : zmk(0, 0);
            wv[q] = e[q] < r1 ? __ldg(w + e[q]) : zmk(0, 0);
        }
        for (int v0 = 0; v0 < nv; v0 += VB) {
            double t[32];
#pragma unroll
            for (int b = 0; b < VB; b++) {
                z2 su = zmk(0, 0), sw = zmk(0, 0);
#pragma unroll
                for (int q = 0; q < R; q++) {
                    const z2 x = (v0 + b < nv && e[q] < r1) ? __ldg(V + (v0 + b) * ldv + e[q]) : zmk(0, 0);
                    zfma_conj(su, x, uv[q]);
                    zfma_conj(sw, x, wv[q]);
                }
                t[4 * b + 0] = su.x;
                t[4 * b + 1] = su.y;
                t[4 * b + 2] = sw.x;
                t[4 * b + 3] = sw.y;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const bool hi = lane & o;
#pragma unroll
                for (int k = 0; k < o; k++) {
                    const double send = hi ? t[k] : t[k + o];
                    const double keep = hi ? t[k + o] : t[k];
                    t[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            // lane L holds value L = 4 b + {0: Re u, 1: Im u, 2: Re w, 3: Im w}
            const int b = lane >> 2, part = lane & 3;
            if (v0 + b < nv) {
                const int slot = ((part >> 1) ? NVMAX : 0) + v0 + b;
                acc[warp][2 * slot + (part & 1)] += t[0];
            }
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < 2 * NVMAX; v += blockDim.x) {
        if ((v & (NVMAX - 1)) >= nv) continue;
        z2 s = zmk(0, 0);
        for (int q = 0; q < KT / 32; q++) s = zadd(s, zmk(acc[q][2 * v], acc[q][2 * v + 1]));
        partial[(long long)blockIdx.x * 2 * NVMAX + v] = s;
    }
}

// One warp.  d: the reduced sweep-1 sums (d[q] = V_q^H u_j, d[j + 1 + q] = V_q^H w_j, q <= j; one allreduce).  H: device Hessenberg,
// column-major with leading dimension NVMAX + 1.  Writes the sweep-2 coefficients ca (= a / nu), ce (= e) and
// sc = {1 / nu, sigma / nu}, and for the host: out[0 .. j] = final column j - 1 (rows 0 .. j), out[NVMAX .. NVMAX + j]
// = pending column j, out[2 NVMAX] = (nu, 0).
__global__ void k_dcgs2_coef(const z2* __restrict__ d, int j, z2* __restrict__ H, z2* __restrict__ ca,
                             z2* __restrict__ ce, double* __restrict__ sc, z2* __restrict__ out)
{
    constexpr int LD = NVMAX + 1;
    __shared__ z2 as[NVMAX];
    const int lane = threadIdx.x;
    double na = 0.0;
    z2 ab = zmk(0, 0);
    for (int i = lane; i < j; i += 32) {
        const z2 a = d[i];
        as[i] = a;
        na += zabs2(a);
        zfma_conj(ab, a, d[j + 1 + i]);
    }
    na = warp_sum(na);
    ab = warp_sum(ab);
    const double alpha = d[j].x;
    const z2 c = d[2 * j + 1];
    const double nu2 = alpha - na;
    const double nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
    const double inv = nu > 0.0 ? 1.0 / nu : 0.0;
    if (j >= 1) {   // finish column j - 1
        for (int i = lane; i < j; i += 32) H[(j - 1) * LD + i] = zadd(H[(j - 1) * LD + i], as[i]);
        if (lane == 0) H[(j - 1) * LD + j] = zmk(nu, 0.0);
    }
    for (int i = lane; i < j; i += 32) out[2 * NVMAX + 2 + i] = as[i];   // u_j = nu v_j + V_j a: column j of R
    __syncwarp();
    const z2 q = j >= 1 ? zscale(as[j - 1], nu) : zmk(0, 0);
    const z2 hjj = zscale(zsub(zscale(zsub(c, ab), inv), q), inv);
    const z2 sigma = zadd(zscale(q, inv), hjj);
    const z2 sinv = zscale(sigma, inv);
    for (int i = lane; i < j; i += 32) {
        z2 p = zmk(0, 0);   // (H(0:j, 0:j) a)_i, columns k >= i - 1 only (Hessenberg), increasing k
        for (int k = i > 0 ? i - 1 : 0; k < j; k++) zfma(p, H[k * LD + i], as[k]);
        const z2 h = zscale(zsub(d[j + 1 + i], p), inv);
        H[j * LD + i] = h;
        out[NVMAX + i] = h;
        const z2 e = zsub(zadd(zscale(p, inv), h), zmul(as[i], sinv));
        ce[i] = e;
        ca[i] = zscale(as[i], inv);
    }
    for (int i = lane; i <= j && j >= 1; i += 32) out[i] = H[(j - 1) * LD + i];
    if (lane == 0) {
        H[j * LD + j] = hjj;
        out[NVMAX + j] = hjj;
        out[2 * NVMAX] = zmk(nu, 0.0);
        sc[0] = inv;
        sc[1] = sigma.x * inv;
        sc[2] = sigma.y * inv;
    }
}

// Close column j with the re-orthogonalisation of u_{j+1} (cycle end): d[q] = V_q^H u_{j+1}, q <= j + 1.
// H(0:j, j) += a, H(j+1, j) = nu; out[0 .. j+1] = the final column.
__global__ void k_dcgs2_close(const z2* __restrict__ d, int j, z2* __restrict__ H, z2* __restrict__ out)
{
    constexpr int LD = NVMAX + 1;
    const int lane = threadIdx.x;
    double na = 0.0;
    for (int i = lane; i <= j; i += 32) na += zabs2(d[i]);
    na = warp_sum(na);
    const double nu2 = d[j + 1].x - na;
    const double nu = nu2 > 0.0 ? sqrt(nu2) : 0.0;
    for (int i = lane; i <= j; i += 32) {
        const z2 h = zadd(H[j * LD + i], d[i]);
        H[j * LD + i] = h;
        out[i] = h;
    }
    if (lane == 0) {
        H[j * LD + j + 1] = zmk(nu, 0.0);
        out[j + 1] = zmk(nu, 0.0);
    }
}

// Sweep 2: slot j <- v_j = u_j / nu - sum_q ca_q V_q;  slot j + 1 <- u_{j+1} = w / nu - (sigma / nu) u_j - sum_q ce_q V_q
// (q < j); partial[blk] = ||u_{j+1}||^2 over the block.  V slot j is read and written by the same thread.
__global__ void __launch_bounds__(KT) k_dcgs2_update(z2* V, long long ldv, int j, const z2* __restrict__ w,
                                                     const z2* __restrict__ ca, const z2* __restrict__ ce,
                                                     const double* __restrict__ sc, long long n,
                                                     double* __restrict__ partial)
{
    __shared__ z2 cs[2 * NVMAX];
    __shared__ double sh[KT / 32];
    for (int v = threadIdx.x; v < j; v += blockDim.x) {
        cs[v] = ca[v];
        cs[NVMAX + v] = ce[v];
    }
    __syncthreads();
    const double inv = sc[0];
    const z2 sinv = zmk(sc[1], sc[2]);
    z2* uj = V + j * ldv;
    z2* un = uj + ldv;
    long long r0, r1;
    chunk_of(n, r0, r1);
    double s = 0.0;
    // the coefficients are read from shared memory ahead of each basis load and the loop is unrolled by 4, so four
    // basis loads are in flight per thread (c3, 105 steps: 54.0 -> 49.5 ms; two rows per thread 53.2; the same loop
    // with the shared-memory reads inside the FMAs 75 ms)
    for (long long e = r0 + threadIdx.x; e < r1; e += blockDim.x) {
        z2 av = zmk(0, 0), ev = zmk(0, 0);
#pragma unroll 4
        for (int v = 0; v < j; v++) {
            const z2 ca_v = cs[v], ce_v = cs[NVMAX + v];
            const z2 x = __ldg(V + v * ldv + e);
            zfma(av, ca_v, x);
            zfma(ev, ce_v, x);
        }
        const z2 u = uj[e];
        const z2 vj = zsub(zscale(u, inv), av);
        z2 nx = zscale(__ldg(w + e), inv);
        nx = zsub(nx, zmul(sinv, u));
        nx = zsub(nx, ev);
        uj[e] = vj;
        un[e] = nx;
        s += zabs2(nx);
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out[q] = sum_blk partial[blk][v]; out_plus[q] = add[q] + out[q] (if given); one CTA, index order.  Values
// v = q < nv, and (off2 > 0) a second group v = off2 + (q - nv), packed behind the first: out[nv .. 2 nv).
__global__ void k_reduce_z(const z2* __restrict__ partial, int nblk, int nv, z2* __restrict__ out,
                           z2* __restrict__ out_plus, const z2* __restrict__ add, int stride, int off2)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nval = off2 ? 2 * nv : nv;
    for (int q = warp; q < nval; q += blockDim.x >> 5) {
        const int v = q < nv ? q : off2 + (q - nv);
        z2 s = zmk(0, 0);
        for (int b = lane; b < nblk; b += 32) s = zadd(s, partial[(long long)b * stride + v]);
        s = warp_sum(s);
        if (lane == 0) {
            out[q] = s;
            if (out_plus) out_plus[q] = zadd(add[q], s);
        }
    }
}

// norm = sqrt(sum partial); out_slot (complex) = (norm, 0)
__global__ void k_reduce_norm(const double* __restrict__ partial, int nblk, z2* out_slot, double* out_norm)
{
    const int lane = threadIdx.x;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[b];
    s = warp_sum(s);
    if (lane == 0) {
        const double nrm = sqrt(s);
        if (out_slot) *out_slot = zmk(nrm, 0.0);
        if (out_norm) *out_norm = nrm;
    }
}

__global__ void __launch_bounds__(KT) k_scale(const z2* __restrict__ w, const double* __restrict__ norm,
                                              z2* __restrict__ v, long long n)
{
    const double nr = *norm;
    const double inv = nr != 0.0 ? 1.0 / nr : 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
        v[e] = zscale(w[e], inv);
}

// t = sum_v y[v] V_v
__global__ void __launch_bounds__(KT) k_combine(const z2* __restrict__ V, long long ldv, int nv,
                                                const z2* __restrict__ y, z2* __restrict__ t, long long n)
{
    __shared__ z2 ys[NVMAX];
    for (int v = threadIdx.x; v < nv; v += blockDim.x) ys[v] = y[v];
    __syncthreads();
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        z2 acc = zmk(0, 0);
        for (int v = 0; v < nv; v++) zfma(acc, ys[v], __ldg(V + v * ldv + e));
        t[e] = acc;
    }
}

__global__ void __launch_bounds__(KT) k_axpy(z2* __restrict__ x, const z2* __restrict__ z, long long n)
{
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
        x[e] = zadd(x[e], z[e]);
}

__global__ void __launch_bounds__(KT) k_copy(z2* __restrict__ d, const z2* __restrict__ s, long long n)
{
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
        d[e] = s[e];
}

__global__ void __launch_bounds__(KT) k_norm_partial(const z2* __restrict__ x, long long n, double* __restrict__ partial)
{
    __shared__ double sh[KT / 32];
    long long r0, r1;
    chunk_of(n, r0, r1);
    double s = 0.0;
    for (long long e = r0 + threadIdx.x; e < r1; e += blockDim.x) s += zabs2(x[e]);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

struct RankPtrs { const double* p[16]; };
// out[i] = sum_r p[r][i] in rank order (loopback allreduce)
__global__ void k_sum_ranks(RankPtrs ptrs, int nranks, int count, double* __restrict__ out)
{
    for (int i = threadIdx.x; i < count; i += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; r++) s += ptrs.p[r][i];
        out[i] = s;
    }
}

int ew_grid(long long n)
{
    long long b = (n + KT - 1) / KT;
    if (b > 148LL * 8) b = 148LL * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

void launch_spmv(const z2* A7, const z2* x, z2* y, const StencilGeom& G, cudaStream_t s, int a0, int a1, int b0,
                 int b1)
{
    // each CTA walks several grid rows j (x rows j-1, j, j+1 stay in L1 between iterations) instead of one
    const int nx = G.nx - a0 - a1, ny = G.ny - b0 - b1;
    if (nx <= 0 || ny <= 0) return;
    const int gx = (nx + KT - 1) / KT;
    int gy = std::max(1, 148 * 64 / gx);
    if (gy > ny) gy = ny;
    if (G.ns == 9) k_spmv<9><<<dim3(gx, gy), KT, 0, s>>>(A7, x, y, G, a0, a1, b0, b1);
    else k_spmv<7><<<dim3(gx, gy), KT, 0, s>>>(A7, x, y, G, a0, a1, b0, b1);
}
void launch_spmv_frame(const z2* A7, const z2* x, z2* y, const StencilGeom& G, int a0, int a1, int b0, int b1,
                       cudaStream_t s)
{
    const long long n = (long long)(b0 + b1) * G.nx + (long long)(a0 + a1) * std::max(G.ny - b0 - b1, 0);
    if (n <= 0) return;
    if (G.ns == 9) k_spmv_frame<9><<<ew_grid(n), KT, 0, s>>>(A7, x, y, G, a0, a1, b0, b1);
    else k_spmv_frame<7><<<ew_grid(n), KT, 0, s>>>(A7, x, y, G, a0, a1, b0, b1);
}
void launch_residual(const z2* A7, const z2* x, const z2* b, z2* r, const StencilGeom& G, double* partial, int nblk,
                     cudaStream_t s)
{
    if (G.ns == 9) k_residual<9><<<nblk, KT, 0, s>>>(A7, x, b, r, G, partial);
    else k_residual<7><<<nblk, KT, 0, s>>>(A7, x, b, r, G, partial);
}
void launch_copy_rect(const z2* src, int si0, int sj0, long long sstride, z2* dst, int di0, int dj0, long long dstride,
                      int i0, int i1, int j0, int j1, cudaStream_t s, bool add)
{
    const long long n = (long long)(i1 - i0) * (j1 - j0);
    if (n <= 0) return;
    k_copy_rect<<<ew_grid(n), KT, 0, s>>>(src, si0, sj0, sstride, dst, di0, dj0, dstride, i0, i1, j0, j1, add ? 1 : 0);
}
void launch_band_mask(z2* v, int i0, int i1, int j0, int j1, const unsigned char* bx, const unsigned char* by,
                      cudaStream_t s)
{
    const long long n = (long long)(i1 - i0) * (j1 - j0);
    if (n <= 0) return;
    k_band_mask<<<ew_grid(n), KT, 0, s>>>(v, i0, i1, j0, j1, bx, by);
}
void launch_pack_rects(z2* ext, int e_i0, int e_j0, long long stride, const int4* rects, const long long* off,
                       int nrects, long long max_area, z2* buf, bool unpack, cudaStream_t s)
{
    if (nrects <= 0 || max_area <= 0) return;
    const int gx = (int)std::min<long long>((max_area + KT - 1) / KT, 64);
    k_pack_rects<<<dim3(gx, nrects), KT, 0, s>>>(ext, e_i0, e_j0, stride, rects, off, buf, unpack ? 1 : 0);
}
void launch_reduce_sq(const double* partial, int nblk, double* sq, cudaStream_t s)
{
    k_reduce_sq<<<1, 32, 0, s>>>(partial, nblk, sq);
}
void launch_finish_norm(const double* sq, z2* out_slot, double* out_norm, cudaStream_t s)
{
    k_finish_norm<<<1, 1, 0, s>>>(sq, out_slot, out_norm);
}
void launch_zadd(const z2* a, const z2* b, z2* out, int nv, cudaStream_t s) { k_zadd<<<1, 64, 0, s>>>(a, b, out, nv); }
void launch_multidot(const z2* V, long long ldv, int nv, const z2* w, long long n, z2* partial, int nblk,
                     cudaStream_t s)
{
    k_multidot<4><<<nblk, KT, 0, s>>>(V, ldv, nv, w, n, partial);
}
void launch_axpy_dot(const z2* V, long long ldv, int nv, const z2* h, z2* w, long long n, z2* partial, int nblk,
                     cudaStream_t s)
{
    k_axpy_dot<4><<<nblk, KT, 0, s>>>(V, ldv, nv, h, w, n, partial);
}
void launch_multiaxpy(const z2* V, long long ldv, int nv, const z2* h, z2* w, long long n, double* partial_norm,
                      int nblk, cudaStream_t s)
{
    k_multiaxpy<<<nblk, KT, 0, s>>>(V, ldv, nv, h, w, n, partial_norm);
}
void launch_reduce_z(const z2* partial, int nblk, int nv, z2* out, z2* out_plus, const z2* add, cudaStream_t s)
{
    k_reduce_z<<<1, 512, 0, s>>>(partial, nblk, nv, out, out_plus, add, NVMAX, 0);
}
void launch_multidot2(const z2* V, long long ldv, int nv, const z2* u, const z2* w, long long n, z2* partial, int nblk,
                      cudaStream_t s)
{
    // c3, 105 steps (ms): transposing reduction R = 2 52.8, R = 4 54.8, R = 1 72.1; per-value shuffle trees with
    // 4-vector batches (R = 4) 56.7
    k_multidot2<2><<<nblk, KT, 0, s>>>(V, ldv, nv, u, w, n, partial);
}
void launch_reduce_z2(const z2* partial, int nblk, int nv, z2* out, cudaStream_t s)
{
    k_reduce_z<<<1, 512, 0, s>>>(partial, nblk, nv, out, nullptr, nullptr, 2 * NVMAX, NVMAX);
}
void launch_dcgs2_coef(const z2* d, int j, z2* H, z2* ca, z2* ce, double* sc, z2* out, cudaStream_t s)
{
    k_dcgs2_coef<<<1, 32, 0, s>>>(d, j, H, ca, ce, sc, out);
}
void launch_dcgs2_close(const z2* d, int j, z2* H, z2* out, cudaStream_t s)
{
    k_dcgs2_close<<<1, 32, 0, s>>>(d, j, H, out);
}
void launch_dcgs2_update(z2* V, long long ldv, int j, const z2* w, const z2* ca, const z2* ce, const double* sc,
                         long long n, double* partial, int nblk, cudaStream_t s)
{
    k_dcgs2_update<<<nblk, KT, 0, s>>>(V, ldv, j, w, ca, ce, sc, n, partial);
}
void launch_reduce_norm(const double* partial, int nblk, z2* out_slot, double* out_norm, cudaStream_t s)
{
    k_reduce_norm<<<1, 32, 0, s>>>(partial, nblk, out_slot, out_norm);
}
void launch_scale_by_norm(const z2* w, const double* norm, z2* v, long long n, cudaStream_t s)
{
    k_scale<<<ew_grid(n), KT, 0, s>>>(w, norm, v, n);
}
void launch_combine(const z2* V, long long ldv, int nv, const z2* y, z2* t, long long n, cudaStream_t s)
{
    k_combine<<<ew_grid(n), KT, 0, s>>>(V, ldv, nv, y, t, n);
}
void launch_axpy(z2* x, const z2* z, long long n, cudaStream_t s) { k_axpy<<<ew_grid(n), KT, 0, s>>>(x, z, n); }
void launch_sum_ranks(const double* const* ptrs, int nranks, int count, double* out, cudaStream_t s)
{
    RankPtrs rp{};
    for (int r = 0; r < nranks && r < 16; r++) rp.p[r] = ptrs[r];
    k_sum_ranks<<<1, 128, 0, s>>>(rp, nranks, count, out);
}
void launch_copy(z2* dst, const z2* src, long long n, cudaStream_t s) { k_copy<<<ew_grid(n), KT, 0, s>>>(dst, src, n); }
void launch_norm_partial(const z2* x, long long n, double* partial, int nblk, cudaStream_t s)
{
    k_norm_partial<<<nblk, KT, 0, s>>>(x, n, partial);
}
