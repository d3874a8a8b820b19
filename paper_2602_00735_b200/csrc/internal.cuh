// internal.cuh -- shared device/host definitions of libhelm (product code; independent of oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "helm.h"

// The dynamic shared-memory limit of a kernel is a per-function attribute shared by every context of the process, and
// contexts may configure / launch from concurrent host threads (loopback ranks): raise it monotonically under one lock
// (a context lowering it between another context's set and launch would make that launch fail).  Also sets
// NonPortableClusterSizeAllowed when `nonportable`.  Defined in helm_api.cu.
void raise_smem_attr(const void* fn, int smem, bool nonportable = false);

// ---------------------------------------------------------------------------------------------------
// complex128 helpers (double2 = (re, im))
// ---------------------------------------------------------------------------------------------------
typedef double2 z2;

__host__ __device__ __forceinline__ z2 zmk(double r, double i) { return make_double2(r, i); }
__host__ __device__ __forceinline__ z2 zadd(z2 a, z2 b) { return zmk(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ z2 zsub(z2 a, z2 b) { return zmk(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ z2 zmul(z2 a, z2 b) { return zmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__host__ __device__ __forceinline__ z2 zscale(z2 a, double s) { return zmk(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ z2 zconj(z2 a) { return zmk(a.x, -a.y); }
__host__ __device__ __forceinline__ double zabs2(z2 a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ z2 zinv(z2 a)
{
    double d = a.x * a.x + a.y * a.y;
    return zmk(a.x / d, -a.y / d);
}
__host__ __device__ __forceinline__ z2 zdiv(z2 a, z2 b) { return zmul(a, zinv(b)); }
// acc += a * b
__device__ __forceinline__ void zfma(z2& acc, z2 a, z2 b)
{
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void zfma_conj(z2& acc, z2 a, z2 b)
{
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}

// ---------------------------------------------------------------------------------------------------
// Problem geometry on the device (global PML ramps) and per-subdomain descriptors.
// Positions along an axis are integers in thirds of a cell ("X3"): triangle centroids sit at 3i+1 or
// 3i+2, node n at 3n, so PML depth is an integer times h/3 (D5).
// ---------------------------------------------------------------------------------------------------
struct Geom {
    double k, h, h3, sigma0, kappa;   // h3 = h / 3; kappa = profile width kappa_g
    int N;                            // cells per side
    int nf;                           // free nodes per side = N - 1
    int ng;                           // global PML cells per side
    long lo3, hi3;                    // Omega_int = nodes [n_g, N - n_g]  -> 3 n_g, 3 (N - n_g)
    int elem;                         // HELM_ELEM_P1 / HELM_ELEM_Q1
    int frame;                        // 0 BJ frame, 1 paper frame (Omega = (0,1)^2, PML inside; D19)
    double lo_u, hi_u;                // Q1 path: Omega_int in cell units (node 0 at 0), ramps start there
    double pml_c;                     // paper frame: g(t) = pml_c t^3
};

// One subdomain as seen by the local operator / factor / apply kernels.
struct SubDesc {
    int m;          // block size: local free nodes per row (x)
    int nb;         // number of block rows (local free nodes per column, y)
    int tw;         // twist block row
    int lo, hi;     // owned block rows [lo, hi]
    int olo, ohi;   // owned columns [olo, ohi] within a row
    int gx0, gy0;   // global node index of local node (t = 0, row 0)
    int ilo3, ihi3; // int box x-range in thirds (local ramps start there) ...
    int jlo3, jhi3; // ... and y-range
    int flags;      // bit0 x-lower PML, bit1 x-upper, bit2 y-lower, bit3 y-upper
    int cx0, cx1;   // local columns [cx0, cx1) and rows [cy0, cy1) whose six triangles all have gamma = 1:
    int cy0, cy1;   //   their couplings equal the constant interior stencil (apply skips those loads)
    int fx0, fx1;   // full box in cells (= node indices of its faces): only triangles of these cells count
    int fy0, fy1;
    int imp;        // impedance faces: bit0 x-lower, bit1 x-upper, bit2 y-lower, bit3 y-upper
    int s0x, s1x;   // block cells [s0, s1) per axis (linear-ramp partition of unity)
    int s0y, s1y;
    int ns;         // stencil slots per local row: 7 (P1) or 9 (Q1)
    long long fac_off;   // complex offset of block 0 of the explicit inverses (blocks m x m, column-major)
    long long stc_off;   // complex offset of the local stencil [nb][7][m]
    long long pou_off;   // ramp-PoU mode: offset of this subdomain's weighted solution [lo..hi][olo..ohi]
};

// linear-ramp PoU factor along one axis at node x: 0 -> 1 across [s0-d, s0+d], 1 -> 0 across
// [s1-d, s1+d], 1 toward dOmega; d = overlap delta
__host__ __device__ __forceinline__ double chi_ramp(int x, int s0, int s1, int d, bool lo, bool hi)
{
    if (lo && x <= s0 - d) return 0.0;
    if (hi && x >= s1 + d) return 0.0;
    if (lo && x < s0 + d) return (double)(x - (s0 - d)) / (2.0 * d);
    if (hi && x > s1 - d) return (double)(s1 + d - x) / (2.0 * d);
    return 1.0;
}

enum { SL_C = 0, SL_E = 1, SL_W = 2, SL_N = 3, SL_S = 4, SL_NE = 5, SL_SW = 6, SL_NW = 7, SL_SE = 8 };

#define HELM_CUDA_OK(expr)                                                                   \
    do {                                                                                     \
        cudaError_t e__ = (expr);                                                            \
        if (e__ != cudaSuccess) return set_err(ctx, HELM_ECUDA, "%s: %s (%s:%d)", #expr,     \
                                               cudaGetErrorString(e__), __FILE__, __LINE__); \
    } while (0)

// kernel launchers (defined in the .cu files)
void launch_assemble_global(const Geom& g, z2* A, int ns, int i0, int i1, int j0, int j1, cudaStream_t s);
void launch_assemble_local(const Geom& g, const SubDesc* d_desc, int nsub, z2* stencil, int max_n, cudaStream_t s);
void launch_rhs(const Geom& g, int nsrc, const double* d_xy, const z2* d_amp, double sigma, z2* f_work, z2* b,
                int i0, int i1, int j0, int j1, cudaStream_t s);
int factor_smem_bytes(int m_max);
constexpr int M_SMEM = 112;   // largest block the shared-memory factorisation holds; larger blocks use clusters
void launch_factor(const SubDesc* d_desc, const SubDesc* h_desc, int nsub, int m_max, const z2* stencil, z2* dinv,
                   int* d_err, cudaStream_t s);

struct ApplyArgs {
    const SubDesc* desc;
    const int* order;       // subdomains in processing order
    int nsub;
    const z2* dinv;
    const z2* stencil;
    const z2* in;           // input vector (possibly with ghost frame)
    int in_i0, in_j0;       // node index of in[0]
    long long in_stride;
    z2* out;                // owned output
    int out_i0, out_j0;
    long long out_stride;
    z2* scratch;            // per-CTA [max_rows][m_max]
    long long scratch_per_cta;
    z2 cS, cSW, cN, cNE;    // couplings of the constant interior stencil
    z2 cSE, cNW;            // ... and the Q1 corner couplings
    int ns;                 // local stencil slots (7 P1, 9 Q1)
    z2* pou_buf;            // ramp-PoU mode: weighted local solutions (else nullptr: owner write to out)
    int delta;              // overlap width (ramp half-width)
};
void launch_pou_gather(const SubDesc* desc, const int* candx, const int* candy, int bx0, int bx1, int by0, int by1,
                       const z2* pou_buf, z2* out, int oi0, int oj0, long long ostride, int i0, int i1, int j0, int j1,
                       cudaStream_t s);
int apply_configure(int m_max, int nslots, int* block_threads, int* smem_bytes, int* slot_bytes, int* ctas_per_sm);
// cluster-split apply for few large subdomains (apply_split.cu)
int split_configure(int m_max, int G, int ctas_per_sm, int* block_threads, int* smem_bytes, int* slot_bytes, int* ncw,
                    int* nslots);
int max_split_clusters(int G, int block, int smem);
int launch_apply_split(const ApplyArgs& a, int nsub, int G, int block, int smem, int slot_bytes, int ncw, int m_max,
                       int nslots, cudaStream_t s);
void launch_relayout(const SubDesc* desc, const int2* blocks, int nblocks, z2* dinv, z2* tmp, long long tmp_per_cta,
                     int grid, int G, cudaStream_t s);
void launch_apply(const ApplyArgs& a, int grid, int block, int smem, int slot_bytes, int nslots, cudaStream_t s);

// owned rows [i0, i0+nx) x [j0, j0+ny) of the 7- or 9-point operator; x read from a buffer with origin (xi0, xj0).
// Rows whose node lies in [ci0, ci1) x [cj0, cj1) -- all six triangles inside Omega_int, gamma = 1 --
// share one stencil c7 (copied from an assembled interior row, so bitwise equal to A7 there) and skip the
// seven coefficient loads.
struct StencilGeom {
    int i0, j0, nx, ny, nf;
    int xi0, xj0;
    long long xstride;
    int ci0, ci1, cj0, cj1;
    int ns;                 // 7 (P1) or 9 (Q1) slots
    z2 c7[9];
};
void launch_spmv(const z2* A7, const z2* x, z2* y, const StencilGeom& G, cudaStream_t s, int a0 = 0, int a1 = 0,
                 int b0 = 0, int b1 = 0);
void launch_spmv_frame(const z2* A7, const z2* x, z2* y, const StencilGeom& G, int a0, int a1, int b0, int b1,
                       cudaStream_t s);
void launch_residual(const z2* A7, const z2* x, const z2* b, z2* r, const StencilGeom& G, double* partial, int nblk,
                     cudaStream_t s);
void launch_copy_rect(const z2* src, int si0, int sj0, long long sstride, z2* dst, int di0, int dj0, long long dstride,
                      int i0, int i1, int j0, int j1, cudaStream_t s, bool add = false);
void launch_reduce_sq(const double* partial, int nblk, double* sq, cudaStream_t s);
void launch_band_mask(z2* v, int i0, int i1, int j0, int j1, const unsigned char* bx, const unsigned char* by,
                      cudaStream_t s);
void launch_pack_rects(z2* ext, int e_i0, int e_j0, long long stride, const int4* rects, const long long* off,
                       int nrects, long long max_area, z2* buf, bool unpack, cudaStream_t s);
void launch_finish_norm(const double* sq, z2* out_slot, double* out_norm, cudaStream_t s);
void launch_zadd(const z2* a, const z2* b, z2* out, int nv, cudaStream_t s);
void launch_multidot(const z2* V, long long ldv, int nv, const z2* w, long long n, z2* partial, int nblk,
                     cudaStream_t s);
void launch_axpy_dot(const z2* V, long long ldv, int nv, const z2* h, z2* w, long long n, z2* partial, int nblk,
                     cudaStream_t s);
void launch_multiaxpy(const z2* V, long long ldv, int nv, const z2* h, z2* w, long long n, double* partial_norm,
                      int nblk, cudaStream_t s);
void launch_reduce_z(const z2* partial, int nblk, int nv, z2* out, z2* out_plus, const z2* add, cudaStream_t s);
void launch_multidot2(const z2* V, long long ldv, int nv, const z2* u, const z2* w, long long n, z2* partial, int nblk,
                      cudaStream_t s);
void launch_reduce_z2(const z2* partial, int nblk, int nv, z2* out, cudaStream_t s);
void launch_dcgs2_coef(const z2* d, int j, z2* H, z2* ca, z2* ce, double* sc, z2* out, cudaStream_t s);
void launch_dcgs2_close(const z2* d, int j, z2* H, z2* out, cudaStream_t s);
void launch_dcgs2_update(z2* V, long long ldv, int j, const z2* w, const z2* ca, const z2* ce, const double* sc,
                         long long n, double* partial, int nblk, cudaStream_t s);
void launch_reduce_norm(const double* partial, int nblk, z2* out_slot, double* out_norm, cudaStream_t s);
void launch_scale_by_norm(const z2* w, const double* norm, z2* v, long long n, cudaStream_t s);
void launch_combine(const z2* V, long long ldv, int nv, const z2* y, z2* t, long long n, cudaStream_t s);
void launch_axpy(z2* x, const z2* z, long long n, cudaStream_t s);
void launch_copy(z2* dst, const z2* src, long long n, cudaStream_t s);
void launch_sum_ranks(const double* const* ptrs, int nranks, int count, double* out, cudaStream_t s);
void launch_norm_partial(const z2* x, long long n, double* partial, int nblk, cudaStream_t s);

// ---------------------------------------------------------------------------------------------------------------------
// Shared-factor apply (batch.cu, D28): subdomains with bitwise-equal local operators form a class; one
// representative is factored and the class's inverses are applied to BATCH_NT subdomains at a time on DMMA.
// ---------------------------------------------------------------------------------------------------------------------
#define BATCH_NT 16
struct CplConst { z2 cS, cSW, cN, cNE, cSE, cNW; int ns; };   // constant interior couplings (apply fast path)
struct BatchTile { int cls, first, cnt, pad; };                // members[first .. first + cnt) of class cls
struct BatchClass { long long off; int rep, mp, S, pad; };     // batch-layout factor offset, representative, padded m, stride
struct BatchArgs {
    const SubDesc* desc;
    const BatchTile* tiles;
    int ntiles;
    const int* members;     // subdomain indices, grouped per tile
    const BatchClass* cls;
    const z2* dinvB;        // class factors, batch layout
    const z2* stencil;
    const z2* in;
    int in_i0, in_j0;
    long long in_stride;
    z2* out;
    int out_i0, out_j0;
    long long out_stride;
    z2* scratch;            // per CTA [max(hi - lo + 1)][BATCH_NT][mp_max]
    long long scratch_per_cta;
    CplConst cc;
    z2* pou_buf;
    int delta;
};
int batch_configure(int mpmax, int* block, int* smem, int* slot_bytes, int* nslots, int* ctas_per_sm);
int launch_apply_batch(const BatchArgs& a, int grid, int block, int smem, int slot_bytes, int nslots, int mpmax,
                       int split, cudaStream_t s);   // split: clusters of two CTAs per tile; returns the cudaError_t
void launch_relayout_batch(const z2* dinv, long long fac_off, int m, int nb, z2* dst, int mp, int S, cudaStream_t s);
void launch_stencil_eq(const SubDesc* desc, const z2* stc, const int2* pairs, int npairs, int* diff, cudaStream_t s);
