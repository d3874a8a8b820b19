// ring.cuh -- device helpers shared by the streaming apply kernels (apply.cu, batch.cu): mbarrier-guarded TMA bulk-copy
// rings, the twisted step sequence of one local solve and the coupling rows L_i / U_i.
#pragma once
#include "internal.cuh"

namespace ring {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
// TMA bulk copy global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// named barrier 1 over the consumer warps (the producer warp never joins it)
__device__ __forceinline__ void consumer_bar(int nthreads)
{
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// The block steps of one twisted local solve, in streaming order:
//   T  z_i = Q_i^-1 (b_i - U_i z_{i+1})           i = nb-1 .. tw+1
//   B  y_i = P_i^-1 (b_i - L_i y_{i-1})           i = 0 .. tw-1
//   Z  x_tw = Z^-1 (b_tw - L_tw y_{tw-1} - U_tw z_{tw+1})
//   D  x_i = y_i - P_i^-1 (U_i x_{i+1})           i = tw-1 .. lo   (owned rows only)
//   U  x_i = z_i - Q_i^-1 (L_i x_{i-1})           i = tw+1 .. hi   (owned rows only)
enum { PH_T = 0, PH_B = 1, PH_Z = 2, PH_D = 3, PH_U = 4 };

struct Step { int ph, i; };

__device__ __forceinline__ int nsteps(const SubDesc& d) { return d.nb + d.hi - d.lo; }

__device__ __forceinline__ Step step_of(const SubDesc& d, int s)
{
    const int nT = d.nb - 1 - d.tw, nB = d.tw, nD = d.tw - d.lo;
    if (s < nT) return {PH_T, d.nb - 1 - s};
    s -= nT;
    if (s < nB) return {PH_B, s};
    s -= nB;
    if (s == 0) return {PH_Z, d.tw};
    s -= 1;
    if (s < nD) return {PH_D, d.tw - 1 - s};
    s -= nD;
    return {PH_U, d.tw + 1 + s};
}

// A coupling row (L_i or U_i) at node t: r += d v[t] + lo v[t-1] + hi v[t+1].  U_i: d = N, lo = NW, hi = NE;
// L_i: d = S, lo = SW, hi = SE (NW / SE exist for the 9-point Q1 stencil only, D18; zero for P1).
struct Cp { z2 d, lo, hi; };

__device__ __forceinline__ Cp load_upper(const z2* row, int m, int t, bool cst, const CplConst& a)
{
    Cp c;
    c.d = cst ? a.cN : __ldg(row + SL_N * m + t);
    c.hi = cst ? a.cNE : __ldg(row + SL_NE * m + t);
    c.lo = a.ns == 9 ? (cst ? a.cNW : __ldg(row + SL_NW * m + t)) : zmk(0, 0);
    return c;
}
__device__ __forceinline__ Cp load_lower(const z2* row, int m, int t, bool cst, const CplConst& a)
{
    Cp c;
    c.d = cst ? a.cS : __ldg(row + SL_S * m + t);
    c.lo = cst ? a.cSW : __ldg(row + SL_SW * m + t);
    c.hi = a.ns == 9 ? (cst ? a.cSE : __ldg(row + SL_SE * m + t)) : zmk(0, 0);
    return c;
}

// r -= C v (minus) or r += C v, in the fixed order d, lo, hi
__device__ __forceinline__ void cpl_apply(z2& r, const Cp& c, const z2* v, int t, int m, bool minus)
{
    const double s = minus ? -1.0 : 1.0;
    zfma(r, zmk(s * c.d.x, s * c.d.y), v[t]);
    if (t > 0) zfma(r, zmk(s * c.lo.x, s * c.lo.y), v[t - 1]);
    if (t + 1 < m) zfma(r, zmk(s * c.hi.x, s * c.hi.y), v[t + 1]);
}

}  // namespace ring
