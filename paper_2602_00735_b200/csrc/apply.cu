// apply.cu -- K4: the fused RAS-PML preconditioner application z = sum_j R~_j^T A_j^-1 R_j r.
//
// One persistent CTA per (SM x occupancy) walks a static list of subdomains.  Per subdomain it performs
//   restrict   b_i = (R_j r) on block row i, read straight from r (rows are contiguous: x-fastest),
//   solve      the twisted block-tridiagonal substitution with the explicit Schur-complement inverses
//              written by factor.cu:
//                T  z_i = Q_i^-1 (b_i - U_i z_{i+1})           i = nb-1 .. tw+1
//                B  y_i = P_i^-1 (b_i - L_i y_{i-1})           i = 0 .. tw-1
//                Z  x_tw = Z^-1 (b_tw - L_tw y_{tw-1} - U_tw z_{tw+1})
//                D  x_i = y_i - P_i^-1 (U_i x_{i+1})           i = tw-1 .. lo   (owned rows only)
//                U  x_i = z_i - Q_i^-1 (L_i x_{i-1})           i = tw+1 .. hi   (owned rows only)
//   prolong    z[g] = x_i[t] for the owned nodes of block j only (restricted owner write, D10) -- no
//              atomics, each global node written exactly once.
// The dense m x m inverse blocks dominate the bytes.  They are streamed HBM -> shared
// memory by one producer thread with cp.async.bulk (TMA bulk copies) into a ring of `nslots` slots (2 by default,
// ~17 KB each, with 4 CTAs per SM -- see SLOT_TARGET) guarded by mbarriers (full: complete_tx, empty: one arrive per
// consumer warp), so the stream runs ahead of the serial block-row dependency chain.  Consumer thread t owns row t of every block: the GEMV reads column
// c of the column-major block (consecutive lanes -> consecutive 16-byte words, conflict-free) and the
// broadcast operand rhs[c].
#include <stdlib.h>

#include <mutex>

#include "internal.cuh"
#include "ring.cuh"

namespace {

constexpr int NS = 8;              // ring slots of the read probe; k_apply takes its ring depth at launch
// bytes per ring slot (rounded down to whole groups of 4 columns of m_max).  Swept at c3 (m = 88, 128-thread CTAs,
// 4 per SM), apply ms: 2 slots x 16.9 KB 8.88, 6 x 5.6 KB 8.95, 3 x 11.3 KB 9.06, 2 x 22.5 KB 9.21, 8 x 11.3 KB (two
// 163-register CTAs per SM) 9.35 -- a short ring of large chunks over more CTAs wins.  HELM_APPLY_SLOTB overrides.
constexpr int SLOT_TARGET = 20000;

// the bulk-copy ring and the twisted step order are shared with the tensor-core apply (ring.cuh)
using ring::bulk_g2s;
using ring::consumer_bar;
using ring::mbar_arrive;
using ring::mbar_arrive_expect_tx;
using ring::mbar_init;
using ring::mbar_wait;
using ring::nsteps;
using ring::PH_B;
using ring::PH_D;
using ring::PH_T;
using ring::PH_U;
using ring::PH_Z;
using ring::Step;
using ring::step_of;

// A coupling row (L_i or U_i) at node t: r += d v[t] + lo v[t-1] + hi v[t+1].  U_i: d = N, lo = NW, hi = NE;
// L_i: d = S, lo = SW, hi = SE (NW / SE exist for the 9-point Q1 stencil only, D18; zero for P1).
struct Cp { z2 d, lo, hi; };

// operands a consumer thread needs for one step, loaded one step ahead
struct Pre {
    z2 b;         // restricted input b_i[t]      (T, B, Z)
    Cp c;         // coupling: T, D -> U_i;  B, U, Z -> L_i  (the Z step's U_i is loaded when used: once per
                  // subdomain, and keeping it here would spill the carried operands at every step)
    z2 yz;        // y_i / z_i from scratch       (D, U)
};

__device__ __forceinline__ Cp load_upper(const z2* row, int m, int t, bool cst, const ApplyArgs& a)
{
    Cp c;
    c.d = cst ? a.cN : __ldg(row + SL_N * m + t);
    c.hi = cst ? a.cNE : __ldg(row + SL_NE * m + t);
    c.lo = a.ns == 9 ? (cst ? a.cNW : __ldg(row + SL_NW * m + t)) : zmk(0, 0);
    return c;
}
__device__ __forceinline__ Cp load_lower(const z2* row, int m, int t, bool cst, const ApplyArgs& a)
{
    Cp c;
    c.d = cst ? a.cS : __ldg(row + SL_S * m + t);
    c.lo = cst ? a.cSW : __ldg(row + SL_SW * m + t);
    c.hi = a.ns == 9 ? (cst ? a.cSE : __ldg(row + SL_SE * m + t)) : zmk(0, 0);
    return c;
}

// r -= C v (sign < 0) or r += C v, in the fixed order d, lo, hi
__device__ __forceinline__ void cpl_apply(z2& r, const Cp& c, const z2* v, int t, int m, bool minus)
{
    const double s = minus ? -1.0 : 1.0;
    zfma(r, zmk(s * c.d.x, s * c.d.y), v[t]);
    if (t > 0) zfma(r, zmk(s * c.lo.x, s * c.lo.y), v[t - 1]);
    if (t + 1 < m) zfma(r, zmk(s * c.hi.x, s * c.hi.y), v[t + 1]);
}

__device__ __forceinline__ void prefetch(Pre& p, const SubDesc& d, Step st, int t, const ApplyArgs& a,
                                         const z2* scr)
{
    if (t >= d.m) return;
    const z2* row = a.stencil + d.stc_off + (long long)st.i * a.ns * d.m;
    if (st.ph <= PH_Z) {
        const long long gi = d.gx0 + t - a.in_i0, gj = d.gy0 + st.i - a.in_j0;
        p.b = __ldg(a.in + gi + a.in_stride * gj);
    }
    // nodes whose cells all have gamma = 1 carry the constant interior couplings: no load
    const bool cst = t >= d.cx0 && t < d.cx1 && st.i >= d.cy0 && st.i < d.cy1;
    // the first step of each chain has no coupling term
    if ((st.ph == PH_T && st.i == d.nb - 1) || (st.ph == PH_B && st.i == 0)) return;
    if (st.ph == PH_Z) {
        if (st.i > 0) p.c = load_lower(row, d.m, t, cst, a);
        return;
    }
    if (st.ph == PH_T || st.ph == PH_D) p.c = load_upper(row, d.m, t, cst, a);
    else p.c = load_lower(row, d.m, t, cst, a);
    if (st.ph >= PH_D) p.yz = scr[(long long)(st.i - d.lo) * d.m + t];
}

__device__ __forceinline__ void apply_body(const ApplyArgs& a, int nc_warps, int slot_bytes, int NSL)
{
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSL * slot_bytes);
    uint64_t* empty = full + NSL;
    z2* vb = reinterpret_cast<z2*>(empty + NSL);   // bottom chain carry / down-expansion carry
    const int nct = nc_warps * 32;                // consumer threads
    z2* vt = vb + nct + 1;                        // top chain carry / up-expansion carry
    z2* rhs = vt + nct + 1;                       // GEMV operand

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < NSL; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], nc_warps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == nc_warps) {
        // ---------------------------------------------------------------- producer: stream the factors
        if (lane != 0) return;
        uint32_t slot = 0, ph = 0;
        for (int w = blockIdx.x; w < a.nsub; w += gridDim.x) {
            const SubDesc d = a.desc[a.order[w]];
            const int kc = slot_bytes / (d.m * (int)sizeof(z2)) / 4 * 4;
            const int S = nsteps(d);
            for (int s = 0; s < S; s++) {
                const Step st = step_of(d, s);
                const z2* blk = a.dinv + d.fac_off + (long long)st.i * d.m * d.m;
                for (int c0 = 0; c0 < d.m; c0 += kc) {
                    const int nc = min(kc, d.m - c0);
                    mbar_wait(&empty[slot], ph ^ 1);
                    const uint32_t bytes = (uint32_t)(nc * d.m * sizeof(z2));
                    mbar_arrive_expect_tx(&full[slot], bytes);
                    bulk_g2s(ring + (size_t)slot * slot_bytes, blk + (long long)c0 * d.m, bytes, &full[slot]);
                    if (++slot == (uint32_t)NSL) {
                        slot = 0;
                        ph ^= 1;
                    }
                }
            }
        }
        return;
    }

    // -------------------------------------------------------------------- consumers: solve the chain
    const int t = tid;
    uint32_t slot = 0, ph = 0;
    z2* scr = a.scratch + (long long)blockIdx.x * a.scratch_per_cta;
    for (int w = blockIdx.x; w < a.nsub; w += gridDim.x) {
        const SubDesc d = a.desc[a.order[w]];
        const int m = d.m;
        const bool act = t < m;
        const int kc = slot_bytes / (m * (int)sizeof(z2)) / 4 * 4;
        const int S = nsteps(d);
        Pre cur, nxt;
        prefetch(cur, d, step_of(d, 0), t, a, scr);
        for (int s = 0; s < S; s++) {
            const Step st = step_of(d, s);
            if (s + 1 < S) prefetch(nxt, d, step_of(d, s + 1), t, a, scr);
            // ---- right-hand side of this block step
            z2 r = zmk(0, 0);
            if (act) {
                switch (st.ph) {
                case PH_T:   // b_i - U_i z_{i+1}
                    r = cur.b;
                    if (st.i < d.nb - 1) cpl_apply(r, cur.c, vt, t, m, true);
                    break;
                case PH_B:   // b_i - L_i y_{i-1}
                    r = cur.b;
                    if (st.i > 0) cpl_apply(r, cur.c, vb, t, m, true);
                    break;
                case PH_Z:
                    r = cur.b;
                    if (st.i > 0) cpl_apply(r, cur.c, vb, t, m, true);
                    if (st.i < d.nb - 1) {
                        const z2* row = a.stencil + d.stc_off + (long long)st.i * a.ns * d.m;
                        const bool cst = t >= d.cx0 && t < d.cx1 && st.i >= d.cy0 && st.i < d.cy1;
                        cpl_apply(r, load_upper(row, m, t, cst, a), vt, t, m, true);
                    }
                    break;
                case PH_D:   // U_i x_{i+1}
                    cpl_apply(r, cur.c, vb, t, m, false);
                    break;
                default:     // PH_U: L_i x_{i-1}
                    cpl_apply(r, cur.c, vt, t, m, false);
                    break;
                }
                rhs[t] = r;
            }
            consumer_bar(nct);
            // ---- GEMV with the streamed block: acc = Dinv_i rhs.  Canonical order (shared with k_apply_split):
            // four partial sums over the columns c = 0, 1, 2, 3 (mod 4), each in increasing c, then (s0+s1)+(s2+s3);
            // kc is a multiple of 4, so a chunk-relative residue is the global one
            z2 s0 = zmk(0, 0), s1 = zmk(0, 0), s2 = zmk(0, 0), s3 = zmk(0, 0);
            for (int c0 = 0; c0 < m; c0 += kc) {
                const int nc = min(kc, m - c0);
                mbar_wait(&full[slot], ph);
                const z2* col = reinterpret_cast<const z2*>(ring + (size_t)slot * slot_bytes);
                if (act) {
                    int c = 0;
#pragma unroll 2
                    for (; c + 3 < nc; c += 4) {
                        zfma(s0, col[(size_t)c * m + t], rhs[c0 + c]);
                        zfma(s1, col[(size_t)(c + 1) * m + t], rhs[c0 + c + 1]);
                        zfma(s2, col[(size_t)(c + 2) * m + t], rhs[c0 + c + 2]);
                        zfma(s3, col[(size_t)(c + 3) * m + t], rhs[c0 + c + 3]);
                    }
                    if (c < nc) zfma(s0, col[(size_t)c * m + t], rhs[c0 + c]);
                    if (c + 1 < nc) zfma(s1, col[(size_t)(c + 1) * m + t], rhs[c0 + c + 1]);
                    if (c + 2 < nc) zfma(s2, col[(size_t)(c + 2) * m + t], rhs[c0 + c + 2]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[slot]);
                if (++slot == (uint32_t)NSL) {
                    slot = 0;
                    ph ^= 1;
                }
            }
            const z2 acc = zadd(zadd(s0, s1), zadd(s2, s3));
            // ---- finish the step
            if (act) {
                z2 x;
                switch (st.ph) {
                case PH_T:
                    vt[t] = acc;
                    if (st.i <= d.hi) scr[(long long)(st.i - d.lo) * m + t] = acc;
                    break;
                case PH_B:
                    vb[t] = acc;
                    if (st.i >= d.lo) scr[(long long)(st.i - d.lo) * m + t] = acc;
                    break;
                default:
                    if (st.ph == PH_Z) {
                        x = acc;
                        vb[t] = x;
                        vt[t] = x;
                    } else if (st.ph == PH_D) {
                        x = zsub(cur.yz, acc);
                        vb[t] = x;
                    } else {
                        x = zsub(cur.yz, acc);
                        vt[t] = x;
                    }
                    if (t >= d.olo && t <= d.ohi) {
                        if (a.pou_buf) {
                            // linear-ramp PoU: chi_j-weighted solution into the subdomain's slot; the
                            // gather kernel sums the <= 4 covering subdomains in index order
                            const double w = chi_ramp(d.gx0 + t, d.s0x, d.s1x, a.delta, d.flags & 1, d.flags & 2) *
                                             chi_ramp(d.gy0 + st.i, d.s0y, d.s1y, a.delta, d.flags & 4, d.flags & 8);
                            a.pou_buf[d.pou_off + (t - d.olo) + (long long)(d.ohi - d.olo + 1) * (st.i - d.lo)] =
                                zscale(x, w);
                        } else {
                            const long long gi = d.gx0 + t - a.out_i0, gj = d.gy0 + st.i - a.out_j0;
                            a.out[gi + a.out_stride * gj] = x;
                        }
                    }
                    break;
                }
            }
            consumer_bar(nct);
            cur = nxt;
        }
    }
}

// One instance per CTA-size class so that the register budget matches the block: m <= 224 (the BASELINE.json
// configs, m <= 91), m <= 480, m <= 992 (the paper's ~300-400-node-wide subdomains, D21).
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) k_apply(ApplyArgs a, int nc_warps, int slot_bytes, int nslots)
{
    apply_body(a, nc_warps, slot_bytes, nslots);
}

const void* apply_fn(int block)
{
    if (block <= 128) return (const void*)k_apply<128, 4>;
    if (block <= 256) return (const void*)k_apply<256, 1>;
    if (block <= 512) return (const void*)k_apply<512, 1>;
    return (const void*)k_apply<1024, 1>;
}

// Ramp-PoU prolongation: out(g) = sum over the <= 2 x 2 subdomains whose chi is positive at g
// of their weighted local solutions, summed in ascending subdomain index (deterministic).  Only subdomains of this
// rank's block range [bx0, bx1) x [by0, by1) contribute (descriptors are indexed locally); on several ranks the rest
// arrives through the additive reverse halo exchange.  candx / candy: per node index, the (up to) two blocks along
// that axis, -1 padded.  Nodes [i0, i1) x [j0, j1) are written to out at origin (oi0, oj0), stride ostride.
__global__ void k_pou_gather(const SubDesc* __restrict__ desc, const int* __restrict__ candx,
                             const int* __restrict__ candy, int bx0, int bx1, int by0, int by1,
                             const z2* __restrict__ buf, z2* __restrict__ out, int oi0, int oj0, long long ostride,
                             int i0, int i1, int j0, int j1)
{
    const int w = i1 - i0;
    const long long n = (long long)w * (j1 - j0);
    const int lw = bx1 - bx0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int i = i0 + (int)(e % w), j = j0 + (int)(e / w);
        z2 acc = zmk(0, 0);
        for (int b = 0; b < 2; b++) {
            const int by = candy[2 * j + b];
            if (by < by0 || by >= by1) continue;   // -1 padding fails by < by0 as well
            for (int a = 0; a < 2; a++) {
                const int bx = candx[2 * i + a];
                if (bx < bx0 || bx >= bx1) continue;
                const SubDesc d = desc[(bx - bx0) + lw * (by - by0)];
                const long long off = d.pou_off + (i - (d.gx0 + d.olo)) + (long long)(d.ohi - d.olo + 1) * (j - (d.gy0 + d.lo));
                acc = zadd(acc, buf[off]);
            }
        }
        out[(i - oi0) + ostride * (j - oj0)] = acc;
    }
}

int slot_bytes_for(int m_max)
{
    static const int target = [] { const char* e = getenv("HELM_APPLY_SLOTB"); return e ? atoi(e) : SLOT_TARGET; }();
    int kc = target / (m_max * (int)sizeof(z2)) / 4 * 4;   // whole groups of 4 columns (canonical GEMV order)
    if (kc < 4) kc = 4;
    return kc * m_max * (int)sizeof(z2);
}

}  // namespace

int apply_configure(int m_max, int nslots, int* block_threads, int* smem_bytes, int* slot_bytes, int* ctas_per_sm)
{
    const int ncw = (m_max + 31) / 32;
    *block_threads = 32 * (ncw + 1);
    *slot_bytes = slot_bytes_for(m_max);
    *smem_bytes = nslots * *slot_bytes + 2 * nslots * 8 + 3 * (32 * ncw + 1) * (int)sizeof(z2);
    const void* fn = apply_fn(*block_threads);
    raise_smem_attr(fn, *smem_bytes);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, *block_threads, *smem_bytes);
    *ctas_per_sm = occ;
    return ncw;
}

void launch_pou_gather(const SubDesc* desc, const int* candx, const int* candy, int bx0, int bx1, int by0, int by1,
                       const z2* pou_buf, z2* out, int oi0, int oj0, long long ostride, int i0, int i1, int j0, int j1,
                       cudaStream_t s)
{
    const long long n = (long long)(i1 - i0) * (j1 - j0);
    if (n <= 0) return;
    long long g = (n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    k_pou_gather<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(desc, candx, candy, bx0, bx1, by0, by1, pou_buf, out, oi0, oj0,
                                                      ostride, i0, i1, j0, j1);
}

void launch_apply(const ApplyArgs& a, int grid, int block, int smem, int slot_bytes, int nslots, cudaStream_t s)
{
    raise_smem_attr(apply_fn(block), smem);
    const int cls = block <= 128 ? 3 : (block <= 256 ? 0 : (block <= 512 ? 1 : 2));
    const int ncw = block / 32 - 1;
    if (cls == 3) k_apply<128, 4><<<grid, block, smem, s>>>(a, ncw, slot_bytes, nslots);
    else if (cls == 0) k_apply<256, 1><<<grid, block, smem, s>>>(a, ncw, slot_bytes, nslots);
    else if (cls == 1) k_apply<512, 1><<<grid, block, smem, s>>>(a, ncw, slot_bytes, nslots);
    else k_apply<1024, 1><<<grid, block, smem, s>>>(a, ncw, slot_bytes, nslots);
}

// ---------------------------------------------------------------------------------------------------------------------
// Read-bandwidth probe (measurement aid for the roofline, not part of the method): the same persistent bulk-copy ring
// as k_apply streaming a buffer HBM -> shared memory with no arithmetic, so bench.py can quote the attainable
// read-stream bandwidth beside the measured copy (read + write) peak of MEASURED_PEAKS.json.
namespace {
// mode 0: chunk c goes to CTA c mod grid (all CTAs sweep one narrow address window together);
// mode 1: CTA b streams its own contiguous 1/grid of the buffer (independent sequential streams, as k_apply does)
__global__ void k_read_probe(const unsigned char* __restrict__ buf, long long bytes, int chunk, double* sink, int mode)
{
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * chunk);
    uint64_t* empty = full + NS;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < NS; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long nchunks = bytes / chunk;
    const long long per = (nchunks + gridDim.x - 1) / gridDim.x;
    const long long c_begin = mode ? blockIdx.x * per : blockIdx.x;
    const long long c_end = mode ? min(nchunks, c_begin + per) : nchunks;
    const long long c_step = mode ? 1 : gridDim.x;
    if (tid == 32) {   // producer
        uint32_t k = 0;
        for (long long c = c_begin; c < c_end; c += c_step, k++) {
            const uint32_t slot = k % NS, ph = (k / NS) & 1;
            mbar_wait(&empty[slot], ph ^ 1);
            mbar_arrive_expect_tx(&full[slot], (uint32_t)chunk);
            bulk_g2s(smem + (size_t)slot * chunk, buf + c * chunk, (uint32_t)chunk, &full[slot]);
        }
    } else if (tid < 32) {   // consumer warp: touch one word per lane of every chunk
        double acc = 0.0;
        uint32_t k = 0;
        for (long long c = c_begin; c < c_end; c += c_step, k++) {
            const uint32_t slot = k % NS, ph = (k / NS) & 1;
            mbar_wait(&full[slot], ph);
            acc += reinterpret_cast<const double*>(smem + (size_t)slot * chunk)[tid];
            __syncwarp();
            if (tid == 0) mbar_arrive(&empty[slot]);
        }
        if (acc == 12345.678) *sink = acc;   // keeps the reads live
    }
}
}  // namespace

extern "C" int helm_probe_read_bandwidth(long long bytes, int reps, double* gbps)
{
    return helm_probe_read_bandwidth_mode(bytes, reps, 0, gbps);
}

extern "C" int helm_probe_read_bandwidth_mode(long long bytes, int reps, int mode, double* gbps)
{
    if (bytes < (1 << 24) || reps < 1 || !gbps || mode < 0 || mode > 1) return HELM_EINVAL;
    const int chunk = 12288;
    bytes = bytes / chunk * chunk;
    unsigned char* buf = nullptr;
    double* sink = nullptr;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) {
        cudaGetLastError();
        return HELM_ENOMEM;
    }
    cudaMalloc(&sink, sizeof(double));
    cudaMemset(buf, 0, bytes);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int smem = NS * chunk + 2 * NS * 8;
    raise_smem_attr((const void*)k_read_probe, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_read_probe<<<2 * nsm, 64, smem>>>(buf, bytes, chunk, sink, mode);   // warm-up
    cudaEventRecord(e0);
    for (int r = 0; r < reps; r++) k_read_probe<<<2 * nsm, 64, smem>>>(buf, bytes, chunk, sink, mode);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(buf);
    cudaFree(sink);
    if (err != cudaSuccess) return HELM_ECUDA;
    *gbps = (double)bytes * reps / (ms * 1e-3) / 1e9;
    return HELM_OK;
}
