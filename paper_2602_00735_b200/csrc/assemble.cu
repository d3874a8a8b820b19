// assemble.cu -- structured-mesh assembly of the PML operators on the device.
//
//   K1 assemble_global : ns coefficients per free row of A (eq. (weak)), SoA slots [ns][n_local]
//   K2 assemble_local  : ns coefficients per local free node of every A_j, [nb][ns][m] per subdomain
//   K10 rhs            : f at the free nodes (sum of Gaussians, D14) then b = M f with the P1 / Q1 mass stencil
// ns = 7 for P1 on the SW->NE split (D1), 9 for the bilinear Q1 elements of the paper's experiments (D18).
//
// Each row is gathered from the six triangles around its node (a per-row formulation; the oracle
// scatters element matrices instead).  PML coefficients D = diag(gamma^-2), beta = gamma'/gamma^3
// are frozen at the triangle centroid (D5); gamma_i = 1 + i g_i' with the profile
// g(t) = sigma0 t^3/(3 kappa^2), linear beyond kappa (BASELINE.json configs[0]; D3).  Lower-side ramps
// are g_i(x) = -g(a - x), so gamma' = -i g''(a - x) there (D4).
#include "internal.cuh"

namespace {

__device__ __forceinline__ void ramp_d(long d3, bool upper, const Geom& g, z2& gam, z2& dgam)
{
    double t = (double)d3 * g.h3;
    double g1, g2;
    if (t <= g.kappa) {
        g1 = g.sigma0 * t * t / (g.kappa * g.kappa);
        g2 = 2.0 * g.sigma0 * t / (g.kappa * g.kappa);
    } else {
        g1 = g.sigma0;
        g2 = 0.0;
    }
    gam = zmk(1.0, g1);
    dgam = zmk(0.0, upper ? g2 : -g2);
}

// global scaling g_i: ramps above node N - n_g and below node n_g
__device__ __forceinline__ void gamma_global(long X3, const Geom& g, z2& gam, z2& dgam)
{
    if (X3 > g.hi3) ramp_d(X3 - g.hi3, true, g, gam, dgam);
    else if (X3 < g.lo3) ramp_d(g.lo3 - X3, false, g, gam, dgam);
    else { gam = zmk(1.0, 0.0); dgam = zmk(0.0, 0.0); }
}

// local scaling g_j^i: upper ramp from b_j, lower ramp from a_j, global g_i in between; only on
// faces carrying a local PML (kappa_{j,l/u} != 0)
__device__ __forceinline__ void gamma_local(long X3, long a3, long b3, bool has_lo, bool has_hi, const Geom& g,
                                            z2& gam, z2& dgam)
{
    if (has_hi && X3 > b3) ramp_d(X3 - b3, true, g, gam, dgam);
    else if (has_lo && X3 < a3) ramp_d(a3 - X3, false, g, gam, dgam);
    else gamma_global(X3, g, gam, dgam);
}

// The six triangles around node (i, j): cell offset, triangle (0 = lower SW->NE half, 1 = upper half) and
// the node's vertex index in that triangle.  Triangle vertices relative to the cell corner:
//   lower {(0,0),(1,0),(1,1)}, upper {(0,0),(1,1),(0,1)}  (D1); h * grad phi: see TG.
struct TriRef { int cdx, cdy, tri, a; };
__constant__ TriRef c_tris[6] = { {-1, -1, 0, 2}, {-1, -1, 1, 1}, {0, -1, 1, 2},
                                  {-1, 0, 0, 1},  {0, 0, 0, 0},   {0, 0, 1, 0} };
__constant__ int c_tv[2][3][2] = { { {0, 0}, {1, 0}, {1, 1} }, { {0, 0}, {1, 1}, {0, 1} } };
__constant__ double c_tg[2][3][2] = { { {-1, 0}, {1, -1}, {0, 1} }, { {0, -1}, {1, 0}, {-1, 1} } };
__constant__ int c_c3[2][2] = { {2, 1}, {1, 2} };   // centroid offset in thirds

__device__ __forceinline__ int slot_of(int dx, int dy)
{
    // (0,0) C, (1,0) E, (-1,0) W, (0,1) N, (0,-1) S, (1,1) NE, (-1,-1) SW
    if (dy == 0) return dx == 0 ? SL_C : (dx > 0 ? SL_E : SL_W);
    if (dx == 0) return dy > 0 ? SL_N : SL_S;
    return dx > 0 ? SL_NE : SL_SW;
}

// Row of node (i, j) (global node indices): A[p][q] = 1/2 (D11 gx_p gx_q + D22 gy_p gy_q)
//   - h/6 (beta1 gx_q + beta2 gy_q) - k^2 h^2 / 24 (1 + delta_pq), with g = h grad phi.
// Only triangles of cells in [cx0, cx1) x [cy0, cy1) contribute (the domain of the form: Omega, or the full
// box of a subdomain -- relevant for nodes on an impedance face).
template <class GammaFn>
__device__ void node_row(int i, int j, const Geom& g, GammaFn gam_at, z2 row[7], int cx0, int cx1, int cy0, int cy1)
{
    for (int s = 0; s < 7; s++) row[s] = zmk(0.0, 0.0);
    const double kh2_24 = g.k * g.k * g.h * g.h / 24.0;
    const double h6 = g.h / 6.0;
#pragma unroll
    for (int e = 0; e < 6; e++) {
        const TriRef T = c_tris[e];
        const int ci = i + T.cdx, cj = j + T.cdy, tri = T.tri, a = T.a;
        if (ci < cx0 || ci >= cx1 || cj < cy0 || cj >= cy1) continue;
        z2 gx, dgx, gy, dgy;
        gam_at(0, 3L * ci + c_c3[tri][0], gx, dgx);
        gam_at(1, 3L * cj + c_c3[tri][1], gy, dgy);
        const z2 ix = zinv(gx), iy = zinv(gy);
        const z2 D11 = zmul(ix, ix), D22 = zmul(iy, iy);
        const z2 b1 = zmul(dgx, zmul(D11, ix)), b2 = zmul(dgy, zmul(D22, iy));
        const double gxa = c_tg[tri][a][0], gya = c_tg[tri][a][1];
        for (int q = 0; q < 3; q++) {
            const double gxq = c_tg[tri][q][0], gyq = c_tg[tri][q][1];
            z2 v = zadd(zscale(D11, 0.5 * gxa * gxq), zscale(D22, 0.5 * gya * gyq));
            v = zsub(v, zscale(zadd(zscale(b1, gxq), zscale(b2, gyq)), h6));
            v.x -= kh2_24 * (q == a ? 2.0 : 1.0);
            const int dx = T.cdx + c_tv[tri][q][0], dy = T.cdy + c_tv[tri][q][1];
            const int s = slot_of(dx, dy);
            row[s] = zadd(row[s], v);
        }
    }
}


// ------------------------------------------------------------------------------------------------ Q1 (D18-D20)
// PML coefficients at x = (ci + xi) h.  Depth below / above a ramp start r (cell units) is (r - ci) - xi resp.
// (ci - r) + xi, scaled by h.  Profile: paper frame g(t) = pml_c t^3, else the BJ profile.
__device__ __forceinline__ void ramp_q(double t, bool upper, const Geom& g, z2& gam, z2& dgam)
{
    double g1, g2;
    if (g.frame == 1) {
        g1 = 3.0 * g.pml_c * t * t;
        g2 = 6.0 * g.pml_c * t;
    } else if (t <= g.kappa) {
        g1 = g.sigma0 * t * t / (g.kappa * g.kappa);
        g2 = 2.0 * g.sigma0 * t / (g.kappa * g.kappa);
    } else {
        g1 = g.sigma0;
        g2 = 0.0;
    }
    gam = zmk(1.0, g1);
    dgam = zmk(0.0, upper ? g2 : -g2);
}

__device__ __forceinline__ void gamma_global_q(int ci, double xi, const Geom& g, z2& gam, z2& dgam)
{
    const double up = ((double)ci - g.hi_u) + xi, dn = (g.lo_u - (double)ci) - xi;
    if (up > 0.0) ramp_q(up * g.h, true, g, gam, dgam);
    else if (dn > 0.0) ramp_q(dn * g.h, false, g, gam, dgam);
    else { gam = zmk(1.0, 0.0); dgam = zmk(0.0, 0.0); }
}

// local scaling g_j^i; a, b = int box faces (cell / node index)
__device__ __forceinline__ void gamma_local_q(int ci, double xi, int a, int b, bool has_lo, bool has_hi, const Geom& g,
                                              z2& gam, z2& dgam)
{
    const double up = (double)(ci - b) + xi, dn = (double)(a - ci) - xi;
    if (has_hi && up > 0.0) ramp_q(up * g.h, true, g, gam, dgam);
    else if (has_lo && dn > 0.0) ramp_q(dn * g.h, false, g, gam, dgam);
    else gamma_global_q(ci, xi, g, gam, dgam);
}

__device__ __forceinline__ int slot9(int dx, int dy)
{
    if (dy == 0) return dx == 0 ? SL_C : (dx > 0 ? SL_E : SL_W);
    if (dx == 0) return dy > 0 ? SL_N : SL_S;
    if (dx > 0) return dy > 0 ? SL_NE : SL_SE;
    return dy > 0 ? SL_NW : SL_SW;
}

// Row of node (i, j) from its four cells (bilinear basis phi_a = N_ax(xi) N_ay(eta), a = ax + 2 ay):
//   A_e[a][b] = sum_q h^2/4 [D11 dx phi_a dx phi_b + D22 dy phi_a dy phi_b - (beta . grad phi_b) phi_a - k^2 phi_a phi_b]
// with the 2 x 2 Gauss rule; D11, beta_1 depend on x only, D22, beta_2 on y only.  Cells outside [cx0, cx1) x
// [cy0, cy1) do not contribute.
template <class GammaFn>
__device__ void node_row_q1(int i, int j, const Geom& g, GammaFn gam_at, z2 row[9], int cx0, int cx1, int cy0, int cy1)
{
    for (int s = 0; s < 9; s++) row[s] = zmk(0.0, 0.0);
    const double gq[2] = {0.5 - 0.5 / sqrt(3.0), 0.5 + 0.5 / sqrt(3.0)};
    const double w = 0.25 * g.h * g.h, ih = 1.0 / g.h, k2 = g.k * g.k;
#pragma unroll
    for (int cc = 0; cc < 4; cc++) {
        const int ax = 1 - (cc & 1), ay = 1 - (cc >> 1);   // this node's vertex in cell (i - ax, j - ay)
        const int ci = i - ax, cj = j - ay;
        if (ci < cx0 || ci >= cx1 || cj < cy0 || cj >= cy1) continue;
        z2 D11[2], D22[2], b1[2], b2[2];
        for (int q = 0; q < 2; q++) {
            z2 ga, dga;
            gam_at(0, ci, gq[q], ga, dga);
            z2 iv = zinv(ga);
            D11[q] = zmul(iv, iv);
            b1[q] = zmul(dga, zmul(D11[q], iv));
            gam_at(1, cj, gq[q], ga, dga);
            iv = zinv(ga);
            D22[q] = zmul(iv, iv);
            b2[q] = zmul(dga, zmul(D22[q], iv));
        }
        for (int b = 0; b < 4; b++) {
            const int bx = b & 1, by = b >> 1;
            z2 v = zmk(0.0, 0.0);
            for (int qx = 0; qx < 2; qx++)
                for (int qy = 0; qy < 2; qy++) {
                    const double Nx[2] = {1.0 - gq[qx], gq[qx]}, Ny[2] = {1.0 - gq[qy], gq[qy]};
                    const double dN[2] = {-ih, ih};
                    const double pa = Nx[ax] * Ny[ay], pax = dN[ax] * Ny[ay], pay = Nx[ax] * dN[ay];
                    const double pb = Nx[bx] * Ny[by], pbx = dN[bx] * Ny[by], pby = Nx[bx] * dN[by];
                    z2 t = zadd(zscale(D11[qx], pax * pbx), zscale(D22[qy], pay * pby));
                    t = zsub(t, zscale(zadd(zscale(b1[qx], pbx), zscale(b2[qy], pby)), pa));
                    t.x -= k2 * pa * pb;
                    v = zadd(v, zscale(t, w));
                }
            const int s = slot9(bx - ax, by - ay);
            row[s] = zadd(row[s], v);
        }
    }
}

__constant__ int c_sdx[9] = { 0, 1, -1, 0, 0, 1, -1, -1, 1 };
__constant__ int c_sdy[9] = { 0, 0, 0, 1, -1, 1, -1, 1, -1 };

__global__ void k_assemble_global(Geom g, z2* __restrict__ A, int ns, int i0, int i1, int j0, int j1)
{
    const long long w = i1 - i0, n = w * (long long)(j1 - j0);
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const int i = i0 + (int)(r % w), j = j0 + (int)(r / w);
        z2 row[9];
        if (g.elem == HELM_ELEM_Q1)
            node_row_q1(i, j, g, [&](int, int ci, double xi, z2& ga, z2& dga) { gamma_global_q(ci, xi, g, ga, dga); },
                        row, 0, g.N, 0, g.N);
        else
            node_row(i, j, g, [&](int, long X3, z2& ga, z2& dga) { gamma_global(X3, g, ga, dga); }, row, 0, g.N, 0,
                     g.N);
        for (int s = 0; s < ns; s++) {
            const int qi = i + c_sdx[s], qj = j + c_sdy[s];
            const bool free_q = qi >= 1 && qi <= g.nf && qj >= 1 && qj <= g.nf;
            A[s * n + r] = free_q ? row[s] : zmk(0.0, 0.0);
        }
    }
}

__global__ void k_assemble_local(Geom g, const SubDesc* __restrict__ desc, z2* __restrict__ stc)
{
    const SubDesc d = desc[blockIdx.y];
    const int n = d.m * d.nb;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int t = r % d.m, row_i = r / d.m;
        const int i = d.gx0 + t, j = d.gy0 + row_i;
        z2 rowv[9];
        if (d.ns == 9)
            node_row_q1(i, j, g,
                        [&](int axis, int ci, double xi, z2& ga, z2& dga) {
                            if (axis == 0) gamma_local_q(ci, xi, d.ilo3 / 3, d.ihi3 / 3, d.flags & 1, d.flags & 2, g, ga, dga);
                            else gamma_local_q(ci, xi, d.jlo3 / 3, d.jhi3 / 3, d.flags & 4, d.flags & 8, g, ga, dga);
                        },
                        rowv, d.fx0, d.fx1, d.fy0, d.fy1);
        else
            node_row(i, j, g,
                     [&](int axis, long X3, z2& ga, z2& dga) {
                         if (axis == 0) gamma_local(X3, d.ilo3, d.ihi3, d.flags & 1, d.flags & 2, g, ga, dga);
                         else gamma_local(X3, d.jlo3, d.jhi3, d.flags & 4, d.flags & 8, g, ga, dga);
                     },
                     rowv, d.fx0, d.fx1, d.fy0, d.fy1);
        if (d.imp) {
            // RAS-PML-Imp: -i k int_face u v on faces of Omega_j not on dOmega; P1 / Q1 trace = the
            // 1-D linear edge mass (h/6)[[2,1],[1,2]] per edge of length h (no PML metric)
            const double w1 = g.k * g.h / 6.0;   // -i k h/6 = (0, -w1)
            auto edge = [&](int slot) {
                rowv[SL_C].y -= 2.0 * w1;
                rowv[slot].y -= w1;
            };
            if (((d.imp & 1) && i == d.fx0) || ((d.imp & 2) && i == d.fx1)) {   // face x = const: edges along y
                if (j - 1 >= d.fy0) edge(SL_S);
                if (j + 1 <= d.fy1) edge(SL_N);
            }
            if (((d.imp & 4) && j == d.fy0) || ((d.imp & 8) && j == d.fy1)) {   // face y = const: edges along x
                if (i - 1 >= d.fx0) edge(SL_W);
                if (i + 1 <= d.fx1) edge(SL_E);
            }
        }
        z2* out = stc + d.stc_off + (long long)row_i * d.ns * d.m + t;
        for (int s = 0; s < d.ns; s++) {
            const int qt = t + c_sdx[s], qr = row_i + c_sdy[s];
            const bool inside = qt >= 0 && qt < d.m && qr >= 0 && qr < d.nb;   // Dirichlet on dOmega_j (D9)
            out[s * d.m] = inside ? rowv[s] : zmk(0.0, 0.0);
        }
    }
}

// f at the free nodes of [i0-1, i1] x [j0-1, j1] (clipped), stored with a one-node frame
__global__ void k_rhs_f(Geom g, int nsrc, const double* __restrict__ xy, const z2* __restrict__ amp, double sigma,
                        z2* __restrict__ f, int i0, int i1, int j0, int j1)
{
    const int fw = i1 - i0 + 2, fh = j1 - j0 + 2;
    const long long n = (long long)fw * fh;
    const double c = 1.0 / (2.0 * M_PI * sigma * sigma), e = 1.0 / (2.0 * sigma * sigma);
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const int i = i0 - 1 + (int)(r % fw), j = j0 - 1 + (int)(r / fw);
        z2 acc = zmk(0.0, 0.0);
        if (i >= 1 && i <= g.nf && j >= 1 && j <= g.nf) {
            const double x = (i - g.ng) * g.h, y = (j - g.ng) * g.h;
            for (int s = 0; s < nsrc; s++) {
                const double dx = x - xy[2 * s], dy = y - xy[2 * s + 1];
                const double w = c * exp(-(dx * dx + dy * dy) * e);
                acc = zadd(acc, zscale(amp[s], w));
            }
        }
        f[r] = acc;
    }
}

// b = M f: consistent P1 mass stencil on the SW->NE mesh: centre h^2/2, E W N S NE SW h^2/12 (PML-free,
// the k^2 u v term of eq. (weak) carries no gamma)
__global__ void k_rhs_b(Geom g, const z2* __restrict__ f, z2* __restrict__ b, int i0, int i1, int j0, int j1)
{
    const int w = i1 - i0, fw = w + 2;
    const long long n = (long long)w * (j1 - j0);
    const bool q1 = g.elem == HELM_ELEM_Q1;
    // P1: centre h^2/2, E W N S NE SW h^2/12.  Q1 (tensor product of the 1-D (h/6)[4, 1]): centre 16 h^2/36, edge
    // neighbours 4 h^2/36, corners h^2/36
    const double mc = q1 ? 16.0 * g.h * g.h / 36.0 : g.h * g.h / 2.0;
    const double mo = q1 ? 4.0 * g.h * g.h / 36.0 : g.h * g.h / 12.0;
    const double mk = q1 ? g.h * g.h / 36.0 : 0.0;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const int li = (int)(r % w) + 1, lj = (int)(r / w) + 1;
        const z2* fc = f + li + (long long)fw * lj;
        z2 acc = zscale(fc[0], mc);
        z2 o = zadd(zadd(fc[1], fc[-1]), zadd(fc[fw], fc[-fw]));
        if (q1) {
            const z2 c = zadd(zadd(fc[fw + 1], fc[-fw - 1]), zadd(fc[fw - 1], fc[-fw + 1]));
            acc = zadd(acc, zscale(c, mk));
        } else {
            o = zadd(o, zadd(fc[fw + 1], fc[-fw - 1]));
        }
        b[r] = zadd(acc, zscale(o, mo));   // f is 0 at Dirichlet nodes (frame filled with zeros there)
    }
}

int grid_for(long long n, int threads)
{
    long long b = (n + threads - 1) / threads;
    if (b > 148LL * 32) b = 148LL * 32;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

void launch_assemble_global(const Geom& g, z2* A, int ns, int i0, int i1, int j0, int j1, cudaStream_t s)
{
    const long long n = (long long)(i1 - i0) * (j1 - j0);
    k_assemble_global<<<grid_for(n, 256), 256, 0, s>>>(g, A, ns, i0, i1, j0, j1);
}

void launch_assemble_local(const Geom& g, const SubDesc* d_desc, int nsub, z2* stencil, int max_n, cudaStream_t s)
{
    // blockIdx.y = subdomain (nsub <= 65535 per launch chunk)
    const int per = 256;
    for (int base = 0; base < nsub; base += 65535) {
        const int cnt = nsub - base < 65535 ? nsub - base : 65535;
        dim3 grid((max_n + per - 1) / per, cnt);
        k_assemble_local<<<grid, per, 0, s>>>(g, d_desc + base, stencil);
    }
}

void launch_rhs(const Geom& g, int nsrc, const double* d_xy, const z2* d_amp, double sigma, z2* f_work, z2* b,
                int i0, int i1, int j0, int j1, cudaStream_t s)
{
    const long long nf = (long long)(i1 - i0 + 2) * (j1 - j0 + 2);
    k_rhs_f<<<grid_for(nf, 256), 256, 0, s>>>(g, nsrc, d_xy, d_amp, sigma, f_work, i0, i1, j0, j1);
    const long long n = (long long)(i1 - i0) * (j1 - j0);
    k_rhs_b<<<grid_for(n, 256), 256, 0, s>>>(g, f_work, b, i0, i1, j0, j1);
}
