/*
 * helm.h -- C ABI of libhelm: the B200-native (sm_100a) hot path of the one-level restricted additive
 * Schwarz method with PML transmission conditions (RAS-PML) of arXiv 2602.00735 for P1, complex-valued,
 * high-frequency 2D Helmholtz systems, used as a right preconditioner inside restarted GMRES.
 *
 * Citations: "P:n" = the paper's text line n with the section / equation named; D-numbers are
 * the readings in DESIGN.md section 3.  All vectors are complex128 (IEEE fp64 re/im interleaved,
 * == cuDoubleComplex == torch.complex128), indexed over the free nodes (i, j), 1 <= i, j <= N-1, of the
 * uniform mesh, x-fastest: g = (i - 1) + (N - 1) (j - 1).
 *
 * Ownership: the context owns every device allocation it makes (operators, factors, Krylov basis,
 * scratch).  The caller owns every vector argument; "_dev" pointers are device memory holding this
 * rank's owned rectangle (helm_layout), "_host" pointers are host memory.  Work is ordered on the CUDA
 * stream given to helm_setup; functions return once the work is enqueued unless stated otherwise.
 *
 * Errors: every int-returning function returns HELM_OK (0), a positive solver status, or a negative
 * error code; helm_last_error() then describes it.  A context stays destroyable after any error.
 *
 * No CPU fallback: every arithmetic step runs in the library's own CUDA kernels.
 */
#ifndef HELM_H
#define HELM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } helm_z;
typedef struct helm_ctx helm_ctx;

enum {
    HELM_OK = 0,
    HELM_NOT_CONVERGED = 2,   /* maxit reached; x holds the last iterate */
    HELM_BREAKDOWN = 3,       /* NaN / Inf in the Arnoldi process */
    HELM_DIVERGED = 4,        /* Richardson: relative residual above 1e6 or not finite */
    HELM_EINVAL = -1,         /* bad argument or unsupported parameter combination */
    HELM_ENOMEM = -2,         /* device allocation failed */
    HELM_ECUDA = -3,          /* CUDA runtime error */
    HELM_ENCCL = -4,          /* multi-rank communication error / not built with NCCL */
    HELM_EZEROPIVOT = -5,     /* singular Schur complement block: message names subdomain, block, row */
    HELM_ELAYOUT = -6,        /* a subdomain extension leaves Omega (blocks smaller than delta + kappa) */
    HELM_ESTATE = -7          /* apply / gmres before helm_factor */
};

enum {
    HELM_BC_DIRICHLET = 0,   /* RAS-PML-Drch: u = 0 on dOmega_j, P:131-137, P:152 (D9); the hot path */
    HELM_BC_IMPEDANCE = 1    /* RAS-PML-Imp: d_nu u - i k u = 0 on the faces of Omega_j not on dOmega */
};

/* Problem and decomposition (P:36-62 problem, P:71-92 covering; BASELINE.json configs). */
typedef struct {
    double k;            /* wavenumber (> 0); constant wave speed c = 1 */
    int ppw;             /* points per wavelength: n_int = round(ppw k / 2 pi) cells on (0,1), h = 1/n_int (D2) */
    int n_pml_global;    /* global PML cells per side; PML profile width kappa_g = n_pml_global * h (D3) */
    double sigma0;       /* profile g(t) = sigma0 t^3 / (3 kappa_g^2), linear beyond kappa_g */
    int nsub_x, nsub_y;  /* Cartesian subdomain grid */
    int n_ovlp, n_pml;   /* overlap delta / local PML kappa in cells per interior face; < 0 => max(2, round(1.59 ln k)) */
    int local_bc;        /* HELM_BC_DIRICHLET or HELM_BC_IMPEDANCE */
    int gpu_grid_x, gpu_grid_y;   /* rank grid over the subdomain grid; product == nranks (0,0 => most square) */
    int pou;             /* HELM_POU_OWNER: restricted owner write (D10, the hot path); HELM_POU_RAMP: linear
                            ramps across the overlaps, blocks >= 2 delta cells; on several ranks the sums over
                            covering subdomains cross rank boundaries (additive reverse halo exchange), so ramp needs a
                            communicator (NCCL or loopback), not a communication-free shard */
    /* The paper's own workload (D18-D22).  Zero-initialised fields give
     * the BASELINE.json problem above. */
    int elem;            /* HELM_ELEM_P1: P1 on the SW->NE split, 7-point stencil (D1); HELM_ELEM_Q1: bilinear
                            elements, 9-point stencil, 2 x 2 Gauss quadrature of D and beta (D18) */
    int n_cells;         /* > 0 selects the paper frame (D19): Omega = (0,1)^2 itself is n_cells x n_cells cells and
                            the global PML lies inside it; ppw, n_pml_global and sigma0 are then unused.  Needs Q1. */
    double kappa_g;      /* paper frame: global PML width; Omega_int = (kappa_g, 1 - kappa_g)^2 (3 lambda) */
    double pml_c;        /* paper frame: PML profile g(t) = pml_c t^3 (10 k) */
} helm_params;

enum { HELM_POU_OWNER = 0, HELM_POU_RAMP = 1 };
enum { HELM_ELEM_P1 = 0, HELM_ELEM_Q1 = 1 };

typedef struct {
    long long n_free_global;  /* (N-1)^2 */
    int N_cells;              /* cells per side including the global PML: n_int + 2 n_pml_global */
    int n_int;                /* cells across Omega_int = (0,1) */
    int n_ovlp, n_pml;        /* resolved widths */
    int owned_i0, owned_i1;   /* this rank's owned free nodes: i in [owned_i0, owned_i1) (1-based node index) */
    int owned_j0, owned_j1;   /* ... and j in [owned_j0, owned_j1) */
    long long n_local;        /* (owned_i1 - owned_i0) * (owned_j1 - owned_j0): length of every _dev vector */
    int n_sub;                /* total subdomains */
    int n_sub_local;          /* subdomains whose factors this rank holds */
    int m_max;                /* largest local block size (free nodes per local row) */
    long long local_unknowns; /* sum over local subdomains of n_j */
    long long factor_bytes;   /* bytes of explicit Schur-complement inverses held by this rank */
    long long apply_bytes;    /* algorithmic DRAM bytes one helm_precond_apply moves on this rank */
    long long band_bytes;     /* the same operator as band L+U factors + gather + write (SURVEY 8(d) B_apply) */
    long long spmv_bytes;     /* algorithmic bytes of one helm_matvec on this rank */
    int stencil_slots;        /* coefficients per row of A (helm_export_stencil): 7 (P1) or 9 (Q1) */
    int overlap_interior;     /* multi-rank: subdomains applied while the halo is in flight (0: no overlap) */
    long long factor_flop;    /* real FP64 flops of helm_factor's block inversions: sum over blocks of 8 m^3 (one
                                 complex multiply-add per entry and pivot of Gauss-Jordan); after helm_factor, over
                                 the factored class representatives only (D28) */
} helm_layout;

typedef struct {
    int iterations;      /* Arnoldi steps (one A B^-1 product each) */
    int restarts;        /* completed cycles minus one */
    int status;          /* HELM_OK, HELM_NOT_CONVERGED, HELM_BREAKDOWN */
    int applies;         /* preconditioner applications issued: DCGS2 (default) one per Arnoldi step, plus the
                            discarded lookahead step at a cycle's end on several ranks; undelayed CGS2 one per
                            step plus one per cycle end */
    double relres_est;   /* |g_{j+1}| / ||b|| of the last Givens step */
    double relres_true;  /* ||b - A x|| / ||b|| recomputed at the last cycle end */
    double* history;     /* caller-owned host buffer for relres_est per iteration, or NULL */
    int history_cap;
} helm_gmres_info;

/* Create a context: grid, decomposition, device assembly of the global operator A (eq. (weak))
 * and of every local operator A_j.  rank / nranks: this process's place in the job; nranks > 1
 * with nccl_unique_id (128 bytes from helm_nccl_unique_id, identical on all ranks) creates an NCCL
 * communicator over which halos and GMRES inner products are exchanged (collective: every rank calls it);
 * nranks > 1 with nccl_unique_id == NULL creates a communication-free shard (see the _ext entry points).
 * cuda_stream: cudaStream_t or NULL (legacy default stream).  Allocates the operators. */
int helm_setup(const helm_params* params, int rank, int nranks, const void* nccl_unique_id,
               void* cuda_stream, helm_ctx** out);
/* (nranks == 1 with a non-NULL nccl_unique_id runs the multi-rank code path over a one-rank NCCL communicator:
 *  ghost-framed buffers and an NCCL allreduce of every inner product -- the NCCL data plane on one GPU.) */

/* Which transport this context's collectives use, and the communicator's size and this rank's place in it as the
 * transport reports them (ncclCommCount / ncclCommUserRank for NCCL).  Host only. */
enum { HELM_TRANSPORT_NONE = 0, HELM_TRANSPORT_NCCL = 1, HELM_TRANSPORT_LOOPBACK = 2, HELM_TRANSPORT_SHARD = 3 };
int helm_comm_info(const helm_ctx* ctx, int* transport, int* comm_nranks, int* comm_rank);

/* Test aid: the NCCL transport of the halo exchange (the grouped ncclSend / ncclRecv every exchange phase posts) run on
 * this context's communicator with every rank sending nmsg (1..4) messages of nelem - q complex elements (nelem >= nmsg)
 * to ITSELF --
 * the same function exchange phases call, executable on a single GPU.  *mismatches = received elements that differ
 * from what was sent (0 on success).  HELM_ENCCL without a communicator. */
int helm_nccl_selftest(helm_ctx* ctx, long long nelem, int nmsg, long long* mismatches);

/* Fill *out with the layout of this rank.  Synchronous, host only. */
int helm_get_layout(const helm_ctx* ctx, helm_layout* out);

/* b = M f_I: f = sum_s amp_s (2 pi sigma^2)^-1 exp(-|x - xy_s|^2 / (2 sigma^2)) at the free nodes, M the
 * consistent P1 mass matrix (D14).  xy_host: 2*nsrc doubles (x0,y0,x1,y1,...), amp_host: nsrc values,
 * both host memory; b_dev: n_local values. */
int helm_rhs(helm_ctx* ctx, int nsrc, const double* xy_host, const helm_z* amp_host, double sigma, helm_z* b_dev);

/* Factor every local operator of this rank once (setup; P:143-147 A_j^-1): twisted block-tridiagonal
 * LU with explicit inverses of the Schur-complement blocks.  Synchronises the stream;
 * HELM_EZEROPIVOT names the first singular block.  Idempotent. */
int helm_factor(helm_ctx* ctx);

/* y = A x (7-point P1 stencil of eq. (weak)).  x_dev, y_dev: n_local values, distinct. */
int helm_matvec(helm_ctx* ctx, const helm_z* x_dev, helm_z* y_dev);

/* z = B^-1 r = sum_j R~_j^T A_j^-1 R_j r: restrict to every PML-extended subdomain, exact local
 * solves, restricted owner write (chi_j = indicator of block j, D10).  r_dev, z_dev: n_local values, distinct. */
int helm_precond_apply(helm_ctx* ctx, const helm_z* r_dev, helm_z* z_dev);

/* Same with host buffers: r_host -> device, apply, device -> z_host; synchronous (end-to-end path). */
int helm_precond_apply_host(helm_ctx* ctx, const helm_z* r_host, helm_z* z_host);

/* Right-preconditioned restarted GMRES(restart), 1 <= restart <= 63, on A (B^-1 u) = b, x = B^-1 u (D13):
 * x_dev in: initial guess, out: solution.  rtol on ||b - A x|| / ||b||; rtol <= 0 runs exactly maxit
 * iterations.  Synchronous.  Returns HELM_OK / HELM_NOT_CONVERGED / HELM_BREAKDOWN or an error.
 * Orthogonalisation: classical Gram-Schmidt with one re-orthogonalisation pass (CGS2), by default with that pass
 * delayed into the next step's projection sweep (DCGS2: two sweeps over the basis per step instead of
 * three; the same vectors in exact arithmetic) and the cycle's solution update formed from the steps' own applies
 * (x += Z R^-1 y: one apply per iteration, none per restart); helm_set_orthogonalisation selects the undelayed form.
 * An initial guess that already meets rtol returns at once with 0 iterations.  info->applies counts applies. */
int helm_gmres(helm_ctx* ctx, const helm_z* b_dev, helm_z* x_dev, int restart, double rtol, int maxit,
               helm_gmres_info* info);

enum { HELM_ORTH_DCGS2 = 0, HELM_ORTH_CGS2 = 1 };
/* GMRES orthogonalisation of this context (default HELM_ORTH_DCGS2).  HELM_EINVAL for another mode.  Every rank of
 * a multi-rank run must select the same mode. */
int helm_set_orthogonalisation(helm_ctx* ctx, int mode);

/* Copy the first nv vectors of the GMRES basis left by the last helm_gmres call (V slots 0 .. nv-1, each n_local
 * values, x-fastest) to out_dev (nv * n_local values; device memory).  Diagnostic (orthogonality tests).
 * HELM_ESTATE before any helm_gmres, HELM_EINVAL if nv exceeds the basis capacity (largest restart + 1 so far). */
int helm_get_krylov_basis(helm_ctx* ctx, int nv, helm_z* out_dev);

/* Same with host b / x (copied in and out inside the call). */
int helm_gmres_host(helm_ctx* ctx, const helm_z* b_host, helm_z* x_host, int restart, double rtol, int maxit,
                    helm_gmres_info* info);

/* Algorithm 1 RAS_IterSolve in discrete form: u <- u + B^-1 (b - A u) from the
 * initial guess in x_dev until ||b - A u|| <= rtol ||b|| (HELM_OK), maxit steps (HELM_NOT_CONVERGED), or the
 * relative residual exceeds 1e6 / is not finite (HELM_DIVERGED).  One apply, one SpMV per step; synchronous. */
typedef struct {
    int iterations;
    int status;
    double relres;       /* final ||b - A u|| / ||b|| */
    double* history;     /* caller-owned host buffer for the relative residual after each step, or NULL */
    int history_cap;
} helm_richardson_info;
int helm_richardson(helm_ctx* ctx, const helm_z* b_dev, helm_z* x_dev, double rtol, int maxit,
                    helm_richardson_info* info);

/* Practical improvement (i) of the paper (section 3): "the right-hand side of (local-ras-discrete) is
 * nonzero only in overlapping regions, and thus the communication of the local residuals can be restricted to these
 * regions".  With the owner partition of unity (the default, D10) helm_richardson restricts the residual of every step
 * after the first to the interface band -- node indices s_p - 1, s_p of every interior block boundary, per axis; outside
 * it the residual is rounding noise (pinned on the oracle) and is set to exactly 0 -- and on several ranks the apply's
 * halo exchange carries only the band part of the ghost frame.  on = 1 (default with the owner PoU) / 0 (Algorithm 1
 * with the full residual).  HELM_EINVAL for on = 1 with the ramp PoU (its residual fills the whole overlap). */
int helm_set_residual_band(helm_ctx* ctx, int on);

/* Traffic of this context's collectives since the last reset: out4 = {complex elements sent and received by halo
 * exchanges, halo messages posted, allreduces issued}; reset != 0 zeroes them after reading.  Host only. */
int helm_comm_counters(helm_ctx* ctx, int reset, long long* out4);

/* Shared factors (D28; P:85-94 defines A_j, P:143-147 its use).  Subdomains whose assembled local operators
 * are bitwise equal (with c = 1, the interior subdomains are translates of one another) form a class; helm_factor
 * factors one representative per class and every member uses its inverses, and when the classes are large the apply
 * runs class tiles of 16 subdomains as complex GEMMs on the FP64 tensor cores (k_apply_batch).  Filled after
 * helm_factor (HELM_ESTATE before): out6 = {classes, shared-factor apply on (1) / off (0), tiles of that apply,
 * factor bytes held on the device, algorithmic flops of one apply (8 m^2 per block step of every subdomain: one
 * complex m x m matrix-vector product), flops the tensor-core apply issues (whole 16-column tiles, m padded to a
 * multiple of 8; 0 when off)}; class_of (may be NULL) receives n_sub_local class indices, cap entries at most.
 * Environment (read at helm_setup): HELM_SHARE_FACTORS=0 factors every subdomain (one class each);
 * HELM_APPLY_BATCH=1 / 0 forces the tensor-core apply on / off (default: on when the whole problem has at least
 * as many subdomains as the GPU has SMs and m_max <= 128).  Host only. */
int helm_factor_classes(const helm_ctx* ctx, long long* out6, int* class_of, int cap);

/* Host logic, no GPU: this rank's apply-frame halo volume in complex elements -- out4 = {sent full, sent band, received
 * full, received band} (band = the section 3(i) restriction) -- and the band sub-rectangles (i0, i1, j0, j1 per
 * rectangle, node indices, canonical packing order) of message `msg` of helm_halo_schedule(width 0), side 0 = its
 * send rectangle, 1 = its receive rectangle; returns the rectangle count (at most cap written). */
int helm_halo_band_counts(const helm_params* params, int rank, int nranks, long long* out4);
int helm_halo_band_rects(const helm_params* params, int rank, int nranks, int msg, int side, int* out, int cap);

/* Parity export: the global operator as S slot arrays [S][n_local], S = helm_layout.stencil_slots (slot order
 * centre, E, W, N, S, NE, SW, and for Q1 NW, SE; a slot pointing at a Dirichlet node is 0).  out_dev: S * n_local
 * values. */
int helm_export_stencil(helm_ctx* ctx, helm_z* out_dev);

/* Kernel timing of the apply kernel: when enabled, CUDA events bracket every launch of the fused apply
 * kernel on the context's stream; helm_profile_read synchronises and returns the summed milliseconds
 * and count of the timed apply launches, and the number of libhelm kernels launched by helm_matvec /
 * helm_precond_apply / helm_gmres since the last read (then resets both). */
int helm_profile_enable(helm_ctx* ctx, int on);
int helm_profile_read(helm_ctx* ctx, double* apply_ms, int* apply_launches, int* total_launches);

/* ---------------------------------------------------------------------------------------------------
 * Multi-rank layout (one process per GPU).  The P_x x P_y subdomain grid is cut into a
 * gpu_grid_x x gpu_grid_y rank grid (rank = rx + gpu_grid_x * ry); each rank owns the union of its blocks'
 * owned nodes (a rectangle) and the factors of its subdomains.  Before an apply a rank needs its input on
 * ext = owned rectangle grown toward every neighbouring rank by delta + kappa - 1 nodes below and
 * delta + kappa above (the full boxes of its edge subdomains reach that far, with half-open
 * ownership, D10); the SpMV needs 1 node.  Exchanges run in two phases (x, then y over the x-extended
 * range, which carries the corners).  These two functions are pure host logic (no CUDA) so that the
 * exchange schedule can be verified on CPU.
 * ------------------------------------------------------------------------------------------------- */
typedef struct {
    int gx, gy, rx, ry;
    int owned_i0, owned_i1, owned_j0, owned_j1;   /* free nodes [i0,i1) x [j0,j1), 1-based node index */
    int ext_i0, ext_i1, ext_j0, ext_j1;           /* apply input rectangle incl. ghosts */
    int halo_lo, halo_hi;                         /* ghost layers below / above: delta+kappa-1, delta+kappa */
    int nbr[4];                                   /* neighbour ranks: -x, +x, -y, +y (-1: none) */
    int n_sub_local;
} helm_plan;

typedef struct {
    int phase;                  /* 0: x exchange, 1: y exchange (after phase 0 is unpacked) */
    int peer;                   /* rank to send to and receive from */
    int send_i0, send_i1, send_j0, send_j1;   /* rectangle (node indices) packed and sent to peer */
    int recv_i0, recv_i1, recv_j0, recv_j1;   /* rectangle received from peer into the ghost frame */
} helm_msg;

int helm_plan_rank(const helm_params* params, int rank, int nranks, helm_plan* out);
/* Messages of one exchange for `rank`: width 0 = the apply frame (halo_lo below, halo_hi above), width W in
 * [1, halo_hi] = W layers on both sides.  Returns the count (<= 4) or a negative error.  A message's send
 * and receive rectangles may differ in shape (a rank sends halo_hi layers down, receives halo_lo). */
int helm_halo_schedule(const helm_params* params, int rank, int nranks, int width, helm_msg* out, int cap);

/* 128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it); HELM_ENCCL without NCCL. */
int helm_nccl_unique_id(void* out128);

/* Test transport: rank `rank` of an in-process group `group` (>= 0) of `nranks` (2..16) contexts on ONE device, each
 * driven by its own host thread and stream.  Every collective entry point (apply, matvec, gmres, richardson, the
 * norms) then runs the full multi-rank code path -- ghost frames, the two-phase halo schedule, reductions -- with the
 * NCCL calls replaced by device-to-device copies between the group's buffers ordered by host barriers (allreduce sums
 * the ranks in rank order).  No kernel waits on another.  All ranks of a group must call the same functions in the
 * same order from concurrent threads; helm_destroy leaves the group. */
int helm_setup_loopback(const helm_params* params, int rank, int nranks, int group, void* cuda_stream, helm_ctx** out);

/* Communication-free sharded entry points: the caller supplies the input already extended with ghosts.
 * ext_dev covers the plan's ext rectangle (apply) / the owned rectangle grown by one node toward every
 * neighbour (matvec), x-fastest.  Valid on every context, including nranks > 1 contexts created with
 * nccl_unique_id == NULL (which cannot run helm_gmres / helm_precond_apply / helm_matvec). */
int helm_precond_apply_ext(helm_ctx* ctx, const helm_z* ext_dev, helm_z* z_dev);
int helm_matvec_ext(helm_ctx* ctx, const helm_z* ext1_dev, helm_z* y_dev);

/* Measurement aid (not part of the method): read bandwidth of the bulk-copy streaming pattern k_apply uses, over a
 * freshly allocated device buffer of `bytes` (>= 16 MiB, larger than L2 for a meaningful figure), `reps` timed passes
 * on the legacy default stream.  Synchronous; *gbps = bytes * reps / time.  HELM_ENOMEM if the buffer cannot be
 * allocated. */
int helm_probe_read_bandwidth(long long bytes, int reps, double* gbps);
/* Same with an access-pattern mode: 0 (the call above) hands chunk c to CTA c mod grid, so all CTAs sweep one narrow
 * address window together; 1 gives every CTA its own contiguous 1/grid of the buffer -- independent sequential
 * streams, the pattern of the apply kernel (each CTA streams its own subdomains' factors). */
int helm_probe_read_bandwidth_mode(long long bytes, int reps, int mode, double* gbps);

/* Measurement aid (not part of the method): FP64 peak of this GPU, the roofline denominator of the setup factorisation.
 * mode 0: tensor-core DMMA (mma.sync m8n8k4 f64) issue rate; mode 1: plain DFMA.  Synchronous; *tflops measured with
 * CUDA events over one launch of independent chains on every SM. */
int helm_probe_fp64_tflops(int mode, double* tflops);

const char* helm_last_error(const helm_ctx* ctx);
void helm_destroy(helm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* HELM_H */
