/*
 * quapi.h -- C ABI of the B200-native QUAPI tensor-propagator library (libquapi.so).
 *
 * What it computes: the reduced density matrix rho(t_k) of an open quantum system in the
 * Feynman-Vernon model (N. S. Dattani, arXiv 1205.6872, PAPER.md = P:<line>):
 *   rho(t_N) = Eq. 8: sum over forward/backward paths of the bare propagator pair
 *              <s+_{k+1}|e^{-iH dt}|s+_k><s-_k|e^{+iH dt}|s-_{k+1}>, rho(0), and the discretised
 *              influence functional Eq. 9 with eta coefficients Eqs. 10-16
 *              of the bath response Eq. 4 for spectral density J(w) (Eq. 3, Eq. 21) at T.
 *   Memory truncation: pairs with lag k-k' <= Delta k_max (= dkmax, "L") are kept.
 *   Evaluation: the iterative tensor-propagator scheme (Makri-Makarov): the augmented
 *   reduced density matrix (ARDM) of N^L complex FP64 entries (N = M^2 path-pair states) is
 *   propagated in place on the GPU, one launch per time step, with the rho(t) readout of
 *   P:384-390 / P:415-418 fused into the same pass.  Readings of the paper (windows, limits,
 *   conventions) are listed in DESIGN.md §3.
 *
 * The problem statement follows the paper's abstract and §II: system
 * coordinate vector s, Hamiltonian H, spectral density + temperature (or G/alpha given directly),
 * rho(0), time grid {k dt}, Delta k_max; output rho at the requested time indices
 * ("allPointsOrJustFinalPoint", generalised to a list).
 *
 * Conventions
 *   - hbar = k_B = 1.  Complex numbers are qp_c64 {re, im} (binary-compatible with double2 and
 *     std::complex<double>).  Matrices are row-major [M][M].
 *   - Pair state sigma = (a, b) has flat index a*M + b; s+(sigma) = s[a], s-(sigma) = s[b].
 *   - Every function returns a qp_status; none aborts or throws.  On failure qp_last_error()
 *     returns a thread-local message naming the violated invariant (e.g. "config: H not
 *     Hermitian (max |H - H^+| = ...)", "capacity: need 4294967296 B ...").
 *   - Ownership: the caller owns every host array passed in or out and every device buffer
 *     (the Python layer allocates them with PyTorch).  The library owns only the opaque plan.
 *   - Streams are the caller's cudaStream_t passed as void*; all device work is enqueued on it.
 *     Functions marked [sync] synchronise that stream before returning.
 *   - Thread-compatible: distinct plans may be used concurrently from different threads.
 */
#ifndef QUAPI_H
#define QUAPI_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } qp_c64;

typedef enum {
    QP_OK = 0,
    QP_ERR_ARG = 1,        /* NULL pointer / bad argument to an API call                      */
    QP_ERR_CONFIG = 2,     /* invalid physics input (Hermiticity, trace, dt, M, L, out_steps)  */
    QP_ERR_CAPACITY = 3,   /* ARDM + workspace do not fit (message carries the byte count)     */
    QP_ERR_QUADRATURE = 4, /* eta quadrature did not converge (message names class and lag)    */
    QP_ERR_CUDA = 6,       /* CUDA runtime error (message carries cudaGetErrorString)          */
    QP_ERR_COMM = 7        /* reserved for the sharded path                                    */
} qp_status;

typedef enum {
    QP_J_ZERO = 0,             /* J = 0 (closed system)                                        */
    QP_J_OHMIC_EXP = 1,        /* J = (pi/2) xi w exp(-w/wc)                 (reading C.3-9)   */
    QP_J_DEBYE = 2,            /* J = (pi/2) xi w wc^2/(w^2+wc^2)            (reading C.3-9)   */
    QP_J_SUPEROHMIC_GAUSS = 3, /* J = A w^3 exp(-(w/wc)^2)   Eq. 21, P:291   (reading C.3-5)   */
    QP_J_CALLBACK = 4,         /* J(w) from a caller function, integrated on (0, J_cutoff]     */
    QP_J_G_TABLE = 5,          /* bath given directly as G(m dt/2), m = 0..2L+2, where
                                  G(tau) = int_0^tau int_0^t' alpha(t'-t'') dt'' dt'  -- the
                                  paper's "or the bath response function alpha(t)"     */
    QP_J_ETA_TABLE = 6         /* bath given as its 3L+2 eta classes (qp_plan_eta order) in eta_in,
                                  e.g. computed on the device by qp_eta_device                  */
} qp_bath_kind;

typedef struct {
    int32_t M;               /* OQS Hilbert-space dimension; 2 <= M <= 4 on the GPU path       */
    const double *s;         /* [M] coupling-coordinate eigenvalues (basis of H and rho0)      */
    const qp_c64 *H;         /* [M*M] Hermitian (|H - H^+| <= 1e-12)                           */
    const qp_c64 *rho0;      /* [M*M] Hermitian, trace 1 (<= 1e-12)                            */
    int32_t kind;            /* qp_bath_kind                                                    */
    double coupling;         /* xi (Ohmic, Debye) or A (super-Ohmic Gaussian)                   */
    double omega_c;          /* cutoff frequency wc > 0 (unused for ZERO / CALLBACK / G_TABLE)  */
    double kT;               /* k_B T >= 0 (0 => coth = 1)                                       */
    double (*J)(double w, void *user); /* QP_J_CALLBACK only: J(w) for w > 0; must be thread-safe */
    void *J_user;            /* passed back to J                                                 */
    double J_cutoff;         /* QP_J_CALLBACK only: upper integration limit (J ~ 0 beyond)      */
    const qp_c64 *G_in;      /* QP_J_G_TABLE only: [2*dkmax+3] values G(m dt/2)                 */
    double dt;               /* time step > 0                                                    */
    int64_t n_steps;         /* N_t >= 0: last time index; t = n_steps * dt                     */
    int32_t dkmax;           /* L = Delta k_max, 2 <= L <= 40 (N^L <= 4e12 entries)              */
    const int64_t *out_steps;/* sorted unique step indices in [0, n_steps]; NULL => all         */
    int64_t n_out;           /* length of out_steps, >= 0 (ignored when out_steps == NULL)      */
    int64_t max_bytes;       /* capacity budget for ARDM + workspace: > 0 => this many bytes;
                                0 => the free memory of the current CUDA device at plan creation
                                (no check when no device is visible); < 0 => no check           */
    const qp_c64 *eta_in;    /* QP_J_ETA_TABLE only: [3*dkmax+2] eta classes, qp_plan_eta order   */
    int32_t fuse_steps;      /* cap on the time steps fused into one pass over the ARDM, 0..4;
                                0 => the library's choice (4 for M = 2 with L >= 6, else 3; 2 for
                                M = 3; 1 for M = 4; persistent plans: 1).  Results
                                agree to rounding for every choice.                              */
    uint32_t flags;          /* QP_FLAG_* below; 0 for the default plan                          */
} qp_problem;

/* Plan options (qp_problem.flags).  They select among equivalent kernel paths (same result to
   rounding) and exist for testing and measurement:
   QP_FLAG_NO_TMA           -- M = 2: no TMA-staged kernels: at most 3 fused steps, plain loads
                               instead of the per-warp TMA-staged rounds;
   QP_FLAG_GENERIC_MOMENTS  -- M = 2, s = (+s, -s): the generic per-class moments instead of the
                               symmetric four-sum moments;
   QP_FLAG_NO_PERSIST       -- no persistent path: a small ARDM (<= QP_PERSIST_MAX_BYTES) otherwise
                               runs all slide steps of a qp_steps call in one single-CTA launch
                               with the ARDM and the tables in shared memory, one step at a time
                               (DESIGN.md §5). */
#define QP_FLAG_NO_TMA 1u
#define QP_FLAG_GENERIC_MOMENTS 2u
#define QP_FLAG_NO_PERSIST 4u
#define QP_PERSIST_MAX_BYTES (64ll << 10)

typedef struct qp_plan qp_plan;

typedef struct {
    int32_t M, N, L;         /* N = M^2                                                          */
    int64_t ardm_entries;    /* N^L                                                              */
    int64_t ardm_bytes;      /* 16 N^L: the single in-place ARDM buffer the caller allocates     */
    int64_t work_bytes;      /* device workspace the caller allocates (tables, partials, rho)    */
    double pmc_bytes;        /* the paper's PMC = 64 M^(2(L+1)) (Eqs. 18-19) -- reported only  */
    int64_t n_out;           /* number of rho outputs                                            */
    int64_t n_steps;
    int64_t bytes_per_step;  /* algorithmic HBM bytes of one slide step: 2 * 16 * N^L            */
    int32_t lattice;         /* 1 if s is an arithmetic progression (fewer Delta-s classes)      */
    int32_t n_classes;       /* D: number of nonzero Delta-s classes used by the kernels         */
    int32_t grid, block;     /* slide-kernel launch configuration                                */
    int32_t tile_fibres;     /* fibres per tile                                                  */
    double setup_seconds;    /* host time spent in qp_plan_create (validation, U, eta, tables)  */
    int64_t init_h2d_bytes;  /* bytes qp_init copies host->device (tables, A_0, rho(0))         */
    int32_t fuse_steps;      /* time steps fused into one pass over the ARDM (slide kernel)      */
    double setup_ms[3];      /* host setup phases: validate + U, eta quadrature, factor tables    */
    int32_t persistent;      /* 1: the slide steps of a qp_steps call run in one single-CTA launch
                                (ARDM <= QP_PERSIST_MAX_BYTES; confirmed at qp_init against the
                                device's shared memory, else 0: one launch per step); 0: one
                                launch per fusion group                                          */
} qp_sizes;

/* Host only (no GPU needed): validate (a1), U = e^{-iH dt} and the pair propagator K (a2),
   eta by omega-quadrature (a3), factor tables and launch schedule (a4).  *out owned by caller,
   free with qp_plan_destroy.  Errors: QP_ERR_ARG, QP_ERR_CONFIG, QP_ERR_QUADRATURE,
   QP_ERR_CAPACITY (only when max_bytes > 0: ARDM + workspace exceed it). */
qp_status qp_plan_create(const qp_problem *prob, qp_plan **out);
/* Capacity (a1) of the plan as configured (unsharded: ARDM + workspace; sharded: two shard buffers +
   workspace) against max_bytes (> 0), else the free memory of the current CUDA device (no check
   when no device is visible, or max_bytes < 0).  Call before allocating.  Error: QP_ERR_CAPACITY
   with the byte counts. */
qp_status qp_plan_check(const qp_plan *plan);
qp_status qp_plan_query(const qp_plan *plan, qp_sizes *out);

/* eta classes used by the plan (units: the eta of Eqs. 10-16), written as
   [self_interior (Eq. 11), self_end (Eqs. 13/14), eta_1..eta_L (Eq. 10), E_1..E_L (Eqs. 15/16),
    TI_1..TI_L (Eq. 12)]  = 3L+2 values.  cap = capacity of out in elements. */
qp_status qp_plan_eta(const qp_plan *plan, qp_c64 *out, int64_t cap);
/* U = e^{-iH dt} [M*M] as used by the plan. */
qp_status qp_plan_propagator(const qp_plan *plan, qp_c64 *U_out);

/* Enqueue: copy the plan's tables into d_work (H2D) and write A_0 into d_ardm:
   A_0(sigma_0) = rho0(sigma_0) I(sigma_0, sigma_0; eta_00)  -- the k = 0 term of Eq. 8
   with the end-point self class of Eq. 13 (reading C.3-2); rho(t_0) = rho0 (reading C.3-8).
   d_ardm: >= ardm_bytes, 16-byte aligned; d_work: >= work_bytes, 256-byte aligned.  Both device,
   caller-owned.  Errors: QP_ERR_ARG (NULL / misaligned), QP_ERR_CUDA. */
qp_status qp_init(qp_plan *plan, void *d_ardm, void *d_work, void *stream);
/* Enqueue time steps k = k_begin .. k_end-1 (1 <= k_begin <= k_end <= n_steps+1) of the iterative
   tensor propagator -- the evaluation of Eq. 8 with the influence functional of Eq. 9
    by propagating the augmented reduced density matrix (Makri-Makarov), the
   propagation the paper's GPU program runs with BSXFUN.  Step k turns
   A_{k-1} into A_k in place (growth for k < L: the tensor gains digit k; slide for k >= L: the
   oldest point sigma_{k-L} is summed out) and, when k is an output step, reduces rho(t_k) from
   A_{k-1} in the same pass -- the summation the paper times separately ("line 169").
   Slide steps are fused in groups of fuse_steps (aligned on k - L) into one kernel launch, i.e.
   one pass over the ARDM.  Steps must be enqueued in order after qp_init.  Returns the number of
   kernels launched in *n_launch (may be NULL).  Errors: QP_ERR_ARG (order, NULL), QP_ERR_CUDA. */
qp_status qp_steps(qp_plan *plan, int64_t k_begin, int64_t k_end, void *d_ardm, void *d_work, void *stream,
                   int64_t *n_launch);
/* [sync] Copy every requested rho(t_k) to the host: rho_out[n_out][M][M] (caller-owned, row-major),
   the paper's output "at all time points or just the final one" (allPointsOrJustFinalPoint,
   P:444-449, generalised to a list).  Outputs whose step has not been enqueued yet are undefined. */
qp_status qp_read_rho(const qp_plan *plan, const void *d_work, qp_c64 *rho_out, void *stream);
/* [sync] Whole run -- the paper's program from its inputs to rho(t) at the
   requested times: qp_init + qp_steps(1, n_steps+1) + qp_read_rho. */
qp_status qp_run(qp_plan *plan, void *d_ardm, void *d_work, void *stream, qp_c64 *rho_out);

/* ---------------------------------------------------------------- sharded execution (multi-GPU)
   SURVEY §8(e): G ranks (one per GPU) each hold, during segment j, the ARDM entries whose z shard
   ring slots Z_j (the z most recently written slots at the segment start k_j = L + j (L - z)) take
   one of the rank's owned value combos (a fixed, balanced range c_lo .. c_lo + n_own - 1): one block
   of N^(L-z) entries per combo, the other slots in ascending order.  The L - z slide steps of a
   segment never contract a shard slot, so they run shard-locally with the combo's Eq. 9 factors
   folded in.  No rank ever holds the N^L ARDM:
     - qp_init(plan, d_xbuf, d_work): tables, A_0 into the exchange buffer;
     - qp_shard_steps, k = 1 .. L-z-1: growth replicated in d_xbuf (N^(k+1) <= N^(L-z) entries);
       k = L-z .. L-1: the growth steps that add the shard digits, computed for this rank's combos
       only from the replicated A_{L-z-1} into d_local; k >= L: slide steps within the segment;
     - between segments: qp_shard_pack (d_local -> d_xbuf, send order), the caller's all-to-all
       (d_xbuf -> d_local, counts from qp_shard_counts, ordered by rank), qp_shard_unpack
       (d_local -> d_xbuf, next layout); the CALLER THEN SWAPS d_local and d_xbuf.
   Memory per rank: two buffers of local_entries (16 B each) + workspace (qp_plan_check).
   Readouts: steps k <= L - z are complete on every rank; later steps are this rank's partial sums
   (each prefix of the shard digits counted by exactly one rank); qp_shard_combine sums the ranks'
   outputs in rank order on the device. */
typedef struct {
    int32_t n_ranks, rank;
    int32_t shard_slots;       /* z                                                                 */
    int32_t segment_steps;     /* L - z steps between re-shards                                     */
    int64_t local_entries;     /* this rank's ARDM entries (n_own * N^(L-z))                        */
    int64_t max_local_entries; /* over ranks                                                        */
    int64_t exchange_entries;  /* entries this rank sends (and receives) per re-shard               */
    int64_t work_bytes;        /* workspace including the shard launch tables                       */
    int64_t xbuf_entries;      /* exchange buffer entries (>= local_entries, >= N^(L-z))            */
} qp_shard_sizes;

/* Host only; once, before qp_init (the workspace grows: query work_bytes again).  2 <= n_ranks.
   Errors: QP_ERR_ARG (called twice or after qp_init), QP_ERR_CONFIG (L too small for n_ranks),
   QP_ERR_CAPACITY (max_bytes > 0 and two shard buffers + workspace exceed it). */
qp_status qp_shard_configure(qp_plan *plan, int32_t n_ranks, int32_t rank);
qp_status qp_shard_query(const qp_plan *plan, qp_shard_sizes *out);
/* entries sent to / received from every rank at each re-shard: [n_ranks] each */
qp_status qp_shard_counts(const qp_plan *plan, int64_t *send_counts, int64_t *recv_counts);
/* Enqueue steps k_begin .. k_end-1 in order: growth (k < L, not mixed with slide steps in one call)
   or slide steps inside the current segment.  d_local, d_xbuf: device, local_entries / xbuf_entries
   complex entries, caller-owned.  Errors: QP_ERR_ARG (order, segment bounds), QP_ERR_CUDA. */
qp_status qp_shard_steps(qp_plan *plan, int64_t k_begin, int64_t k_end, void *d_local, void *d_xbuf, void *d_work,
                         void *stream, int64_t *n_launch);
/* Re-shard from segment j to j + 1 (at the segment's end): pack d_local -> d_xbuf in send order
   [destination rank][my block][destination's combo of Z_{j+1}][other slots]; after the caller's
   all-to-all into d_local, unpack d_local -> d_xbuf ([source rank][source's combo of Z_j][my new
   block][other slots] -> the segment j+1 layout) and advance j.  The caller then swaps d_local and
   d_xbuf. */
qp_status qp_shard_pack(qp_plan *plan, const void *d_local, void *d_xbuf, void *stream);
qp_status qp_shard_unpack(qp_plan *plan, const void *d_recv, void *d_xbuf, void *stream);
/* [sync] rho of the whole sharded run: d_parts (device, [n_ranks][n_out][M*M], every rank's rho block
   of its d_work in rank order, e.g. from an all-gather) -> rho_out (host [n_out][M][M]): rank 0's value
   for steps k <= L - z, the rank-ordered sum for later steps (fixed order: deterministic). */
qp_status qp_shard_combine(const qp_plan *plan, const void *d_parts, void *d_work, qp_c64 *rho_out, void *stream);
/* Device address offset (bytes) of the rho block [n_out][M*M] inside d_work (for gathering it). */
int64_t qp_rho_offset(const qp_plan *plan);

/* ---------------------------------------------------------------- path filtering
   Sim's on-the-fly filtering of paths, cited by the paper as the way to cut the tensor propagator's
   memory, absent from its program and invited.  Reading C.3-15
   (DESIGN.md): after every step k >= 1 the entries of A_k with |A|^2 < theta^2 are dropped; rho(t_k)
   is read from the filtered A_{k-1}; theta = 0 keeps every entry.  The ARDM is a compacted list of
   (index, value) of the kept entries (24 B each, ping-pong) instead of the dense 16 N^L B: growth and
   slide steps are count / scan / scatter passes over the list (ofpf.cu). */
/* Device bytes of the filter buffer for a list of up to `capacity` entries. */
qp_status qp_filter_query(const qp_plan *plan, int64_t capacity, int64_t *bytes);
/* [sync] Whole filtered run (init, steps 1..n_steps, readouts): d_buf (device, buf_bytes, caller-owned)
   holds the list, d_work (work_bytes) the plan's tables and outputs; rho_out host [n_out][M][M];
   kept_out (host [n_steps + 1] or NULL): entries of the list after each step (kept_out[0]: the nonzero
   entries of A_0).  Errors: QP_ERR_ARG, QP_ERR_CAPACITY (the list outgrew the buffer: message names the
   step), QP_ERR_CUDA. */
qp_status qp_filter_run(qp_plan *plan, double theta, void *d_buf, int64_t buf_bytes, void *d_work, void *stream,
                        qp_c64 *rho_out, int64_t *kept_out);

/* ---------------------------------------------------------------- device eta setup
   Host-setup step a3 on the GPU: every eta class of Eqs. 10-16 (Strang windows, DESIGN.md
   reading C.3-1) for B baths at once -- the setup the paper names as the bottleneck once propagation
   runs on the GPU, and the per-problem tables of temperature / coupling sweeps.
   Each class is the omega-integral of its window kernel on a fixed composite Gauss-Kronrod 21 rule
   (panels short against the integrand's nearest complex singularity; Debye: closed-form tail), one
   8-CTA cluster per (bath, class), deterministic (fixed-order reductions, no atomics). */
typedef struct {
    int32_t kind;            /* QP_J_ZERO, QP_J_OHMIC_EXP, QP_J_DEBYE or QP_J_SUPEROHMIC_GAUSS          */
    double coupling;         /* xi (Ohmic, Debye) or A (super-Ohmic Gaussian), as in qp_problem         */
    double omega_c;          /* > 0                                                                      */
    double kT;               /* >= 0                                                                     */
} qp_bath;
/* Enqueue on `stream`: d_eta[b][c] (device, caller-owned, B*(3*dkmax+2) qp_c64) = eta class c of bath b
   in the qp_plan_eta order [self_interior, self_end, eta_1..L, E_1..L, TI_1..L] for time step dt and
   L = dkmax; d_err (device, B*(3*dkmax+2) doubles, may be NULL) = the summed |K21 - G10| panel
   estimate (a loose upper bound on the quadrature error).  baths: host [B], read before return.
   Errors: QP_ERR_ARG (NULL, B < 1, dt <= 0, L out of range), QP_ERR_CONFIG (kind not one of the four
   analytic families, omega_c <= 0, kT < 0, non-finite coupling), QP_ERR_CUDA (launch). */
qp_status qp_eta_device(const qp_bath *baths, int32_t B, double dt, int32_t dkmax, qp_c64 *d_eta, double *d_err,
                        void *stream);

const char *qp_last_error(void);
void qp_plan_destroy(qp_plan *plan);
/* Library build identification, e.g. "quapi 0.1 sm_100a". */
const char *qp_version(void);

/* ---------------------------------------------------------------- batched sweeps
   B independent problems that share M, s, the bath, dt, L = dkmax, n_steps and out_steps, each with
   its own initial state and its own drive: problem b propagates on the interval (t_{k-1}, t_k] of step
   k with H_b(k) = H0 + f[b * n_steps + k - 1] * H1 -- the driven quantum dot of the paper's Sec. III
   (Omega(t) of P:288), whose rho_11 is swept over pulse areas.  Step k uses the propagator
   pair K_k = U_k (x) conj(U_k), U_k = exp(-i H_b(k) dt) (Eq. 8 with a step-dependent H); everything
   else (eta classes, windows, readout from A_{k-1}) is the single-problem method.  One CTA owns one
   problem for the whole run (one kernel launch, every step inside it). */
typedef struct {
    qp_problem base;         /* shared parameters; base.H = H0, base.rho0 = initial state of every problem
                                unless rho0 below is given (base.rho0 is validated either way)          */
    int32_t B;               /* number of problems >= 1                                                  */
    const qp_c64 *H1;        /* [M*M] Hermitian drive operator, or NULL (no drive)                       */
    const double *f;         /* [B][n_steps] finite drive amplitudes, or NULL (all 0)                    */
    const qp_c64 *rho0;      /* [B][M*M] per-problem initial states (Hermitian, trace 1), or NULL      */
    const qp_bath *baths;    /* [B] per-problem baths (temperature / coupling sweeps),
                                or NULL (every problem uses base's bath).  Their eta classes are
                                computed on the device at qp_batch_run (as qp_eta_device); base's bath
                                is then unused and may be QP_J_ZERO.  Analytic families 0..3 only.   */
} qp_batch;

typedef struct qp_batch_plan qp_batch_plan;

typedef struct {
    int32_t B, M, N, L;
    int64_t ardm_entries;    /* B * N^L                                                                  */
    int64_t ardm_bytes;      /* 16 * B * N^L: the caller's ARDM buffer (problem b at offset 16 b N^L)    */
    int64_t work_bytes;      /* device workspace (tables, drive, initial states, rho outputs)            */
    int64_t n_out, n_steps;
    int32_t block;           /* threads per problem (one CTA per problem)                                */
    double setup_seconds;
} qp_batch_sizes;

/* Host only: validate (base as qp_plan_create; H1 Hermitian; f finite; each rho0 Hermitian with trace
   1), eta and tables of the shared bath.  Errors as qp_plan_create. */
qp_status qp_batch_create(const qp_batch *batch, qp_batch_plan **out);
qp_status qp_batch_query(const qp_batch_plan *plan, qp_batch_sizes *out);
/* Enqueue the whole batched run on `stream` (H2D of the tables, one kernel launch).  If rho_out is
   not NULL, synchronises and writes rho_out[B][n_out][M][M] (host, caller-owned). */
qp_status qp_batch_run(qp_batch_plan *plan, void *d_ardm, void *d_work, void *stream, qp_c64 *rho_out);
void qp_batch_destroy(qp_batch_plan *plan);

#ifdef __cplusplus
}
#endif
#endif
