/*
 * oracle.h -- plain, slow CPU oracle for the QUAPI tensor-propagator step.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under oracle/ is part of the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so.  The oracle shares no code,
 * header, table or constant generator with paper_1205_6872_b200/ (the CUDA
 * path); neither includes nor links the other.
 *
 * Citations: P:<line> = /root/reference/PAPER.md line (section / equation),
 * readings C.3-<n> = the table of readings in DESIGN.md (mirrors SURVEY.md §8(c)).
 * Units: hbar = k_B = 1.
 */
#ifndef QUAPI_ORACLE_H
#define QUAPI_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_J_ZERO = 0, OR_J_OHMIC_EXP = 1, OR_J_DEBYE = 2, OR_J_SUPEROHMIC_GAUSS = 3 };
enum { OR_READING_STRANG = 0, OR_READING_AS_PRINTED = 1 };

typedef struct {
    int32_t M;             /* Hilbert-space dimension of the OQS      */
    const double *s;       /* [M] eigenvalues of the system coupling coordinate      */
    const double *H;       /* [M*M*2] row-major complex (re,im) Hamiltonian            P:192 Eq.8 */
    const double *rho0;    /* [M*M*2] row-major complex initial density matrix         P:192 Eq.8 */
    int32_t kind;          /* OR_J_*                                                   P:155 Eq.3 */
    double coupling;       /* xi (Ohmic/Debye) or A (super-Ohmic Gaussian, Eq. 21)               */
    double omega_c;        /* cutoff frequency                                                    */
    double kT;             /* temperature k_B T (0 => coth = 1)                        P:163 Eq.4 */
    double dt;             /* time step Delta t      */
    int64_t n_steps;       /* N_t: last time index      */
    int32_t L;             /* Delta k_max: memory length                               P:190 Eq.8 */
    const double *G_in;    /* optional [(2L+3)*2]: G(m dt/2), m=0..2L+2, replaces the
                              quadrature (the paper's "alpha(t) given" input)            */
    int32_t reading;       /* OR_READING_STRANG (default) or OR_READING_AS_PRINTED              */
    const double *H_t;     /* optional [n_steps][M*M*2]: time-dependent Hamiltonian, H_t[k-1] acts on
                              the interval (t_{k-1}, t_k] of step k (the driven model of Sec. III,
                              Omega(t) of P:288); NULL => H on every interval        */
    double filter_theta;   /* path filtering (Sim's on-the-fly filtered propagator, cited P:99-103,
                              invited P:265-271; reading C.3-15): after every
                              propagation step k >= 1 the entries of A_k with |A|^2 < theta^2 are set
                              to 0.  0 => no filtering (bit-identical to the plain run)             */
    int64_t *kept;         /* optional [n_steps + 1]: kept[k] = nonzero entries of A_k after filtering
                              (k = 0 .. the last propagated step; rho(t_n) needs A_{n-1} only)      */
} or_problem;

/* G(tau) = int_0^tau dt' int_0^t' dt'' alpha(t'-t'')  (Eq. 4 integrated twice). */
int or_G(const or_problem *p, double tau, double *re, double *im);
/* G(m dt/2) for m = 0..n_m-1 (complex interleaved). Uses G_in if present. */
int or_G_table(const or_problem *p, int32_t n_m, double *out);
/* eta between time points t >= tp for a run whose final point is kfinal
   (kfinal < 0 => "interior" windows for both, i.e. no terminal point).   Eqs. 10-16 */
int or_eta_pair(const or_problem *p, int64_t t, int64_t tp, int64_t kfinal, double *re, double *im);
/* U = exp(-i H dt) via the oracle's own real Jacobi eigensolver (Eq. 8). */
int or_propagator(const or_problem *p, double *U_out);
/* Literal sum over all Feynman paths (Eq. 8 with Eq. 9, sliding-window truncation).
   Writes rho(t_{n_steps}) [M*M*2]. Guard: (M^2)^(n_steps+1) <= 1e7. */
int or_brute_force(const or_problem *p, double *rho_out);
/* Plain iterative tensor propagation (Makri-Makarov).  rho_out[n_out][M][M] complex for the
   requested step indices (sorted ascending, each in [0, n_steps]).  nthreads<=0 => OpenMP
   default.  timings[4] (optional): setup_s, growth_s, slide_s, n_slide_steps. */
int or_run(const or_problem *p, const int64_t *out_steps, int64_t n_out, double *rho_out,
           int32_t nthreads, double *timings);
/* Paper's primary memory cost PMC = 64 M^(2(L+1)) bytes (Eqs. 18-19). */
double or_pmc_bytes(int32_t M, int32_t L);
const char *or_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
