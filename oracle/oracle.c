/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the QUAPI tensor
 * propagator (N. S. Dattani, arXiv 1205.6872).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs.  It shares no code with the
 * CUDA path (paper_1205_6872_b200/) and never calls it.
 *
 * What it computes (citations: P:<line> of /root/reference/PAPER.md):
 *   rho(t_N) of Eq. 8 with the discretised influence functional
 *   Eq. 9, eta coefficients Eqs. 10-16, bath response
 *   Eq. 4 and spectral densities Eq. 3 / Eq. 21.
 *   Readings where the paper is garbled/ambiguous are DESIGN.md §3 (C.3-n).
 *
 * Two evaluations of the same discrete result:
 *   or_brute_force : literal sum over all Feynman paths of Eq. 8 (tiny sizes).
 *   or_run         : plain iterative tensor propagation in a physically shifted
 *                    layout (newest point least significant), copying the tensor
 *                    every step; readout of rho(t_k) from A_{k-1}.
 * Both get eta from G(tau) = int_0^tau int_0^t' alpha(t'-t'') dt'' dt' via the
 * four-corner rule of the window integrals.  G comes from an adaptive
 * Gauss-Kronrod (7,15) quadrature in omega of the twice-integrated Eq. 4.
 *
 * Pins (tests/test_oracle_*.py): G closed forms (Ohmic T=0 log form, Ohmic
 * finite-T log-Gamma form, Debye Matsubara form, 30-digit mpmath), constant-
 * alpha window areas, brute force == iterative, trace == tr rho0 exactly,
 * Hermiticity, zero coupling == U^k rho0 U^+k, pure-dephasing closed form,
 * Rabi sin^2, PMC column of Table I.
 *
 * Build: gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fcx-fortran-rules -fPIC -shared
 */
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <omp.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef double complex cplx;

static __thread char g_err[256];
static int fail(const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return 1;
}
const char *or_last_error(void) { return g_err; }

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ------------------------------------------------------------------------- */
/* Spectral densities J(omega), omega > 0.  Eq. 3, Eq. 21 (P:291,  */
/* reading C.3-5: exp(-(w/wc)^2)), Ohmic / Debye forms of reading C.3-9.       */
/* ------------------------------------------------------------------------- */
static double J_eval(const or_problem *p, double w) {
    const double xi = p->coupling, wc = p->omega_c;
    switch (p->kind) {
    case OR_J_OHMIC_EXP: return 0.5 * M_PI * xi * w * exp(-w / wc);
    case OR_J_DEBYE: return 0.5 * M_PI * xi * w * wc * wc / (w * w + wc * wc);
    case OR_J_SUPEROHMIC_GAUSS: return xi * w * w * w * exp(-(w / wc) * (w / wc));
    default: return 0.0;
    }
}

/* x - sin(x) without cancellation for small x (Taylor series). */
static double x_minus_sin(double x) {
    if (fabs(x) >= 0.5) return x - sin(x);
    double term = x * x * x / 6.0, sum = 0.0;
    for (int n = 1; n < 40; ++n) {
        sum += term;
        term *= -x * x / ((2.0 * n + 2.0) * (2.0 * n + 3.0));
        if (fabs(term) < 1e-20 * fabs(sum)) break;
    }
    return sum;
}

/* Integrand of G(tau):  (1/pi) J(w)/w^2 [ coth(w/2kT)(1 - cos w tau) - i (w tau - sin w tau) ].
   This is Eq. 4 integrated over t'' in [0,t'] and t' in [0,tau]:
   int_0^tau (tau-u) cos(wu) du = (1-cos w tau)/w^2, int_0^tau (tau-u) sin(wu) du = (w tau - sin w tau)/w^2. */
static void G_integrand(const or_problem *p, double tau, double w, double *fr, double *fi) {
    double j = J_eval(p, w) / (w * w) / M_PI;
    double ct = 1.0;
    if (p->kT > 0.0) {
        double y = 0.5 * w / p->kT;
        ct = (y > 40.0) ? 1.0 : 1.0 / tanh(y);
    }
    double h = sin(0.5 * w * tau);
    *fr = j * ct * 2.0 * h * h; /* 1 - cos = 2 sin^2(x/2) */
    *fi = -j * x_minus_sin(w * tau);
}

/* Gauss-Kronrod (7,15) nodes/weights on [-1,1] (standard QUADPACK QK15 values). */
static const double xgk[8] = {0.991455371120812639206854697526329, 0.949107912342758524526189684047851,
                              0.864864423359769072789712788640926, 0.741531185599394439863864773280788,
                              0.586087235467691130294144845693013, 0.405845151377397166906606412076961,
                              0.207784955007898467600689403773245, 0.000000000000000000000000000000000};
static const double wgk[8] = {0.022935322010529224963732008058970, 0.063092092629978553290700663189204,
                              0.104790010322250183839876322541518, 0.140653259715525918745189590510238,
                              0.169004726639267902826583426598550, 0.190350578064785409913256402421014,
                              0.204432940075298892414161999234649, 0.209482141084727828012999174891714};
static const double wg[4] = {0.129484966168869693270611432679082, 0.279705391489276667901467771423780,
                             0.381830050505118944950369775488975, 0.417959183673469387755102040816327};

/* QUADPACK-style error estimate of one real component (QK15). */
static double qk_err(double K, double Gs, double resabs, double resasc) {
    double e = fabs(K - Gs);
    if (resasc != 0.0 && e != 0.0) e = resasc * fmin(1.0, pow(200.0 * e / resasc, 1.5));
    if (resabs > 1e-290) e = fmax(50.0 * 2.220446049250313e-16 * resabs, e);
    return e;
}

static void gk15(const or_problem *p, double tau, double a, double b, double *kr, double *ki, double *err,
                 double *floor_) {
    double c = 0.5 * (a + b), h = 0.5 * (b - a);
    double fr[15], fi[15], x[15], wk[15];
    int n = 0;
    x[n] = c; wk[n++] = wgk[7];
    for (int j = 0; j < 7; ++j) { x[n] = c - h * xgk[j]; wk[n++] = wgk[j]; x[n] = c + h * xgk[j]; wk[n++] = wgk[j]; }
    for (int q = 0; q < 15; ++q) G_integrand(p, tau, x[q], &fr[q], &fi[q]);
    double Kr = 0, Ki = 0, Gr = wg[3] * fr[0], Gi = wg[3] * fi[0], Ar = 0, Ai = 0;
    for (int q = 0; q < 15; ++q) { Kr += wk[q] * fr[q]; Ki += wk[q] * fi[q]; Ar += wk[q] * fabs(fr[q]); Ai += wk[q] * fabs(fi[q]); }
    for (int j = 1; j < 7; j += 2) { /* Gauss-7 nodes are the odd Kronrod abscissae */
        Gr += wg[j / 2] * (fr[1 + 2 * j] + fr[2 + 2 * j]);
        Gi += wg[j / 2] * (fi[1 + 2 * j] + fi[2 + 2 * j]);
    }
    double mr = 0.5 * Kr, mi = 0.5 * Ki, Sr = 0, Si = 0; /* mean over [-1,1] is K/2 */
    for (int q = 0; q < 15; ++q) { Sr += wk[q] * fabs(fr[q] - mr); Si += wk[q] * fabs(fi[q] - mi); }
    *kr = Kr * h; *ki = Ki * h;
    *err = qk_err(Kr * h, Gr * h, Ar * h, Sr * h) + qk_err(Ki * h, Gi * h, Ai * h, Si * h);
    *floor_ = 2.0 * 50.0 * 2.220446049250313e-16 * (Ar + Ai) * h; /* roundoff-limited: cannot do better */
}

/* Neumaier-compensated running sum (the panel sums are long; keeps G at roundoff level). */
typedef struct { double s, c; } ksum;
static void kadd(ksum *k, double x) {
    double t = k->s + x;
    if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x; else k->c += (x - t) + k->s;
    k->s = t;
}

static int adapt(const or_problem *p, double tau, double a, double b, double tol, int depth, ksum *r,
                 ksum *i) {
    double kr, ki, e, fl;
    gk15(p, tau, a, b, &kr, &ki, &e, &fl);
    int ok = (e <= tol) || (e <= 1.01 * fl);
    if (ok || depth >= 30) {
        kadd(r, kr); kadd(i, ki);
        return ok ? 0 : 1;
    }
    double m = 0.5 * (a + b);
    int bad = adapt(p, tau, a, m, 0.5 * tol, depth + 1, r, i);
    bad |= adapt(p, tau, m, b, 0.5 * tol, depth + 1, r, i);
    return bad;
}

/* Debye tail beyond Omega where coth = 1 to double precision:
   (1/pi) int_Omega^inf J/w^2 (1 - i w tau - e^{-i w tau}) dw,  J/w^2/pi = (xi/2) c^2 / (w (w^2+c^2)).
     int_Omega^inf c^2 dw/(w(w^2+c^2))   = (1/2) log(1 + c^2/Omega^2)
     int_Omega^inf c^2 tau dw/(w^2+c^2)  = c tau atan(c/Omega)
     int_Omega^inf g(w) e^{-iw tau} dw   = e^{-i Omega tau} sum_n g^(n)(Omega)/(i tau)^(n+1)
   (repeated integration by parts), g = 1/(w(w^2+c^2)) = sum_m (-c^2)^m w^-(2m+3). */
static cplx debye_tail(const or_problem *p, double tau, double Om) {
    const double c = p->omega_c, xi = p->coupling;
    cplx nonosc = 0.5 * log1p((c / Om) * (c / Om)) - I * c * tau * atan(c / Om);
    cplx sum = 0.0, itau_pow = I * tau; /* (i tau)^(n+1) */
    double prev = INFINITY;
    for (int n = 0; n < 60; ++n) {
        /* g^(n)(Omega) = sum_m (-c^2)^m (-1)^n (2m+3)_n Omega^-(2m+3+n) */
        double gn = 0.0, cm = 1.0;
        for (int m = 0; m < 12; ++m) {
            int k = 2 * m + 3;
            double rising = 1.0;
            for (int q = 0; q < n; ++q) rising *= (double)(k + q);
            double t = cm * rising * pow(Om, -(double)(k + n));
            gn += t;
            cm *= -c * c;
            if (fabs(t) < 1e-22 * fabs(gn)) break;
        }
        if (n % 2 == 1) gn = -gn;
        cplx term = gn / itau_pow;
        double mag = cabs(term);
        if (mag > prev) break; /* asymptotic series: stop before divergence */
        sum += term;
        prev = mag;
        if (mag < 1e-24 * cabs(sum)) break;
        itau_pow *= I * tau;
    }
    cplx osc = cexp(-I * Om * tau) * sum;
    return 0.5 * xi * (nonosc - c * c * osc);
}

int or_G(const or_problem *p, double tau, double *re, double *im) {
    *re = 0.0; *im = 0.0;
    if (p->kind == OR_J_ZERO || tau == 0.0) return 0;
    if (tau < 0.0) { /* G(-t) = conj G(t) since alpha(-t) = conj alpha(t) */
        int r = or_G(p, -tau, re, im);
        *im = -*im;
        return r;
    }
    const double wc = p->omega_c;
    double Om;
    switch (p->kind) {
    case OR_J_OHMIC_EXP: Om = 60.0 * wc; break;      /* e^-60 ~ 1e-26 tail */
    case OR_J_SUPEROHMIC_GAUSS: Om = 12.0 * wc; break; /* e^-144 tail */
    default: /* Debye: analytic tail added below.  Its asymptotic series in 1/(Omega tau) needs
                Omega tau >= 400 to reach rounding level (at Omega tau ~ 13 it stalls near 1e-8) */
        Om = fmax(fmax(200.0 * wc, 80.0 * p->kT), 400.0 / tau); break;
    }
    /* panels no wider than a quarter oscillation period and wc/4 */
    double hpan = fmin(0.25 * wc, 0.5 * M_PI / tau);
    long npan = (long)ceil(Om / hpan);
    ksum r = {0, 0}, i = {0, 0};
    int bad = 0;
    for (long k = 0; k < npan; ++k) {
        double a = Om * (double)k / (double)npan, b = Om * (double)(k + 1) / (double)npan;
        bad |= adapt(p, tau, a, b, 1e-17 / (double)npan + 1e-300, 0, &r, &i);
    }
    if (p->kind == OR_J_DEBYE) {
        cplx t = debye_tail(p, tau, Om);
        kadd(&r, creal(t)); kadd(&i, cimag(t));
    }
    *re = r.s + r.c; *im = i.s + i.c;
    if (bad) return fail("G quadrature did not converge");
    return 0;
}

int or_G_table(const or_problem *p, int32_t n_m, double *out) {
    if (p->G_in) {
        if (n_m > 2 * p->L + 3) return fail("G_table: G_in holds only 2L+3 entries");
        memcpy(out, p->G_in, sizeof(double) * 2 * (size_t)n_m);
        return 0;
    }
    for (int32_t m = 0; m < n_m; ++m)
        if (or_G(p, 0.5 * p->dt * m, &out[2 * m], &out[2 * m + 1])) return 1;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* eta from G (Eqs. 10-16).  Window of time point t in a run ending at kf:    */
/*   reading C.3-1 (Strang): t=0 -> [0,1/2], t=kf -> [kf-1/2,kf], else [t-1/2,t+1/2]  */
/*   as printed:             t=0 -> [0,1/2], t=kf -> [kf-1/2,kf], else [t,t+1]         */
/* (units of dt).  Self term (Eqs. 11,13,14; reading C.3-2 for Eq. 13) = G(width).      */
/* Pair (t > tp): int_{a1}^{a2} int_{b1}^{b2} alpha(t'-t'') = G(a2-b1)+G(a1-b2)-G(a1-b1)-G(a2-b2)  */
/* since G'' = alpha.  All window ends are multiples of 1/2 -> table index 2x.  */
/* ------------------------------------------------------------------------- */
typedef struct { const double *G; int32_t nG; int reading; } eta_ctx;

static cplx Gx(const eta_ctx *c, int64_t twice_x) { /* G(x dt), x = twice_x/2, G(-x)=conj G(x) */
    int64_t m = twice_x < 0 ? -twice_x : twice_x;
    if (m >= c->nG) { fprintf(stderr, "oracle: G index %lld out of table\n", (long long)m); abort(); }
    cplx g = c->G[2 * m] + I * c->G[2 * m + 1];
    return twice_x < 0 ? conj(g) : g;
}

static void window2(const eta_ctx *c, int64_t t, int64_t kf, int64_t *a, int64_t *b) { /* in half steps */
    if (t == 0) { *a = 0; *b = 1; return; }
    if (t == kf) { *a = 2 * kf - 1; *b = 2 * kf; return; }
    if (c->reading == OR_READING_AS_PRINTED) { *a = 2 * t; *b = 2 * t + 2; }
    else { *a = 2 * t - 1; *b = 2 * t + 1; }
}

static cplx eta_of(const eta_ctx *c, int64_t t, int64_t tp, int64_t kf) {
    int64_t a1, a2, b1, b2;
    window2(c, t, kf, &a1, &a2);
    if (t == tp) return Gx(c, a2 - a1);
    window2(c, tp, kf, &b1, &b2);
    return Gx(c, a2 - b1) + Gx(c, a1 - b2) - Gx(c, a1 - b1) - Gx(c, a2 - b2);
}

static int build_G(const or_problem *p, double **G, int32_t *nG) {
    *nG = 2 * p->L + 3;
    *G = (double *)malloc(sizeof(double) * 2 * (size_t)(*nG));
    if (!*G) return fail("oom");
    if (or_G_table(p, *nG, *G)) { free(*G); return 1; }
    return 0;
}

int or_eta_pair(const or_problem *p, int64_t t, int64_t tp, int64_t kfinal, double *re, double *im) {
    double *G; int32_t nG;
    if (t < tp) return fail("eta_pair: need t >= tp");
    if (t - tp > p->L) return fail("eta_pair: lag exceeds L");
    /* G args reach (t-tp)+1; the table covers lags up to L */
    if (build_G(p, &G, &nG)) return 1;
    eta_ctx c = {G, nG, p->reading};
    cplx e = eta_of(&c, t, tp, kfinal < 0 ? INT64_MAX : kfinal);
    *re = creal(e); *im = cimag(e);
    free(G);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Propagator U = exp(-i H dt) (Eq. 8) via cyclic Jacobi on the real   */
/* symmetric embedding H_R = [[A,-B],[B,A]] of H = A + iB:                    */
/* cos(H dt) and sin(H dt) are read off the blocks of cos/sin(H_R dt).         */
/* ------------------------------------------------------------------------- */
static void jacobi_sym(int n, double *a /* n*n, destroyed */, double *v /* n*n eigvecs in columns */,
                       double *ev) {
    for (int i = 0; i < n * n; ++i) v[i] = 0.0;
    for (int i = 0; i < n; ++i) v[i * n + i] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) off += a[i * n + j] * a[i * n + j];
        if (off < 1e-300) break;
        for (int pq = 0; pq < n; ++pq)
            for (int q = pq + 1; q < n; ++q) {
                double apq = a[pq * n + q];
                double app = a[pq * n + pq], aqq = a[q * n + q];
                /* negligible off-diagonal element: zero it instead of rotating (rotations inside a
                   degenerate eigenspace after convergence only accumulate roundoff) */
                if (fabs(app) + 100.0 * fabs(apq) == fabs(app) && fabs(aqq) + 100.0 * fabs(apq) == fabs(aqq)) {
                    a[pq * n + q] = a[q * n + pq] = 0.0;
                    continue;
                }
                double theta = 0.5 * (aqq - app) / apq;
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
                for (int k = 0; k < n; ++k) { /* columns pq, q */
                    double akp = a[k * n + pq], akq = a[k * n + q];
                    a[k * n + pq] = cs * akp - sn * akq;
                    a[k * n + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < n; ++k) { /* rows pq, q */
                    double apk = a[pq * n + k], aqk = a[q * n + k];
                    a[pq * n + k] = cs * apk - sn * aqk;
                    a[q * n + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    double vkp = v[k * n + pq], vkq = v[k * n + q];
                    v[k * n + pq] = cs * vkp - sn * vkq;
                    v[k * n + q] = sn * vkp + cs * vkq;
                }
            }
    }
    for (int i = 0; i < n; ++i) ev[i] = a[i * n + i];
}

int or_propagator(const or_problem *p, double *U_out) {
    const int M = p->M, n = 2 * M;
    double *a = calloc((size_t)n * n, sizeof(double)), *v = calloc((size_t)n * n, sizeof(double));
    double *ev = calloc((size_t)n, sizeof(double));
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            double A = p->H[2 * (i * M + j)], B = p->H[2 * (i * M + j) + 1];
            a[i * n + j] = A; a[i * n + (j + M)] = -B;
            a[(i + M) * n + j] = B; a[(i + M) * n + (j + M)] = A;
        }
    jacobi_sym(n, a, v, ev);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            /* f(H_R) = V f(Lambda) V^T ; Re f(H) = block(0,0), Im f(H) = block(1,0) */
            double cr = 0, ci = 0, sr = 0, si = 0;
            for (int k = 0; k < n; ++k) {
                double c = cos(ev[k] * p->dt), s = sin(ev[k] * p->dt);
                cr += v[i * n + k] * c * v[j * n + k];
                ci += v[(i + M) * n + k] * c * v[j * n + k];
                sr += v[i * n + k] * s * v[j * n + k];
                si += v[(i + M) * n + k] * s * v[j * n + k];
            }
            /* U = cos(H dt) - i sin(H dt) */
            U_out[2 * (i * M + j)] = cr + si;
            U_out[2 * (i * M + j) + 1] = ci - sr;
        }
    free(a); free(v); free(ev);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Shared problem scaffolding                                                 */
/* ------------------------------------------------------------------------- */
typedef struct {
    int M, N;      /* N = M^2 pair states sigma = a*M + b  */
    double *sp, *sm; /* s+(sigma) = s[a], s-(sigma) = s[b]          */
    cplx *K;       /* K[sig' * N + sig] = U[a',a] conj(U[b',b])     (Eq. 8 propagator pair) */
    cplx *rho0;    /* [N]                                            */
    double *G; int32_t nG;
} ctx_t;

static void ctx_free(ctx_t *c) { free(c->sp); free(c->sm); free(c->K); free(c->rho0); free(c->G); }

/* K[sig' * N + sig] = U[a',a] conj(U[b',b]) with U = exp(-i H dt) for the Hamiltonian H (Eq. 8):
   <s+_{k+1}|e^{-iH dt}|s+_k> <s-_k|e^{+iH dt}|s-_{k+1}>. */
static void build_K(const or_problem *p, const double *H, cplx *K) {
    const int M = p->M, N = M * M;
    or_problem q = *p;
    q.H = H;
    double *U = malloc(sizeof(double) * 2 * M * M);
    or_propagator(&q, U);
    for (int a1 = 0; a1 < M; ++a1)
        for (int b1 = 0; b1 < M; ++b1)
            for (int a = 0; a < M; ++a)
                for (int b = 0; b < M; ++b) {
                    cplx ua = U[2 * (a1 * M + a)] + I * U[2 * (a1 * M + a) + 1];
                    cplx ub = U[2 * (b1 * M + b)] + I * U[2 * (b1 * M + b) + 1];
                    K[(a1 * M + b1) * N + (a * M + b)] = ua * conj(ub);
                }
    free(U);
}

/* propagator pair of step k (interval (t_{k-1}, t_k]): the time-dependent H_t[k-1] if given, else c->K */
static const cplx *step_K(const or_problem *p, const ctx_t *c, int64_t k, cplx *buf) {
    if (!p->H_t) return c->K;
    build_K(p, p->H_t + 2 * (size_t)(k - 1) * c->M * c->M, buf);
    return buf;
}

static int validate(const or_problem *p) {
    if (p->M < 1 || p->M > 8 || !p->s || !p->H || !p->rho0) return fail("config: need 1<=M<=8 and s/H/rho0");
    if (p->L < 1 || p->L > 60) return fail("config: L (Delta k_max) must be in [1,60]");
    if (p->n_steps < 0) return fail("config: n_steps < 0");
    if (!(p->dt > 0)) return fail("config: dt must be > 0");
    const int M = p->M;
    double tr_re = 0, tr_im = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j) {
            double hr = p->H[2 * (i * M + j)], hi = p->H[2 * (i * M + j) + 1];
            double gr = p->H[2 * (j * M + i)], gi = p->H[2 * (j * M + i) + 1];
            if (fabs(hr - gr) > 1e-12 || fabs(hi + gi) > 1e-12) return fail("config: H not Hermitian");
            double rr = p->rho0[2 * (i * M + j)], ri = p->rho0[2 * (i * M + j) + 1];
            double qr = p->rho0[2 * (j * M + i)], qi = p->rho0[2 * (j * M + i) + 1];
            if (fabs(rr - qr) > 1e-12 || fabs(ri + qi) > 1e-12) return fail("config: rho0 not Hermitian");
        }
    for (int i = 0; i < M; ++i) { tr_re += p->rho0[2 * (i * M + i)]; tr_im += p->rho0[2 * (i * M + i) + 1]; }
    if (p->H_t)
        for (int64_t k = 0; k < p->n_steps; ++k)
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) {
                    const double *h = p->H_t + 2 * (k * M * M);
                    if (fabs(h[2 * (i * M + j)] - h[2 * (j * M + i)]) > 1e-12 ||
                        fabs(h[2 * (i * M + j) + 1] + h[2 * (j * M + i) + 1]) > 1e-12)
                        return fail("config: H_t not Hermitian");
                }
    if (fabs(tr_re - 1.0) > 1e-12 || fabs(tr_im) > 1e-12) return fail("config: trace(rho0) != 1");
    return 0;
}

static int ctx_init(const or_problem *p, ctx_t *c) {
    memset(c, 0, sizeof *c);
    if (validate(p)) return 1;
    const int M = p->M, N = M * M;
    c->M = M; c->N = N;
    c->sp = malloc(sizeof(double) * N); c->sm = malloc(sizeof(double) * N);
    c->K = malloc(sizeof(cplx) * N * N); c->rho0 = malloc(sizeof(cplx) * N);
    for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b) {
            int sg = a * M + b;
            c->sp[sg] = p->s[a]; c->sm[sg] = p->s[b];
            c->rho0[sg] = p->rho0[2 * sg] + I * p->rho0[2 * sg + 1];
        }
    build_K(p, p->H, c->K);
    if (build_G(p, &c->G, &c->nG)) { ctx_free(c); return 1; }
    return 0;
}

/* Eq. 9 summand for the (later sigma, earlier sigma') pair; Delta s belongs to the later point
   (reading C.3-4):  I = exp( -(s+ - s-)(sigma) * ( eta s+(sigma') - conj(eta) s-(sigma') ) ). */
static cplx infl(const ctx_t *c, int sg, int sgp, cplx eta) {
    double ds = c->sp[sg] - c->sm[sg];
    return cexp(-ds * (eta * c->sp[sgp] - conj(eta) * c->sm[sgp]));
}

double or_pmc_bytes(int32_t M, int32_t L) { return 64.0 * pow((double)M, 2.0 * (L + 1)); }

/* ------------------------------------------------------------------------- */
/* Brute force: literal Eq. 8 sum over paths sigma_0..sigma_N,      */
/* exponent of Eq. 9 with k' >= k - L (reading C.3-3).                          */
/* ------------------------------------------------------------------------- */
int or_brute_force(const or_problem *p, double *rho_out) {
    ctx_t c;
    if (ctx_init(p, &c)) return 1;
    const int N = c.N, M = c.M;
    const int64_t Nt = p->n_steps;
    if (Nt == 0) { /* reading C.3-8: rho(0) = rho0 exactly */
        for (int sg = 0; sg < N; ++sg) { rho_out[2 * sg] = creal(c.rho0[sg]); rho_out[2 * sg + 1] = cimag(c.rho0[sg]); }
        ctx_free(&c);
        return 0;
    }
    double npaths_d = pow((double)N, (double)(Nt + 1));
    if (npaths_d > 1e7) { ctx_free(&c); return fail("brute force guard: N^(Nt+1) > 1e7"); }
    int64_t npaths = (int64_t)llround(npaths_d);
    eta_ctx ec = {c.G, c.nG, p->reading};
    /* eta for every coupled pair (t, tp) of this run */
    int64_t W = Nt + 1;
    cplx *eta = calloc((size_t)(W * W), sizeof(cplx));
    for (int64_t t = 0; t <= Nt; ++t)
        for (int64_t tp = (t - p->L > 0 ? t - p->L : 0); tp <= t; ++tp) eta[t * W + tp] = eta_of(&ec, t, tp, Nt);
    cplx *acc = calloc((size_t)N, sizeof(cplx));
    int *path = malloc(sizeof(int) * (size_t)W);
    /* Kt[t]: propagator pair of the interval (t_t, t_{t+1}] = step t+1 */
    cplx *Kt = malloc(sizeof(cplx) * (size_t)Nt * N * N);
    for (int64_t t = 0; t < Nt; ++t) {
        cplx *buf = Kt + (size_t)t * N * N;
        const cplx *k = step_K(p, &c, t + 1, buf);
        if (k != buf) memcpy(buf, k, sizeof(cplx) * N * N);
    }
    for (int64_t x = 0; x < npaths; ++x) {
        int64_t r = x;
        for (int64_t t = 0; t <= Nt; ++t) { path[t] = (int)(r % N); r /= N; }
        cplx w = c.rho0[path[0]];
        for (int64_t t = 0; t < Nt; ++t) w *= Kt[(size_t)t * N * N + path[t + 1] * N + path[t]];
        if (w == 0) continue;
        cplx phase = 0;
        for (int64_t t = 0; t <= Nt; ++t)
            for (int64_t tp = (t - p->L > 0 ? t - p->L : 0); tp <= t; ++tp) {
                int s1 = path[t], s0 = path[tp];
                double ds = c.sp[s1] - c.sm[s1];
                cplx e = eta[t * W + tp];
                phase += -ds * (e * c.sp[s0] - conj(e) * c.sm[s0]);
            }
        acc[path[Nt]] += w * cexp(phase);
    }
    for (int sg = 0; sg < N; ++sg) { rho_out[2 * sg] = creal(acc[sg]); rho_out[2 * sg + 1] = cimag(acc[sg]); }
    (void)M;
    free(eta); free(acc); free(path); free(Kt); ctx_free(&c);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Iterative tensor propagation (Makri-Makarov), oracle layout:       */
/* A_k holds w_k = min(k+1, L) points sigma_{k-w+1..k};                         */
/* flat index x = sum_i sigma_{k-i} N^i  (i = lag from the newest point).      */
/* ------------------------------------------------------------------------- */
static int64_t ipow(int64_t b, int e) { int64_t r = 1; while (e-- > 0) r *= b; return r; }

/* factor tables for the step that appends point k:  tab[j][sg*N + sgp] = I(sg, sgp; eta(k, k-j))
   with point k interior ("prop", kf = +inf) or terminal ("term", kf = k). */
static void step_tables(const ctx_t *c, const eta_ctx *ec, int64_t k, int L, int64_t kf, cplx *tab) {
    const int N = c->N;
    int jmax = (int)(k < L ? k : L);
    for (int j = 0; j <= jmax; ++j) {
        cplx e = eta_of(ec, k, k - j, kf);
        for (int sg = 0; sg < N; ++sg)
            for (int sgp = 0; sgp < N; ++sgp) tab[(size_t)j * N * N + sg * N + sgp] = infl(c, sg, sgp, e);
    }
}

/* pairwise (tree) sum of n terms -- fixed order independent of threading */
static cplx pairwise(const cplx *v, int64_t n) {
    if (n <= 8) { cplx s = 0; for (int64_t i = 0; i < n; ++i) s += v[i]; return s; }
    int64_t h = n / 2;
    return pairwise(v, h) + pairwise(v + h, n - h);
}

/* rho_k(sg_k) = sum_x K(sg_k, sg_{k-1}) prod_{j=0}^{min(k,L)} I_term(sg_k, sg_{k-j}) A_{k-1}[x]   (k >= 1) */
static void readout(const ctx_t *c, const cplx *K, const cplx *A, int w_old, const cplx *tab_term, int64_t k, int L,
                    cplx *rho) {
    const int N = c->N;
    const int64_t n = ipow(N, w_old), BLK = 4096;
    const int64_t nblk = (n + BLK - 1) / BLK;
    int jmax = (int)(k < L ? k : L);
    cplx *part = malloc(sizeof(cplx) * (size_t)(nblk * N));
#pragma omp parallel
    {
        cplx *buf = malloc(sizeof(cplx) * BLK);
        int *dig = malloc(sizeof(int) * (size_t)(w_old + 1));
#pragma omp for schedule(static)
        for (int64_t b = 0; b < nblk; ++b) {
            int64_t lo = b * BLK, hi = lo + BLK < n ? lo + BLK : n;
            for (int sk = 0; sk < N; ++sk) {
                for (int64_t x = lo; x < hi; ++x) {
                    int64_t r = x;
                    for (int i = 0; i < w_old; ++i) { dig[i] = (int)(r % N); r /= N; } /* dig[i] = sigma_{k-1-i} */
                    cplx f = K[sk * N + dig[0]] * tab_term[sk * N + sk];
                    for (int j = 1; j <= jmax; ++j) f *= tab_term[(size_t)j * N * N + sk * N + dig[j - 1]];
                    buf[x - lo] = f * A[x];
                }
                part[b * N + sk] = pairwise(buf, hi - lo);
            }
        }
        free(buf); free(dig);
    }
    cplx *col = malloc(sizeof(cplx) * (size_t)nblk);
    for (int sk = 0; sk < N; ++sk) {
        for (int64_t b = 0; b < nblk; ++b) col[b] = part[b * N + sk];
        rho[sk] = pairwise(col, nblk);
    }
    free(col); free(part);
}

int or_run(const or_problem *p, const int64_t *out_steps, int64_t n_out, double *rho_out, int32_t nthreads,
           double *timings) {
    double t0 = now_s();
    ctx_t c;
    if (ctx_init(p, &c)) return 1;
    if (nthreads > 0) omp_set_num_threads(nthreads);
    const int N = c.N, L = p->L;
    const int64_t Nt = p->n_steps;
    for (int64_t o = 0; o < n_out; ++o) {
        if (out_steps[o] < 0 || out_steps[o] > Nt || (o > 0 && out_steps[o] <= out_steps[o - 1])) {
            ctx_free(&c);
            return fail("out_steps must be sorted, unique, within [0, n_steps]");
        }
    }
    const int64_t D = ipow(N, L);
    cplx *A = calloc((size_t)D, sizeof(cplx)), *B = calloc((size_t)D, sizeof(cplx));
    cplx *tabp = malloc(sizeof(cplx) * (size_t)(L + 1) * N * N), *tabt = malloc(sizeof(cplx) * (size_t)(L + 1) * N * N);
    if (!A || !B || !tabp || !tabt) { free(A); free(B); free(tabp); free(tabt); ctx_free(&c); return fail("capacity: oracle out of host memory"); }
    eta_ctx ec = {c.G, c.nG, p->reading};
    int64_t o = 0;
    /* k = 0 readout: rho0 exactly (reading C.3-8) */
    if (n_out > 0 && out_steps[0] == 0) {
        for (int sg = 0; sg < N; ++sg) { rho_out[2 * sg] = creal(c.rho0[sg]); rho_out[2 * sg + 1] = cimag(c.rho0[sg]); }
        o = 1;
    }
    /* A_0(sigma_0) = rho0(sigma_0) I(sigma_0, sigma_0; eta_00),  eta_00 = G(1/2) (Eq. 13, reading C.3-2) */
    for (int sg = 0; sg < N; ++sg) A[sg] = c.rho0[sg] * infl(&c, sg, sg, eta_of(&ec, 0, 0, INT64_MAX));
    if (p->kept) {
        int64_t nz = 0;
        for (int sg = 0; sg < N; ++sg) nz += (A[sg] != 0);
        p->kept[0] = nz;
    }
    double t_setup = now_s() - t0, t_grow = 0.0, t_slide = 0.0;
    int64_t n_slide = 0;
    int w_old = 1;
    cplx rho[64];
    cplx *Kbuf = malloc(sizeof(cplx) * (size_t)N * N);
    for (int64_t k = 1; k <= Nt; ++k) {
        double ts = now_s();
        const cplx *Kk = step_K(p, &c, k, Kbuf); /* propagator pair of step k */
        /* readout of rho(t_k) from A_{k-1} (terminal classes) */
        if (o < n_out && out_steps[o] == k) {
            step_tables(&c, &ec, k, L, k, tabt);
            readout(&c, Kk, A, w_old, tabt, k, L, rho);
            for (int sg = 0; sg < N; ++sg) {
                rho_out[2 * (o * N + sg)] = creal(rho[sg]);
                rho_out[2 * (o * N + sg) + 1] = cimag(rho[sg]);
            }
            ++o;
        }
        if (o >= n_out) break; /* nothing further requested */
        /* propagate: A_k = sum_{sigma_{k-L}} K I ... A_{k-1}  (prop classes, point k interior) */
        step_tables(&c, &ec, k, L, INT64_MAX, tabp);
        const int w_new = (int)(k + 1 < L ? k + 1 : L);
        const int contract = (k >= L);
        const int64_t n_new = ipow(N, w_new), top = ipow(N, L - 1);
        const int jmax = (int)(k < L ? k : L);
#pragma omp parallel
        {
            int dig[64];
#pragma omp for schedule(static)
            for (int64_t y = 0; y < n_new; ++y) {
                int64_t r = y;
                for (int i = 0; i < w_new; ++i) { dig[i] = (int)(r % N); r /= N; } /* dig[i] = sigma_{k-i} */
                const int sk = dig[0];
                /* influence factors whose partner point is kept in A_k (lags 0..jin) */
                cplx f = 1.0;
                int jin = contract ? L - 1 : jmax;
                for (int j = 0; j <= jin; ++j) f *= tabp[(size_t)j * N * N + sk * N + dig[j]];
                if (!contract) { /* growth: no sum, old index = y without its newest digit */
                    int64_t x = y / N;
                    B[y] = f * Kk[sk * N + (int)(x % N)] * A[x];
                } else {         /* slide: sum over sigma_{k-L} = most significant digit of the old index */
                    cplx s = 0;
                    for (int so = 0; so < N; ++so) {
                        int64_t x = y / N + (int64_t)so * top; /* sigma_{k-1} = x % N */
                        s += tabp[(size_t)L * N * N + sk * N + so] * Kk[sk * N + (int)(x % N)] * A[x];
                    }
                    B[y] = f * s;
                }
            }
        }
        /* path filtering (reading C.3-15): drop the entries of A_k below theta in magnitude */
        if (p->filter_theta > 0.0) {
            const double th2 = p->filter_theta * p->filter_theta;
#pragma omp parallel for schedule(static)
            for (int64_t y = 0; y < n_new; ++y) {
                const double re = creal(B[y]), im = cimag(B[y]);
                if (re * re + im * im < th2) B[y] = 0;
            }
        }
        if (p->kept) {
            int64_t nz = 0;
#pragma omp parallel for schedule(static) reduction(+ : nz)
            for (int64_t y = 0; y < n_new; ++y) nz += (B[y] != 0);
            p->kept[k] = nz;
        }
        cplx *tmp = A; A = B; B = tmp;
        w_old = w_new;
        double dtk = now_s() - ts;
        if (contract) { t_slide += dtk; ++n_slide; } else t_grow += dtk;
    }
    if (timings) { timings[0] = t_setup; timings[1] = t_grow; timings[2] = t_slide; timings[3] = (double)n_slide; }
    free(A); free(B); free(tabp); free(tabt); free(Kbuf); ctx_free(&c);
    return 0;
}
