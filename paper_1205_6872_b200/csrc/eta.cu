// eta.cu -- host-setup step a3 on the device ("fast eta / G setup"): every eta class of
// Eqs. 10-16 on the Strang windows (reading C.3-1) for B baths at once.
// The paper names this setup as the bottleneck once propagation runs on the GPU.
//
// Each class is the direct omega-integral of its window kernel (the same formulation as the host's
// adaptive quadrature in host.cpp: eta_class; the oracle uses finite differences of G instead):
//   self window of width w0:  (1/pi) int J(w)/w^2 [coth(w/2kT) 2 sin^2(w w0/2) - i (w w0 - sin w w0)] dw
//   later window wa, earlier wb, centre distance dc:
//                             (1/pi) int J(w)/w^2 4 sin(w wa/2) sin(w wb/2) [coth cos(w dc) - i sin(w dc)] dw
// on (0, Om] with a fixed composite Gauss-Kronrod 21-point rule (no adaptivity: every panel is short
// against the integrand's nearest complex singularity, so the 21-point rule is at rounding level):
//   panel width h0 = min(wc/4, pi/(2 span)) (span = the window pair's largest time separation), and
//   h1 = min(h0, pi kT) on [0, 16 pi kT] where the coth poles at +-i 2 pi n kT sit close to the axis.
// Debye's algebraic tail beyond Om is added in closed form (partial fractions + asymptotic series).
//
// Launch: one 8-CTA thread-block cluster per (bath, class); the 8 CTAs take interleaved panels, each
// reduces its panel sums with a fixed shuffle/shared-memory tree, and CTA 0 of the cluster sums the 8
// partials in rank order through distributed shared memory -- no scratch buffer, no atomics, so the
// result is run-to-run bit-identical.
#include <cooperative_groups.h>

#include "qp_internal.h"

namespace cg = cooperative_groups;

namespace qp {
namespace {

constexpr int kEtaCluster = 8;
constexpr int kEtaBlock = 256;

// Gauss-Kronrod 10/21 abscissae (descending, last = 0) and weights; Gauss 10-point weights of the
// odd-indexed Kronrod nodes.
__constant__ double cXgk[11] = {0.995657163025808080735527280689003, 0.973906528517171720077964012084452,
                                0.930157491355708226001207180059508, 0.865063366688984510732096688423493,
                                0.780817726586416897063717578345042, 0.679409568299024406234327365114874,
                                0.562757134668604683339000099272694, 0.433395394129247190799265943165784,
                                0.294392862701460198131126603103866, 0.148874338981631210884826001129720,
                                0.0};
__constant__ double cWgk[11] = {0.011694638867371874278064396062192, 0.032558162307964727478818972459390,
                                0.054755896574351996031381300244580, 0.075039674810919952767043140916190,
                                0.093125454583697605535065465083366, 0.109387158802297641899210590325805,
                                0.123491976262065851077208980725525, 0.134709217311473325928054001771707,
                                0.142775938577060080797094273138717, 0.147739104901338491374841515972068,
                                0.149445554002916905664936468389821};
__constant__ double cWg[5] = {0.066671344308688137593568809893332, 0.149451349150580593145776339657697,
                              0.219086362515982043995534934228163, 0.269266719309996355091226921569469,
                              0.295524224714752870173892994651338};

__constant__ double cWms[13] = {  // 1/(2m+3)!, m = 0..12
    0.16666666666666666, 0.008333333333333333, 0.0001984126984126984, 2.7557319223985893e-06,
    2.505210838544172e-08, 1.6059043836821613e-10, 7.647163731819816e-13, 2.8114572543455206e-15,
    8.22063524662433e-18, 1.9572941063391263e-20, 3.8681701706306835e-23, 6.446950284384474e-26,
    9.183689863795546e-29};

struct Win {
    bool self;
    double w0, wa, wb, dc, span;
};

// class c of the qp_plan_eta order [self_int, self_end, eta_1..L, E_1..L, TI_1..L] (units: time)
__device__ Win window(int c, int L, double dt) {
    Win w{};
    if (c < 2) {
        w.self = true;
        w.w0 = c == 0 ? dt : 0.5 * dt;  // Eq. 11 (interior self, G(1)) / Eqs. 13-14 (end points, G(1/2))
        w.span = w.w0;
        return w;
    }
    const int g = (c - 2) / L, j = (c - 2) % L + 1;
    if (g == 0) { w.wa = dt; w.wb = dt; w.dc = j * dt; }                       // Eq. 10: eta_j
    else if (g == 1) { w.wa = dt; w.wb = 0.5 * dt; w.dc = (j - 0.25) * dt; }  // Eqs. 15-16: edge E(j)
    else { w.wa = 0.5 * dt; w.wb = 0.5 * dt; w.dc = (j - 0.5) * dt; }         // Eq. 12: terminal-initial TI(j)
    w.span = w.dc + 0.5 * (w.wa + w.wb);
    return w;
}

__device__ double spectral(const EtaBath &b, double w) {
    switch (b.kind) {
    case 1: return 0.5 * M_PI * b.xi * w * exp(-w / b.wc);                  // Ohmic-exp
    case 2: return 0.5 * M_PI * b.xi * w * (b.wc * b.wc / (w * w + b.wc * b.wc));  // Debye
    case 3: { const double r = w / b.wc; return b.xi * w * w * w * exp(-r * r); }  // Eq. 21, reading C.3-5
    default: return 0.0;
    }
}

__device__ double coth_half_beta(const EtaBath &b, double w) {  // coth(w / 2kT), expm1: no cancellation at small w
    if (b.kT <= 0.0) return 1.0;
    const double y = w / b.kT;  // 2 * (w / 2kT)
    if (y > 72.0) return 1.0;
    const double em = -expm1(-y);  // 1 - e^{-y}
    return (2.0 - em) / em;
}

// w - sin(w): Taylor series below 0.75 (x^3 sum_m (-1)^m x^(2m) / (2m+3)!)
__device__ double wms(double x) {
    if (fabs(x) >= 0.75) return x - sin(x);
    const double y = x * x;
    double t = cWms[12];
    for (int m = 11; m >= 0; --m) t = cWms[m] - y * t;
    return x * y * t;
}

__device__ double2 integrand(const EtaBath &b, const Win &c, double w) {
    const double j = spectral(b, w) / M_PI;
    const double ct = coth_half_beta(b, w);
    if (c.self) {
        const double h = sin(0.5 * w * c.w0);
        return make_double2(j * ct * 2.0 * h * h / (w * w), -j * wms(w * c.w0) / (w * w));
    }
    const double P = 4.0 * sin(0.5 * w * c.wa) * sin(0.5 * w * c.wb) / (w * w);
    double sd, cd;
    sincos(w * c.dc, &sd, &cd);
    return make_double2(j * P * ct * cd, -j * P * sd);
}

__device__ double2 cdiv(double2 a, double2 b) {
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
__device__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

// Debye tail  int_Om^inf (1/pi) J/w^2 (1 - i w tau - e^{-i w tau}) dw  (coth = 1: beta Om > 40):
//   J/(pi w^2) = (xi/2) c^2/(w (w^2+c^2)) = (xi/2) [1/w - Re 1/(w - ic)]  (partial fractions),
//   non-oscillatory part (xi/2)[(1/2) log(1 + c^2/Om^2) - i c tau atan(c/Om)],
//   oscillatory part e^{-i Om tau} sum_n g^(n)(Om)/(i tau)^(n+1), g = 1/w - Re 1/(w - ic).
__device__ double2 debye_tail(const EtaBath &b, double tau, double Om) {
    if (tau == 0.0) return make_double2(0.0, 0.0);
    const double c = b.wc;
    const double2 non = make_double2(0.5 * log1p((c / Om) * (c / Om)), -c * tau * atan(c / Om));
    double2 sum = make_double2(0.0, 0.0), denom = make_double2(0.0, tau);
    const double2 zinv = cdiv(make_double2(1.0, 0.0), make_double2(Om, -c));
    double2 zpow = zinv;
    double fact = 1.0, prev = 1e300, ompow = 1.0 / Om;
    for (int n = 0; n < 60; ++n) {
        if (n > 0) { fact *= n; zpow = cmul(zpow, zinv); ompow /= Om; }
        const double gn = ((n & 1) ? -1.0 : 1.0) * fact * (ompow - zpow.x);
        const double2 term = cdiv(make_double2(gn, 0.0), denom);
        const double mag = hypot(term.x, term.y);
        if (mag > prev) break;
        sum.x += term.x, sum.y += term.y;
        prev = mag;
        if (mag < 1e-24 * hypot(sum.x, sum.y)) break;
        denom = cmul(denom, make_double2(0.0, tau));
    }
    double so, co;
    sincos(-Om * tau, &so, &co);
    const double2 osc = cmul(make_double2(co, so), sum);
    return make_double2(0.5 * b.xi * (non.x - osc.x), 0.5 * b.xi * (non.y - osc.y));
}

// the window pair's positive corner separations: the closed-form Debye tail is evaluated at each
__device__ void corners(const Win &w, double (&t)[4]) {
    t[0] = w.dc + 0.5 * (w.wa + w.wb), t[1] = w.dc - 0.5 * (w.wa + w.wb);
    t[2] = w.dc - 0.5 * w.wa + 0.5 * w.wb, t[3] = w.dc + 0.5 * w.wa - 0.5 * w.wb;
}

__device__ double upper_limit(const EtaBath &b, const Win &w) {
    switch (b.kind) {
    case 1: return 64.0 * b.wc;                       // e^{-64}: below rounding
    case 3: return 13.0 * b.wc;                       // e^{-169}
    case 2: {  // + closed-form tail (coth = 1 beyond); its asymptotic series needs Om * tau >= 512
        double tmin = w.self ? w.w0 : 1e300, t[4];
        if (!w.self) {
            corners(w, t);
            for (int i = 0; i < 4; ++i)
                if (t[i] > 0.0) tmin = fmin(tmin, t[i]);
        }
        return fmax(fmax(256.0 * b.wc, 80.0 * b.kT), 512.0 / tmin);
    }
    default: return 0.0;
    }
}

// grid.x = kEtaCluster * n_classes, grid.y = B (<= kEtaBatchMax; the baths travel as a kernel parameter).  Output eta[b][c] (and the summed |K21 - G10|
// panel error estimate err[b][c] when err != nullptr).
__global__ void __cluster_dims__(kEtaCluster, 1, 1) __launch_bounds__(kEtaBlock)
    k_eta(const __grid_constant__ EtaBatch baths, int L, double dt, double2 *__restrict__ eta, double *__restrict__ err) {
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int nc = 3 * L + 2;
    const int c = blockIdx.x / kEtaCluster, bi = blockIdx.y;
    const EtaBath b = baths.b[bi];
    const Win win = window(c, L, dt);
    __shared__ double red[kEtaBlock / 32][3];
    __shared__ double part[3];  // this CTA's (re, im, err), read by rank 0 through DSMEM

    double sr = 0.0, si = 0.0, se = 0.0;
    if (b.kind != 0) {
        // three uniform-panel regions: [0, W1] near the coth poles (width h1), [W1, W2] (h0), and the
        // far tail [W2, Om] beyond 64 wc where only the oscillation limits the width (h2)
        const double Om = upper_limit(b, win);
        const double hosc = 0.5 * M_PI / win.span;
        const double h0 = fmin(0.25 * b.wc, hosc);
        const double W1 = b.kT > 0.0 ? fmin(Om, 16.0 * M_PI * b.kT) : 0.0;
        const double h1 = b.kT > 0.0 ? fmin(h0, M_PI * b.kT) : h0;
        const double W2 = fmax(W1, fmin(Om, 64.0 * b.wc));
        const double h2 = fmin(hosc, 8.0 * b.wc);
        const long n1 = W1 > 0.0 ? (long)ceil(W1 / h1) : 0;
        const long n2 = W2 > W1 ? (long)ceil((W2 - W1) / h0) : 0;
        const long n3 = Om > W2 ? (long)ceil((Om - W2) / h2) : 0;
        const long np = n1 + n2 + n3;
        for (long i = (long)rank * kEtaBlock + threadIdx.x; i < np; i += (long)kEtaCluster * kEtaBlock) {
            double lo, hi;
            if (i < n1) { lo = W1 * double(i) / double(n1); hi = W1 * double(i + 1) / double(n1); }
            else if (i < n1 + n2) { const long q = i - n1; lo = W1 + (W2 - W1) * double(q) / double(n2); hi = W1 + (W2 - W1) * double(q + 1) / double(n2); }
            else { const long q = i - n1 - n2; lo = W2 + (Om - W2) * double(q) / double(n3); hi = W2 + (Om - W2) * double(q + 1) / double(n3); }
            const double m = 0.5 * (lo + hi), hw = 0.5 * (hi - lo);
            const double2 f0 = integrand(b, win, m);
            double kr = cWgk[10] * f0.x, ki = cWgk[10] * f0.y, gr = 0.0, gi = 0.0;
#pragma unroll 1
            for (int q = 0; q < 10; ++q) {
                const double2 fa = integrand(b, win, m - hw * cXgk[q]);
                const double2 fb = integrand(b, win, m + hw * cXgk[q]);
                kr += cWgk[q] * (fa.x + fb.x);
                ki += cWgk[q] * (fa.y + fb.y);
                if (q & 1) { gr += cWg[q >> 1] * (fa.x + fb.x); gi += cWg[q >> 1] * (fa.y + fb.y); }
            }
            sr += kr * hw;
            si += ki * hw;
            se += (fabs(kr - gr) + fabs(ki - gi)) * hw;
        }
    }
    // fixed-order block reduction: warp shuffle tree, then warp 0 over the warp partials
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_down_sync(0xffffffffu, sr, o);
        si += __shfl_down_sync(0xffffffffu, si, o);
        se += __shfl_down_sync(0xffffffffu, se, o);
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) { red[wid][0] = sr; red[wid][1] = si; red[wid][2] = se; }
    __syncthreads();
    if (wid == 0) {
        sr = lane < kEtaBlock / 32 ? red[lane][0] : 0.0;
        si = lane < kEtaBlock / 32 ? red[lane][1] : 0.0;
        se = lane < kEtaBlock / 32 ? red[lane][2] : 0.0;
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            sr += __shfl_down_sync(0xffffffffu, sr, o);
            si += __shfl_down_sync(0xffffffffu, si, o);
            se += __shfl_down_sync(0xffffffffu, se, o);
        }
        if (lane == 0) { part[0] = sr; part[1] = si; part[2] = se; }
    }
    cluster.sync();  // every CTA's partial is visible cluster-wide
    if (rank == 0 && threadIdx.x == 0) {
        double tr = 0.0, ti = 0.0, te = 0.0;
        for (int r = 0; r < kEtaCluster; ++r) {  // rank order: deterministic
            const double *p = cluster.map_shared_rank(part, r);
            tr += p[0], ti += p[1], te += p[2];
        }
        if (b.kind == 2) {  // Debye: closed-form tail beyond Om
            const double Om = upper_limit(b, win);
            double2 t;
            if (win.self) {
                t = debye_tail(b, win.w0, Om);
            } else {  // four corners of the window pair (later [a1,a2], earlier [b1,b2])
                double c4[4];
                corners(win, c4);
                const double2 a1 = debye_tail(b, c4[0], Om), a2 = debye_tail(b, c4[1], Om);
                const double2 a3 = debye_tail(b, c4[2], Om), a4 = debye_tail(b, c4[3], Om);
                t = make_double2(a1.x + a2.x - a3.x - a4.x, a1.y + a2.y - a3.y - a4.y);
            }
            tr += t.x, ti += t.y;
        }
        eta[(size_t)bi * nc + c] = make_double2(tr, ti);
        if (err) err[(size_t)bi * nc + c] = te;
    }
    cluster.sync();  // keep every CTA's shared memory alive until rank 0 has read it
}

}  // namespace

cudaError_t launch_eta(const EtaBatch &baths, int B, int L, double dt, double2 *d_eta, double *d_err, cudaStream_t s) {
    const dim3 grid(kEtaCluster * (3 * L + 2), B);
    k_eta<<<grid, kEtaBlock, 0, s>>>(baths, L, dt, d_eta, d_err);
    return cudaGetLastError();
}

}  // namespace qp
