// host.cpp -- host setup and C ABI of libquapi.so (include/quapi.h).
//
// Setup (all on the host, once per plan):
//   a1 validate     : H, rho0 Hermitian, tr rho0 = 1, dt > 0, 2 <= M <= 4, 2 <= L, out_steps
//   a2 propagator   : U = exp(-i H dt) by scaling-and-squaring Taylor (no eigensolver);
//                     K(sig', sig) = U[a',a] conj(U[b',b])  (Eq. 8)
//   a3 eta          : each eta class of Eqs. 10-16 on the Strang windows (DESIGN §3,
//                     reading C.3-1) integrated DIRECTLY in omega with its window kernel
//                       pair  : (1/pi) int J(w) [4 sin(w wa/2) sin(w wb/2)/w^2][coth cos(w dc) - i sin(w dc)]
//                       self  : (1/pi) int J(w)/w^2 [coth (1 - cos w w0) - i (w w0 - sin w w0)]
//                     (adaptive Gauss-Kronrod 10/21; Debye: complex partial-fraction asymptotic tail)
//   a4 tables       : Eq. 9 exponents psi, per-digit-group factor tables, K', beta, offsets
// The CPU oracle (oracle/) computes the same quantities with different formulations and shares
// no code with this file.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <thread>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <string>
#include <vector>

#include "../../include/quapi.h"
#include "qp_internal.h"

using cd = std::complex<double>;

namespace {

thread_local std::string g_err;

qp_status err(qp_status st, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

#define QP_CUDA(call)                                                                           \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess) return err(QP_ERR_CUDA, "cuda: %s at %s:%d", cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

inline double2 d2(cd z) { return make_double2(z.real(), z.imag()); }
inline int64_t ipow(int64_t b, int e) {
    int64_t r = 1;
    while (e-- > 0) r *= b;
    return r;
}
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------------------------------- a2: U
// exp(X), X = -i H dt, by scaling and squaring with a degree-20 Taylor polynomial.
std::vector<cd> expm_taylor(const std::vector<cd> &X, int M) {
    double nrm = 0.0;  // 1-norm
    for (int j = 0; j < M; ++j) {
        double c = 0.0;
        for (int i = 0; i < M; ++i) c += std::abs(X[i * M + j]);
        nrm = std::max(nrm, c);
    }
    int s = 0;
    while (nrm > 0.125) { nrm *= 0.5; ++s; }
    const double scale = std::ldexp(1.0, -s);
    std::vector<cd> Y(M * M), R(M * M, 0.0), T(M * M), tmp(M * M);
    for (int i = 0; i < M * M; ++i) Y[i] = X[i] * scale;
    for (int i = 0; i < M; ++i) R[i * M + i] = 1.0;
    T = R;
    for (int n = 1; n <= 20; ++n) {  // T = Y^n / n!
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) {
                cd acc = 0.0;
                for (int k = 0; k < M; ++k) acc += T[i * M + k] * Y[k * M + j];
                tmp[i * M + j] = acc / double(n);
            }
        T = tmp;
        for (int i = 0; i < M * M; ++i) R[i] += T[i];
    }
    for (int q = 0; q < s; ++q) {
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) {
                cd acc = 0.0;
                for (int k = 0; k < M; ++k) acc += R[i * M + k] * R[k * M + j];
                tmp[i * M + j] = acc;
            }
        R = tmp;
    }
    return R;
}

// ------------------------------------------------------------------------------------- a3: eta
// QK21 (Gauss-Kronrod 10/21) nodes and weights.
const double kXgk[11] = {0.995657163025808080735527280689003, 0.973906528517171720077964012084452,
                         0.930157491355708226001207180059508, 0.865063366688984510732096688423493,
                         0.780817726586416897063717578345042, 0.679409568299024406234327365114874,
                         0.562757134668604683339000099272694, 0.433395394129247190799265943165784,
                         0.294392862701460198131126603103866, 0.148874338981631210884826001129720,
                         0.000000000000000000000000000000000};
const double kWgk[11] = {0.011694638867371874278064396062192, 0.032558162307964727478818972459390,
                         0.054755896574351996031381300244580, 0.075039674810919952767043140916190,
                         0.093125454583697605535065465083366, 0.109387158802297641899210590325805,
                         0.123491976262065851077208980725525, 0.134709217311473325928054001771707,
                         0.142775938577060080797094273138717, 0.147739104901338491374841515972068,
                         0.149445554002916905664936468389821};
const double kWg[5] = {0.066671344308688137593568809893332, 0.149451349150580593145776339657697,
                       0.219086362515982043995534934228163, 0.269266719309996355091226921569469,
                       0.295524224714752870173892994651338};

struct Bath {
    int kind;
    double xi, wc, kT;
    double (*J)(double, void *);
    void *user;
    double cutoff;
    double spectral(double w) const {
        switch (kind) {
        case QP_J_OHMIC_EXP: return 0.5 * M_PI * xi * w * std::exp(-w / wc);
        case QP_J_DEBYE: return 0.5 * M_PI * xi * w * (wc * wc / (w * w + wc * wc));
        case QP_J_SUPEROHMIC_GAUSS: { double r = w / wc; return xi * w * w * w * std::exp(-r * r); }
        case QP_J_CALLBACK: return J(w, user);
        default: return 0.0;
        }
    }
    double coth_half_beta(double w) const {  // coth(w / 2kT)
        if (kT <= 0.0) return 1.0;
        double y = w / (2.0 * kT);
        if (y > 36.0) return 1.0;
        double e = std::exp(-2.0 * y);
        return (1.0 + e) / (1.0 - e);
    }
};

// A window class: "self" triangle of width w0, or a disjoint pair (later width wa, earlier wb,
// centre distance dc).  Units: time (already multiplied by dt).
struct WinClass {
    bool self;
    double w0, wa, wb, dc;
};

// w - sin(w) for the self kernel: x^3 sum_m (-1)^m x^(2m)/(2m+3)!  (Horner in x^2) below 0.75
double wms(double x) {
    if (std::fabs(x) >= 0.75) return x - std::sin(x);
    static const std::array<double, 13> c = [] {  // 1/(2m+3)!
        std::array<double, 13> t{};
        for (int m = 0; m < 13; ++m) {
            double f = 1.0;
            for (int q = 2; q <= 2 * m + 3; ++q) f *= q;
            t[m] = 1.0 / f;
        }
        return t;
    }();
    const double y = x * x;
    double t = c[12];
    for (int m = 11; m >= 0; --m) t = c[m] - y * t;
    return x * y * t;
}

cd kernel(const Bath &b, const WinClass &c, double w) {
    const double j = b.spectral(w) / M_PI;
    const double ct = b.coth_half_beta(w);
    if (c.self) {
        const double h = std::sin(0.5 * w * c.w0);
        return cd(j * ct * 2.0 * h * h / (w * w), -j * wms(w * c.w0) / (w * w));
    }
    const double P = 4.0 * std::sin(0.5 * w * c.wa) * std::sin(0.5 * w * c.wb) / (w * w);
    return cd(j * P * ct * std::cos(w * c.dc), -j * P * std::sin(w * c.dc));
}

struct QK {
    cd val;
    double err, roundoff;
};

QK qk21(const Bath &b, const WinClass &c, double lo, double hi) {
    const double m = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
    cd f[21];
    double wk[21];
    f[0] = kernel(b, c, m);
    wk[0] = kWgk[10];
    for (int i = 0; i < 10; ++i) {
        f[1 + 2 * i] = kernel(b, c, m - h * kXgk[i]);
        f[2 + 2 * i] = kernel(b, c, m + h * kXgk[i]);
        wk[1 + 2 * i] = wk[2 + 2 * i] = kWgk[i];
    }
    cd K = 0.0, Gs = 0.0;
    double absr = 0.0, absi = 0.0;
    for (int q = 0; q < 21; ++q) {
        K += wk[q] * f[q];
        absr += wk[q] * std::fabs(f[q].real());
        absi += wk[q] * std::fabs(f[q].imag());
    }
    for (int i = 1; i < 10; i += 2) Gs += kWg[i / 2] * (f[1 + 2 * i] + f[2 + 2 * i]);
    const cd mean = 0.5 * K;
    double ascr = 0.0, asci = 0.0;
    for (int q = 0; q < 21; ++q) {
        ascr += wk[q] * std::fabs(f[q].real() - mean.real());
        asci += wk[q] * std::fabs(f[q].imag() - mean.imag());
    }
    auto est = [](double d, double asc, double abs_) {
        double e = std::fabs(d);
        if (asc != 0.0 && e != 0.0) e = asc * std::min(1.0, std::pow(200.0 * e / asc, 1.5));
        return std::max(e, 50.0 * 2.2204460492503131e-16 * abs_);
    };
    QK r;
    r.val = K * h;
    r.err = (est((K - Gs).real() * h, ascr * h, absr * h) + est((K - Gs).imag() * h, asci * h, absi * h));
    r.roundoff = 100.0 * 2.2204460492503131e-16 * (absr + absi) * h;
    return r;
}

// adaptive bisection; accumulates into (s, comp) with compensated summation
bool adapt(const Bath &b, const WinClass &c, double lo, double hi, double tol, int depth, cd &s, cd &comp) {
    QK r = qk21(b, c, lo, hi);
    if (r.err <= tol || r.err <= 1.01 * r.roundoff || depth >= 30) {
        cd y = r.val - comp;  // Kahan
        cd t = s + y;
        comp = (t - s) - y;
        s = t;
        return r.err <= tol || r.err <= 1.01 * r.roundoff;
    }
    const double mid = 0.5 * (lo + hi);
    bool ok = adapt(b, c, lo, mid, 0.5 * tol, depth + 1, s, comp);
    ok &= adapt(b, c, mid, hi, 0.5 * tol, depth + 1, s, comp);
    return ok;
}

// Debye tail  int_Om^inf (1/pi) J/w^2 (1 - i w tau - e^{-i w tau}) dw  with coth = 1 (beta Om > 40):
//   J/(pi w^2) = (xi/2) c^2 / (w (w^2 + c^2)) = (xi/2) [1/w - Re 1/(w - ic)]   (partial fractions)
//   non-oscillatory part: (xi/2)[ (1/2) log(1 + c^2/Om^2) - i c tau atan(c/Om) ]
//   oscillatory part: e^{-i Om tau} sum_n g^(n)(Om)/(i tau)^(n+1),  g = 1/w - Re 1/(w - ic).
cd debye_Gtail(const Bath &b, double tau, double Om) {
    if (tau == 0.0) return 0.0;
    const double c = b.wc;
    const cd non = cd(0.5 * std::log1p((c / Om) * (c / Om)), -c * tau * std::atan(c / Om));
    cd sum = 0.0, denom = cd(0.0, tau);  // (i tau)^(n+1)
    const cd z = cd(Om, -c);
    double fact = 1.0, prev = 1e300;
    cd zinv = 1.0 / z, zpow = zinv;  // z^-(n+1)
    double ompow = 1.0 / Om;
    for (int n = 0; n < 60; ++n) {
        if (n > 0) { fact *= n; zpow *= zinv; ompow /= Om; }
        const double gn = ((n % 2) ? -1.0 : 1.0) * fact * (ompow - zpow.real());
        const cd term = gn / denom;
        const double mag = std::abs(term);
        if (mag > prev) break;
        sum += term;
        prev = mag;
        if (mag < 1e-24 * std::abs(sum)) break;
        denom *= cd(0.0, tau);
    }
    const cd osc = std::exp(cd(0.0, -Om * tau)) * sum;
    return 0.5 * b.xi * (non - osc);
}

qp_status eta_class(const Bath &b, const WinClass &c, cd *out, const char *name, int lag) {
    *out = 0.0;
    if (b.kind == QP_J_ZERO) return QP_OK;
    double Om;
    switch (b.kind) {
    case QP_J_OHMIC_EXP: Om = 64.0 * b.wc; break;
    case QP_J_SUPEROHMIC_GAUSS: Om = 13.0 * b.wc; break;
    case QP_J_DEBYE: {  // the closed-form tail's asymptotic series needs Om * tau >= 512 at every corner tau
        double tmin = c.self ? c.w0 : 1e300;
        if (!c.self)
            for (double t : {c.dc + 0.5 * (c.wa + c.wb), c.dc - 0.5 * (c.wa + c.wb), c.dc - 0.5 * c.wa + 0.5 * c.wb,
                             c.dc + 0.5 * c.wa - 0.5 * c.wb})
                if (t > 0.0) tmin = std::min(tmin, t);
        Om = std::max({256.0 * b.wc, 80.0 * b.kT, 512.0 / tmin});
        break;
    }
    default: Om = b.cutoff; break;
    }
    const double span = c.self ? c.w0 : c.dc + 0.5 * (c.wa + c.wb);
    double h = 0.25 * (b.kind == QP_J_CALLBACK ? Om / 64.0 : b.wc);
    h = std::min(h, 0.5 * M_PI / span);
    const long np = std::max(1L, (long)std::ceil(Om / h));
    cd s = 0.0, comp = 0.0;
    bool ok = true;
    for (long i = 0; i < np; ++i) {
        const double lo = Om * double(i) / double(np), hi = Om * double(i + 1) / double(np);
        ok &= adapt(b, c, lo, hi, 1e-17 / double(np), 0, s, comp);
    }
    if (b.kind == QP_J_DEBYE) {
        cd t;
        if (c.self) {
            t = debye_Gtail(b, c.w0, Om);
        } else {  // four corners of the window pair (later [a1,a2], earlier [b1,b2])
            const double t1 = c.dc + 0.5 * (c.wa + c.wb), t2 = c.dc - 0.5 * (c.wa + c.wb);
            const double t3 = c.dc - 0.5 * c.wa + 0.5 * c.wb, t4 = c.dc + 0.5 * c.wa - 0.5 * c.wb;
            t = debye_Gtail(b, t1, Om) + debye_Gtail(b, t2, Om) - debye_Gtail(b, t3, Om) - debye_Gtail(b, t4, Om);
        }
        s += t;
    }
    *out = s - comp;
    if (!ok) return err(QP_ERR_QUADRATURE, "quadrature: eta class %s lag %d did not converge", name, lag);
    return QP_OK;
}

}  // namespace

// ===================================================================================== plan
// One k_fused4 tensor map (slide4.cu): the order of the 11 box bits in the shared-memory stage
// (bit 2 i + b = bit b of inner digit i, 8..10 = bits of the round's fibre index), the TMA
// dimensions built from it, and which dimensions carry the round's outer-fibre coordinate.
struct F4Map {
    int pos[11];
    int lane_swap = 0;       // lane mapping of the phase this map serves (FusedArgs::f4_q1swap / f4_q2swap)
    int ndim = 0;
    cuuint64_t gdim[5];
    cuuint64_t gstr[4];
    cuuint32_t box[5];
    int cdimA = -1, cdimB = -1;
};

struct qp_plan {
    int M = 0, N = 0, L = 0, D = 0;
    bool lattice = false;        // class map used by the kernels
    bool sym = false;            // M = 2 with s = (+s, -s): symmetric-moment kernel
    bool sym3 = false;           // M = 3 with s = (c, 0, -c): k_fused2t (conjugate-pair moments)
    uint32_t flags = 0;          // qp_problem.flags (QP_FLAG_*)
    double dt = 0.0;
    int64_t n_steps = 0;
    std::vector<int64_t> out_steps;
    std::vector<double> s;
    std::vector<cd> H, rho0, U, K;     // K[new*N + old]
    std::vector<double> delta;         // [D]
    // eta classes (Strang windows): self interior, self end, eta_j, E_j, TI_j (j = 1..L)
    cd self_int, self_end;
    std::vector<cd> eta, E, TI;        // index j (0 unused)
    std::vector<cd> A0;                // [N]
    // device image
    std::vector<double2> small;        // SmallLayout
    struct LaunchSet {                 // fused launch over inner slots p0..p0+S-1 (mod L)
        int p0 = 0, S = 1;
        std::vector<double2> inner;    // [S][S][2][D][N]
        std::vector<double2> Etab;     // [S][2][G][D][X]
        std::vector<long long> goff;   // [G][X]
        std::vector<int2> lofs;        // [T]
        std::vector<double2> E0r;      // TMA sets: per round of e0r_F fibres [S][2][D][F] factors + F offsets
        int e0r_F = 0;
        size_t off_E0r = 0;
        size_t off_inner = 0, off_E = 0, off_goff = 0, off_lofs = 0;
        qp::FusedArgs args{};          // table pointers filled in qp_steps
        // k_fused3 TMA view (-1: none).  View A (1 <= p0 <= L-3): run A = slots 0..tma_a-1 (tma_a = p0),
        // run B = the tma_b slots above the inner ones.  View B (p0 = L-2, tma_a = 0): inner digit 2 is
        // slot 0 and the outer slots 1..L-3 are one run.
        int tma_a = -1, tma_b = 0;
        mutable const void *tma_A = nullptr;  // ARDM pointer the cached tensor map was encoded for
        mutable CUtensorMap tmap{};
        // k_fused4 (S = 4): load / store tensor maps of the 8-fibre rounds (f4_layout)
        bool f4 = false;
        F4Map f4map[2];                // [0] load (phase-1 reads conflict-free), [1] store (phase-2 writes)
        int f4_col = 0;                // slot 0 outer: fibres are the 16-B chunks of a stage row
        int f4_swz = 1;                // 128-B swizzle (both maps), else dense stage
        long long f4_nA = 1;
        int f4_c0m = 1;
        mutable CUtensorMap tmapS{};
        // k_fused2t (M = 3 lattice, S = 2, unsharded): view kind (slide2t.cu), -1 none
        int f2t = -1;
        int f2t_p0 = 0, f2t_L = 0;     // position of inner digit 0 in the (local) layout, its digit count
    };
    int group_w = 1;                   // digits per outer digit group (g >= 1) of the factor tables
    int Smax = 1;
    // persistent path (small ARDM): launch-set arguments and per-step readout slots in the workspace
    bool persist = false;
    size_t off_psets = 0, off_pslot = 0;
    size_t small_dyn = 0;              // > 0 after qp_init: k_small runs the slide steps, its dynamic smem
    std::vector<LaunchSet> sets;       // index p0 * Smax + (S - 1)
    size_t off_small = 0, off_part = 0, off_rho = 0, off_cnt = 0, tables_end = 0, work_bytes = 0;
    int64_t ardm_entries = 0;
    int grid[qp::kMaxS + 1] = {0};
    int block = 0;
    double setup_ms[3] = {0, 0, 0};    // validate + U, eta, tables (qp_sizes)
    int64_t max_bytes = 0;             // qp_problem.max_bytes (capacity budget)
    int occ[qp::kMaxS + 1][3] = {};    // resident CTAs per SM of the slide kernel per (S, load path)
    int sms = 0;
    int64_t next_k = 1;
    bool inited = false;
    double setup_seconds = 0.0;
    // ---- sharded execution (multi-GPU); see qp_shard_configure
    struct Shard {
        bool on = false;
        int G = 1, rank = 0, z = 0, seg_len = 0;
        int64_t NZ = 1, blk = 0;                     // combos per shard-slot set, entries per block
        std::vector<int64_t> c_lo, n_own;            // owned combo range per rank
        std::vector<LaunchSet> sets;                 // shard launch sets
        std::map<std::tuple<int, int, int>, size_t> index;  // (zstart, p0, S) -> sets
        int64_t seg = 0;                             // current segment
        int Smax = 1;                                // fusion depth inside segments
    } sh;
    int64_t seg_begin(int64_t j) const { return L + j * sh.seg_len; }
    std::vector<int> zset(int64_t j) const {         // shard slots of segment j, ascending
        std::vector<int> z;
        const int64_t k = seg_begin(j);
        for (int i = 0; i < sh.z; ++i) z.push_back((int)(((k - 1 - i) % L + L) % L));
        std::sort(z.begin(), z.end());
        return z;
    }
    int64_t slot_of(int64_t k) const {
        auto it = std::lower_bound(out_steps.begin(), out_steps.end(), k);
        return (it != out_steps.end() && *it == k) ? int64_t(it - out_steps.begin()) : -1;
    }
};

namespace {

// psi(sigma'; eta) = -(eta s+(sigma') - conj(eta) s-(sigma'))  -- Eq. 9 summand without Delta s(later)
cd psi(const qp_plan &P, int sg, cd e) {
    const double sp = P.s[sg / P.M], sm = P.s[sg % P.M];
    return -(e * sp - std::conj(e) * sm);
}
double dsig(const qp_plan &P, int sg) { return P.s[sg / P.M] - P.s[sg % P.M]; }

void build_classes(qp_plan &P) {
    const int M = P.M;
    bool lat = false;
    if (M > 2) {
        const double u = P.s[1] - P.s[0];
        lat = (u != 0.0);
        for (int a = 0; a < M && lat; ++a)
            if (std::fabs(P.s[a] - (P.s[0] + a * u)) > 1e-15 * std::max(1.0, std::fabs(P.s[a]))) lat = false;
    }
    P.lattice = lat;
    P.sym = (M == 2) && P.s[0] == -P.s[1] && P.s[0] != 0.0 && !(P.flags & QP_FLAG_GENERIC_MOMENTS);
    P.sym3 = (M == 3) && P.s[1] == 0.0 && P.s[0] == -P.s[2] && P.s[0] != 0.0 && !(P.flags & QP_FLAG_GENERIC_MOMENTS);
    P.D = qp::n_classes(M, lat);
    P.delta.assign(P.D, 0.0);
    for (int a = 0; a < M; ++a)
        for (int b = 0; b < M; ++b) {
            const int c = qp::class_of(M, lat, a, b);
            if (c > 0) P.delta[c - 1] = P.s[a] - P.s[b];  // same value for every (a,b) of a lattice class
        }
}

qp_status compute_eta(qp_plan &P, const qp_problem &pr) {
    const int L = P.L;
    const double dt = P.dt;
    P.eta.assign(L + 1, 0.0);
    P.E.assign(L + 1, 0.0);
    P.TI.assign(L + 1, 0.0);
    if (pr.kind == QP_J_ETA_TABLE) {  // eta classes given (e.g. by qp_eta_device), qp_plan_eta order
        auto e = [&](int i) { return cd(pr.eta_in[i].re, pr.eta_in[i].im); };
        P.self_int = e(0);
        P.self_end = e(1);
        for (int j = 1; j <= L; ++j) {
            P.eta[j] = e(1 + j);
            P.E[j] = e(1 + L + j);
            P.TI[j] = e(1 + 2 * L + j);
        }
        return QP_OK;
    }
    if (pr.kind == QP_J_G_TABLE) {  // alpha given as G(m dt/2): four-corner rule, G'' = alpha
        auto G = [&](int m) { return cd(pr.G_in[m].re, pr.G_in[m].im); };  // m = 2 x
        P.self_int = G(2);
        P.self_end = G(1);
        for (int j = 1; j <= L; ++j) {
            P.eta[j] = G(2 * j + 2) + G(2 * j - 2) - 2.0 * G(2 * j);
            P.E[j] = G(2 * j + 1) + G(2 * j - 2) - G(2 * j - 1) - G(2 * j);
            P.TI[j] = G(2 * j) + G(2 * j - 2) - 2.0 * G(2 * j - 1);
        }
        return QP_OK;
    }
    Bath b{pr.kind, pr.coupling, pr.omega_c, pr.kT, pr.J, pr.J_user, pr.J_cutoff};
    // the 3L+2 class integrals are independent: run them on host threads (the paper's §V notes the
    // eta setup becomes the bottleneck once propagation runs on the GPU)
    struct Job { WinClass c; cd *out; const char *name; int lag; qp_status st; std::string msg; };
    std::vector<Job> jobs;
    jobs.push_back({WinClass{true, dt, 0, 0, 0}, &P.self_int, "self_interior", 0, QP_OK, {}});
    jobs.push_back({WinClass{true, 0.5 * dt, 0, 0, 0}, &P.self_end, "self_end", 0, QP_OK, {}});
    for (int j = 1; j <= L; ++j) {
        jobs.push_back({WinClass{false, 0, dt, dt, j * dt}, &P.eta[j], "eta", j, QP_OK, {}});
        jobs.push_back({WinClass{false, 0, dt, 0.5 * dt, (j - 0.25) * dt}, &P.E[j], "edge", j, QP_OK, {}});
        jobs.push_back({WinClass{false, 0, 0.5 * dt, 0.5 * dt, (j - 0.5) * dt}, &P.TI[j], "terminal_initial", j, QP_OK, {}});
    }
    const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::atomic<size_t> next{0};
    auto worker = [&] {
        for (size_t i = next++; i < jobs.size(); i = next++) {
            Job &jb = jobs[i];
            jb.st = eta_class(b, jb.c, jb.out, jb.name, jb.lag);
            if (jb.st) jb.msg = g_err;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
    worker();
    for (auto &th : pool) th.join();
    for (const Job &jb : jobs)
        if (jb.st) return err(jb.st, "%s", jb.msg.c_str());
    return QP_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link against libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
    static const EncodeTiledFn fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (EncodeTiledFn)f;
    }();
    return fn;
}

// k_fused3's TMA view of the ARDM for launch set ls: 5-D tensor of FP64 (run A as 2 x N^a doubles,
// run B, inner d0, d1, d2), box = one round of F outer fibres x N^3 inner entries.  Returns false
// (the kernel then loads with plain LDG) if the driver cannot encode it.
static bool encode_f3_tmap(const qp_plan &P, const qp_plan::LaunchSet &ls, double2 *A, int F) {
    if (ls.tma_A == A) return true;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const int p0 = ls.p0, L = P.L;
    cuuint64_t gdim[5], gstr[4];
    cuuint32_t box[5];
    if (ls.tma_a > 0) {  // view A: (run A as doubles, run B, d0, d1, d2); stage [d2][d1][d0][f]
        const cuuint64_t nA = (cuuint64_t)ipow(P.N, ls.tma_a), nB = (cuuint64_t)ipow(P.N, ls.tma_b);
        const cuuint64_t boxA = std::min<cuuint64_t>(nA, (cuuint64_t)F);
        if (nA * nB < (cuuint64_t)F || (cuuint64_t)F % boxA) return false;
        const cuuint64_t gd[5] = {2 * nA, nB, 4, 4, 4};
        const cuuint64_t gs[4] = {16ull * ipow(P.N, p0 + 3), 16ull * ipow(P.N, p0), 16ull * ipow(P.N, p0 + 1),
                                  16ull * ipow(P.N, p0 + 2)};
        const cuuint32_t bx[5] = {(cuuint32_t)(2 * boxA), (cuuint32_t)(F / boxA), 4, 4, 4};
        std::copy(gd, gd + 5, gdim), std::copy(gs, gs + 4, gstr), std::copy(bx, bx + 5, box);
    } else if (ls.tma_a == -3) {  // view D (p0 = 0): 128-B rows of the 8 entries (d1 & 1, d0), then f,
              // d1 / 2, d2; 128-B swizzle.  stage [d2][d1 / 2][f] rows, 16-B chunk XOR (row & 7)
        if ((cuuint64_t)ipow(P.N, L - 3) < (cuuint64_t)F) return false;
        const cuuint64_t gd[5] = {16, (cuuint64_t)ipow(P.N, L - 3), 2, 4, 1};
        const cuuint64_t gs[4] = {16ull * 64, 16ull * 8, 16ull * 16, 16ull * ipow(P.N, L)};
        const cuuint32_t bx[5] = {16, (cuuint32_t)F, 2, 4, 1};
        std::copy(gd, gd + 5, gdim), std::copy(gs, gs + 4, gstr), std::copy(bx, bx + 5, box);
    } else if (ls.tma_a == -2) {  // view C (p0 = L-1): 128-B rows of the 8 entries
              // (d1, d2 & 1), then f, d2 / 2, d0 = slot L-1; 128-B swizzle.  stage [d0][d2 / 2][f] rows,
              // 16-B chunk XOR (row & 7): the 8 fibres of a quarter-warp hit 8 distinct chunks
        if ((cuuint64_t)ipow(P.N, L - 3) < (cuuint64_t)F) return false;
        const cuuint64_t gd[5] = {16, (cuuint64_t)ipow(P.N, L - 3), 2, 4, 1};
        const cuuint64_t gs[4] = {256, 128, 16ull * ipow(P.N, L - 1), 16ull * ipow(P.N, L)};
        const cuuint32_t bx[5] = {16, (cuuint32_t)F, 2, 4, 1};
        std::copy(gd, gd + 5, gdim), std::copy(gs, gs + 4, gstr), std::copy(bx, bx + 5, box);
    } else {  // view B: slots 0..L-3 (= d2 + 4 f) as 128-B rows of two fibres, d0, d1; 128-B swizzle.
              // stage [d1][d0][f/2] rows of 8 entries (f & 1, d2), 16-B chunk XOR (row & 7)
        if ((cuuint64_t)ipow(P.N, L - 3) < (cuuint64_t)F || F % 2) return false;
        const cuuint64_t gd[5] = {16, (cuuint64_t)ipow(P.N, L - 2) / 8, 4, 4, 1};
        const cuuint64_t gs[4] = {128, 16ull * ipow(P.N, L - 2), 16ull * ipow(P.N, L - 1), 16ull * ipow(P.N, L)};
        const cuuint32_t bx[5] = {16, (cuuint32_t)(F / 2), 4, 4, 1};
        std::copy(gd, gd + 5, gdim), std::copy(gs, gs + 4, gstr), std::copy(bx, bx + 5, box);
    }
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(&ls.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)A, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            ls.tma_a > 0 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    ls.tma_A = A;
    return true;
}

// Persistent grid of one fused launch: fixed per (plan, launch set, device type), so the readout
// order (block partials) is deterministic.
static int slide_path(int S, const qp::FusedArgs &a) {
    return S == 3 ? (a.use_tma ? 2 : (a.lane_map & 1)) : (S == 2 && a.use_tma ? 2 : 0);
}
static int slide_occupancy(const qp_plan &P, int S, int path) {
    if (P.M == 3 && S == 2) return path == 2 ? qp::fused2t_occupancy() : qp::fused2s_occupancy(P.lattice);
    if (P.M == 2 && S == 4) return qp::fused4_occupancy(P.sym);
    if (P.M == 2 && S == 3) return qp::fused3_occupancy(P.sym, path & 1, path == 2);
    return qp::fused_r_occupancy(P.M, P.lattice, P.sym, S);
}
static int launch_grid(qp_plan *P, int S, const qp::FusedArgs &a) {
    const int path = slide_path(S, a);
    int &o = P->occ[S][path];
    if (o == 0) o = std::max(1, slide_occupancy(*P, S, path));
    return std::max(1, std::min<int>({a.n_tiles, P->sms * o, qp::kPartialsMax}));
}
static cudaError_t launch_slide(const qp_plan &P, int S, const qp::FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    if (P.M == 3 && S == 2) {
        qp::Beta2s b{};
        const qp::SmallLayout lay{P.N, P.D, P.L};
        for (int st = 0; st < 2; ++st)
            for (int kap = 0; kap < 2; ++kap)
                for (int d = 0; d < P.D; ++d)
                    for (int v = 0; v < P.N; ++v) b.b[st][kap][d][v] = P.small[lay.beta(a.var[st], kap) + d * P.N + v];
        if (a.use_tma) return qp::launch_fused2t(a, b, ro, grid, s);
        return qp::launch_fused2s(P.lattice, a, b, ro, grid, s);
    }
    if (P.M == 2 && S == 4) return qp::launch_fused4(P.sym, a, ro, grid, s);
    if (P.M == 2 && S == 3) return qp::launch_fused3(P.sym, a, ro, grid, s);
    return qp::launch_fused_r(P.M, P.lattice, P.sym, S, a, ro, grid, s);
}

// ---- k_fused4 stage layouts.  A stage holds one round: 8 outer fibres x the 256 entries of the inner
// digits d0..d3, as 11 box bits.  Under the 128-B swizzle a 16-B access at stage offset o (16-B units)
// hits bank group (o ^ (o >> 3)) & 7, so a quarter-warp (8 lanes) is conflict-free iff the three box
// bits its lanes vary map invertibly (over GF(2)) onto (bit i) ^ (bit i+3), i = 0..2, of the offset.
// Phase 1 (loads): lanes vary (d2, d3 & 1) (q = d2 + 4 d3) or (d3, d2 & 1) (q = d3 + 4 d2); phase 2
// (stores): (d0, d1 & 1) or (d1, d0 & 1).  The fibre bits sit at stage bits 0-2 when ring slot 0 (stride
// 1) is an outer slot, else at bits 8-10; the search orders the inner bits so that the load map serves
// phase 1 and the store map phase 2 with at most 5 TMA dimensions.
static bool gf2_invertible3(const int (&m)[3][3]) {
    int r[3];
    for (int i = 0; i < 3; ++i) r[i] = m[i][0] | (m[i][1] << 1) | (m[i][2] << 2);
    for (int c = 0; c < 3; ++c) {
        int piv = -1;
        for (int i = c; i < 3; ++i)
            if (r[i] >> c & 1) { piv = i; break; }
        if (piv < 0) return false;
        std::swap(r[c], r[piv]);
        for (int i = 0; i < 3; ++i)
            if (i != c && (r[i] >> c & 1)) r[i] ^= r[c];
    }
    return true;
}

bool f4_layout(const qp_plan &P, qp_plan::LaunchSet &ls, const std::vector<int> &pos, const std::vector<int> &inner,
               const std::vector<int> &outer) {
    const int N = P.N;
    if ((int)inner.size() != 4 || outer.size() < 2) return false;
    long long hs[11];  // HBM stride (entries) of each box bit
    for (int i = 0; i < 4; ++i)
        for (int b = 0; b < 2; ++b) hs[2 * i + b] = ipow(N, pos[inner[i]]) << b;
    hs[8] = ipow(N, pos[outer[0]]), hs[9] = 2 * hs[8], hs[10] = ipow(N, pos[outer[1]]);
    // outer runs: consecutive local positions
    std::vector<int> op;
    for (int q : outer) op.push_back(pos[q]);
    std::vector<std::pair<int, int>> runs;  // (first position, length)
    for (size_t i = 0; i < op.size(); ++i) {
        if (i && op[i] == op[i - 1] + 1) runs.back().second++;
        else runs.push_back({op[i], 1});
    }
    const bool typeA = op[0] == 0;
    if (typeA ? runs.size() > 2 : runs.size() != 1) return false;
    const long long nA = typeA ? ipow(N, runs[0].second) : (1ll << 62);
    if (typeA && nA < 4) return false;
    // the inner bits with HBM stride 1, 2, 4 (type I: the lowest 128 B of a fibre)
    int z[3] = {-1, -1, -1};
    for (int r = 0; r < 8; ++r)
        for (int k = 0; k < 3; ++k)
            if (hs[r] == (1ll << k)) z[k] = r;
    if (!typeA && (z[0] < 0 || z[1] < 0)) return false;
    // 128-B swizzle only with 128-B inner box rows (8 HBM-contiguous entries: 8 fibres, or three inner
    // bits); otherwise no swizzle (dense stage, possibly bank-conflicted: odd L only, p0 = 1 or L - 3)
    const bool swz = typeA ? nA >= 8 : z[2] >= 0;
    for (int which = 0; which < 2; ++which) {
        F4Map best{};
        int best_nd = 99;
        for (int swap = 0; swap < (swz ? 2 : 1); ++swap) {
            int qa[3];  // quarter-varying box bits of the phase this map serves
            if (which == 0) { if (swap) qa[0] = 6, qa[1] = 7, qa[2] = 4; else qa[0] = 4, qa[1] = 5, qa[2] = 6; }
            else { if (swap) qa[0] = 2, qa[1] = 3, qa[2] = 0; else qa[0] = 0, qa[1] = 1, qa[2] = 2; }
            // fixed positions: type A fibre bits 0..2; type I (swizzled) the three lowest inner bits 0..2,
            // (unswizzled) nothing but the stride-1 bit at 0; fibre bits at 8..10.  Positions first..5 are
            // chosen (they decide the banks), the rest follow in HBM-stride order.
            std::vector<int> fixed;
            if (typeA) fixed = {8, 9, 10};
            else if (swz) fixed = {z[0], z[1], z[2]};
            else fixed = {z[0]};
            const int first = (int)fixed.size();
            const int nchoose = swz ? 6 - first : 0;
            std::vector<int> cand;
            for (int r = 0; r < 8; ++r)
                if (std::find(fixed.begin(), fixed.end(), r) == fixed.end()) cand.push_back(r);
            std::vector<int> pick(nchoose, 0);
            std::function<void(int, unsigned)> rec = [&](int k, unsigned used) {
                if (k < nchoose) {
                    for (size_t c = 0; c < cand.size(); ++c)
                        if (!(used >> c & 1)) { pick[k] = (int)c; rec(k + 1, used | (1u << c)); }
                    return;
                }
                int order[11];
                for (int t = 0; t < first; ++t) order[t] = fixed[t];
                unsigned used2 = 0;
                for (int t = 0; t < nchoose; ++t) order[first + t] = cand[pick[t]], used2 |= 1u << pick[t];
                std::vector<int> rest;
                for (size_t c = 0; c < cand.size(); ++c)
                    if (!(used2 >> c & 1)) rest.push_back(cand[c]);
                std::sort(rest.begin(), rest.end(), [&](int x, int y) { return hs[x] < hs[y]; });
                for (size_t t = 0; t < rest.size(); ++t) order[first + nchoose + t] = rest[t];
                if (!typeA) order[8] = 8, order[9] = 9, order[10] = 10;
                if (swz) {  // bank condition
                    int m[3][3];
                    for (int i = 0; i < 3; ++i)
                        for (int j = 0; j < 3; ++j) m[i][j] = (order[i] == qa[j]) ^ (order[i + 3] == qa[j]);
                    if (!gf2_invertible3(m)) return;
                }
                // TMA dims
                F4Map mp{};
                for (int t = 0; t < 11; ++t) mp.pos[order[t]] = t;
                mp.lane_swap = swap;
                int nd = 0;
                auto add = [&](cuuint64_t g, cuuint32_t bx, long long stride_entries) {
                    if (nd >= 5) { nd = 6; return; }
                    mp.gdim[nd] = g, mp.box[nd] = bx;
                    if (nd > 0) mp.gstr[nd - 1] = (cuuint64_t)stride_entries * 16;
                    ++nd;
                };
                int t0 = 0;
                if (typeA) {
                    add((cuuint64_t)(2 * nA), (cuuint32_t)(2 * std::min<long long>(nA, 8)), 0);
                    mp.cdimA = 0;
                    if (nA < 8) {  // fibre bit 2 is the first bit of run B
                        if (runs.size() < 2) return;
                        add((cuuint64_t)ipow(N, runs[1].second), (cuuint32_t)(8 / nA), ipow(N, runs[1].first));
                        mp.cdimB = 1;
                    }
                    t0 = 3;
                }
                const int tend = typeA ? 11 : 8;
                for (int t = t0; t < tend;) {  // inner bits: merge runs of doubling stride (dim 0 <= 128 B)
                    int u = t + 1;
                    while (u < tend && hs[order[u]] == 2 * hs[order[u - 1]] && !(!typeA && t == 0 && u - t >= 3)) ++u;
                    const cuuint64_t sz = 1ull << (u - t);
                    if (!typeA && t == 0) add(2 * sz, (cuuint32_t)(2 * sz), 0);  // dim 0 in doubles
                    else add(sz, (cuuint32_t)sz, hs[order[t]]);
                    t = u;
                }
                if (!typeA) {
                    mp.cdimA = nd;
                    add((cuuint64_t)ipow(N, runs[0].second), 8, ipow(N, runs[0].first));
                } else if (nA >= 8 && runs.size() > 1) {
                    mp.cdimB = nd;
                    add((cuuint64_t)ipow(N, runs[1].second), 1, ipow(N, runs[1].first));
                }
                if (nd > 5) return;
                mp.ndim = nd;
                if (nd < best_nd) best = mp, best_nd = nd;
            };
            rec(0, 0);
        }
        if (best_nd > 5) return false;
        for (int d = best.ndim; d < 5; ++d) {  // pad to 5-D with unit dims
            best.gdim[d] = 1, best.box[d] = 1;
            best.gstr[d - 1] = 16;
        }
        ls.f4map[which] = best;
    }
    ls.f4_col = typeA ? 1 : 0;
    ls.f4_swz = swz ? 1 : 0;
    ls.f4_nA = nA;
    ls.f4_c0m = typeA ? 2 : 1;
    return true;
}

static bool encode_f4_tmaps(const qp_plan::LaunchSet &ls, double2 *A) {
    if (ls.tma_A == A) return true;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    for (int w = 0; w < 2; ++w) {
        const F4Map &m = ls.f4map[w];
        CUtensorMap *dst = w == 0 ? &ls.tmap : &ls.tmapS;
        if (enc(dst, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)A, m.gdim, m.gstr, m.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                ls.f4_swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    ls.tma_A = A;
    return true;
}

// k_fused2t's TMA view of the ARDM for launch set ls (slide2t.cu): a 5-D tensor of FP64 whose box is one
// unit of 27 outer fibres x the 81 inner entries (d0 = slot p0, d1 = slot p0 + 1); the same map loads
// and stores.  VK 0 (p0 = 0): [d0 d1][slots 2..L-1]; VK 1 (p0 = L-1): [d1 = slot 0, slot 1][slots 2..L-2][d0];
// VK 2 (2 <= p0 <= L-2): [slots 0..p0-1][d0][d1][slots p0+2..]; VK 3 (p0 = 1): [slot 0, d0][d1][slots 3..].
static bool encode_f2t_tmap(const qp_plan &P, const qp_plan::LaunchSet &ls, double2 *A) {
    if (ls.tma_A == A) return true;
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return false;
    const int L = ls.f2t_L, p0 = ls.f2t_p0;  // the local layout (a shard block lacks the shard slots)
    const cuuint64_t big = 16ull * (cuuint64_t)ipow(9, L);
    cuuint64_t gd[5], gs[4];
    cuuint32_t bx[5];
    auto set = [&](std::initializer_list<cuuint64_t> d, std::initializer_list<cuuint64_t> st, std::initializer_list<cuuint32_t> b) {
        std::copy(d.begin(), d.end(), gd), std::copy(st.begin(), st.end(), gs), std::copy(b.begin(), b.end(), bx);
    };
    // (the two lowest slots are merged into one box dimension of 162 doubles where both lie in the box
    // whole: 27 rows of 1296 B per unit instead of 243 rows of 144 B)
    switch (ls.f2t) {
    case 0:  // [d0 d1 (slots 0, 1)][slots 2..L-1]
        set({162, (cuuint64_t)ipow(9, L - 2), 1, 1, 1}, {16 * 81, big, big, big}, {162, 27, 1, 1, 1});
        break;
    case 1:  // [d1 = slot 0, slot 1][slots 2..L-2][d0 = slot L-1]
        set({162, (cuuint64_t)ipow(9, L - 3), 9, 1, 1}, {16 * 81, 16ull * (cuuint64_t)ipow(9, L - 1), big, big}, {162, 3, 9, 1, 1});
        break;
    case 2:  // [slots 0..p0-1][d0][d1][slots p0+2..L-1]
        set({2ull * (cuuint64_t)ipow(9, p0), 9, 9, (cuuint64_t)ipow(9, L - 2 - p0), 1},
            {16ull * (cuuint64_t)ipow(9, p0), 16ull * (cuuint64_t)ipow(9, p0 + 1), 16ull * (cuuint64_t)ipow(9, p0 + 2), big},
            {54, 9, 9, 1, 1});
        break;
    default:  // p0 = 1: [slot 0, d0 = slot 1][d1 = slot 2][slots 3..L-1]
        set({162, 9, (cuuint64_t)ipow(9, L - 3), 1, 1}, {16 * 81, 16 * 729, big, big}, {162, 9, 3, 1, 1});
        break;
    }
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    if (enc(&ls.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void *)A, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    ls.tma_A = A;
    return true;
}

// TMA fields of one launch of set ls on the ARDM (or local shard block) A; d_work w holds the tables.
static qp_status set_tma(const qp_plan &P, const qp_plan::LaunchSet &ls, qp::FusedArgs &a, double2 *A, char *w) {
    a.use_tma = 0;
    if (ls.f2t >= 0) {
        if (!encode_f2t_tmap(P, ls, A)) return err(QP_ERR_CUDA, "cuda: cannot encode the k_fused2t tensor map (p0 = %d)", ls.p0);
        a.use_tma = 1;
        a.tmap = ls.tmap;
        a.f4_layout = ls.f2t;
        // unit G (first outer fibre) = cB nA + cA: run A (VK 2, 3) as doubles in box dimension 0, the rest in
        // dimension cdimB; VK 0, 1: one coordinate G
        // (VK 1, 3: the unit's 27 fibres are all 9 values of the lowest outer slot x 3 of the next ones: the
        // merged box dimension 0 starts at 0, dimension cdimB at G / 9)
        a.tma_nA = ls.f2t == 2 ? ipow(P.N, ls.f2t_p0) : (ls.f2t == 0 ? 0 : P.N);
        a.tma_c0m = 2;
        a.f4_cdimA[0] = ls.f2t == 0 ? -1 : 0;
        a.f4_cdimB[0] = ls.f2t == 2 ? 3 : (ls.f2t == 3 ? 2 : 1);
        a.E0r = (const double2 *)(w + ls.off_E0r);
        return QP_OK;
    }
    if (ls.S == 4) {
        if (!ls.f4 || !encode_f4_tmaps(ls, A)) return err(QP_ERR_CUDA, "cuda: cannot encode the k_fused4 tensor maps (p0 = %d)", ls.p0);
        a.use_tma = 1;
        a.tmap = ls.tmap;
        a.tmapS = ls.tmapS;
        for (int i = 0; i < 11; ++i) a.f4_lpos[i] = ls.f4map[0].pos[i], a.f4_spos[i] = ls.f4map[1].pos[i];
        a.f4_q1swap = ls.f4map[0].lane_swap;
        a.f4_q2swap = ls.f4map[1].lane_swap;
        a.f4_colregion = ls.f4_col;
        a.f4_swz = ls.f4_swz;
        a.f4_layout = qp::fused4_layout_type(a.f4_lpos, a.f4_spos, a.f4_q1swap, a.f4_q2swap, a.f4_swz);
        for (int m = 0; m < 2; ++m) a.f4_cdimA[m] = ls.f4map[m].cdimA, a.f4_cdimB[m] = ls.f4map[m].cdimB;
        a.tma_nA = ls.f4_nA;
        a.tma_nA_log2 = -1;
        for (int b = 0; b < 62; ++b)
            if ((1LL << b) == a.tma_nA) a.tma_nA_log2 = b;
        a.tma_c0m = ls.f4_c0m;
        a.E0r = (const double2 *)(w + ls.off_E0r);
        return QP_OK;
    }
    if (ls.tma_a != -1 && ls.S == 3 && encode_f3_tmap(P, ls, A, ls.e0r_F)) {
        a.use_tma = 1;
        a.tmap = ls.tmap;
        // TMA box coordinates of unit G (first outer fibre): c0 = tma_c0m (G mod tma_nA), c1 = G / tma_nA
        // (view A: run A as doubles; view B: rows of two fibres; views C, D: one fibre per row group)
        a.tma_nA = ls.tma_a > 0 ? ipow(P.N, ls.tma_a) : (ls.tma_a == 0 ? 2 : 1);
        a.tma_nA_log2 = -1;
        for (int b = 0; b < 62; ++b)
            if ((1LL << b) == a.tma_nA) a.tma_nA_log2 = b;
        a.tma_c0m = ls.tma_a > 0 ? 2 : 0;
        a.tma_view = ls.tma_a > 0 ? 0 : (ls.tma_a == 0 ? 1 : (ls.tma_a == -2 ? 2 : 3));
        a.E0r = (const double2 *)(w + ls.off_E0r);
    }
    return QP_OK;
}

// Tables of one fused launch over inner slots p0..p0+S-1 (mod L) of a local layout from which the
// shard slots `removed` are absent (empty for an unsharded plan).
void build_launch_set(const qp_plan &P, int p0, int S, const std::vector<int> &removed, qp_plan::LaunchSet &ls) {
    const int N = P.N, M = P.M, L = P.L, D = P.D;
    ls.p0 = p0;
    ls.S = S;
    std::vector<int> inner(S), outer;
    for (int i = 0; i < S; ++i) inner[i] = (p0 + i) % L;
    // shard slots (removed) are not stored: the remaining slots keep their order, slot q sits at
    // position pos[q] of the local layout (stride N^pos[q])
    std::vector<int> pos(L, -1);
    for (int q = 0, n = 0; q < L; ++q)
        if (std::find(removed.begin(), removed.end(), q) == removed.end()) pos[q] = n++;
    for (int q = 0; q < L; ++q)
        if (pos[q] >= 0 && std::find(inner.begin(), inner.end(), q) == inner.end()) outer.push_back(q);  // ascending
    const int nout = (int)outer.size();
    // tile digits: the kernel's preferred v, lowered (not below its minimum) so that small problems
    // still have >= ~2 tiles per SM of a 148-SM B200 to spread over the persistent grid
    const bool f3 = (M == 2 && S == 3), f4 = (M == 2 && S == 4), f2s = (M == 3 && S == 2);
    int v = std::min(f4 ? 4 : (f3 ? qp::kFused3TileDigits : (f2s ? 3 : qp::fused_r_tile_digits(M, S))), nout);
    const int vmin = std::min(f4 ? 2 : (f3 ? qp::kFused3TileDigitsMin : (N >= 9 ? 2 : 3)), nout);
    while (v > vmin && std::pow((double)N, nout - v) < 2.0 * 148) --v;
    const int w = std::max(1, P.group_w);
    const int hi = nout - v;
    const int G = 1 + (hi + w - 1) / w;
    const int T = (int)ipow(N, v);
    int X = T;
    for (int g = 1; g < G; ++g) X = std::max<int>(X, (int)ipow(N, std::min(w, hi - (g - 1) * w)));
    auto g_first = [&](int g) { return g == 0 ? 0 : v + (g - 1) * w; };
    auto g_size = [&](int g) { return g == 0 ? v : std::min(w, hi - (g - 1) * w); };
    // outer digit group tables: per sub-step s, kind kap, exponent over the group's digits
    // entry x of group g is exp(delta_d sum_t psi(digit_t of x; lag of digit t)) = the product of per-digit
    // factors exp(delta_d psi(digit; lag)) (kap 0: eta of the lag, propagate; kap 1: E of the lag, terminal)
    ls.Etab.assign((size_t)S * 2 * G * D * X, make_double2(1.0, 0.0));
    for (int st = 0; st < S; ++st)
        for (int g = 0; g < G; ++g) {
            const int i0 = g_first(g), nd = g_size(g);
            std::vector<cd> fac((size_t)2 * D * nd * N);  // [kap][d][t][dig]
            for (int t = 0; t < nd; ++t) {
                const int lag = ((p0 + st - outer[i0 + t]) % L + L) % L;  // 1..L-1
                for (int dig = 0; dig < N; ++dig)
                    for (int kap = 0; kap < 2; ++kap)
                        for (int d = 0; d < D; ++d)
                            fac[(((size_t)kap * D + d) * nd + t) * N + dig] =
                                std::exp(P.delta[d] * psi(P, dig, kap == 0 ? P.eta[lag] : P.E[lag]));
            }
            for (int kap = 0; kap < 2; ++kap)
                for (int d = 0; d < D; ++d) {
                    const cd *fk = fac.data() + ((size_t)kap * D + d) * nd * N;
                    double2 *out = ls.Etab.data() + ((((size_t)st * 2 + kap) * G + g) * D + d) * X;
                    for (int x = 0; x < (int)ipow(N, nd); ++x) {
                        double er = 1.0, ei = 0.0;  // plain complex products (no __muldc3 special-value path)
                        int r = x;
                        for (int t = 0; t < nd; ++t, r /= N) {
                            const cd f = fk[(size_t)t * N + r % N];
                            const double nr = er * f.real() - ei * f.imag();
                            ei = er * f.imag() + ei * f.real();
                            er = nr;
                        }
                        out[x] = make_double2(er, ei);
                    }
                }
        }
    // inner-slot factors: sub-step st, inner digit i != st (new value if i < st, old if i > st)
    ls.inner.assign((size_t)S * S * 2 * D * N, make_double2(1.0, 0.0));
    for (int st = 0; st < S; ++st)
        for (int i = 0; i < S; ++i) {
            if (i == st) continue;
            const int lag = i < st ? st - i : L - (i - st);
            for (int kap = 0; kap < 2; ++kap)
                for (int d = 0; d < D; ++d)
                    for (int sg = 0; sg < N; ++sg)
                        ls.inner[((((size_t)st * S + i) * 2 + kap) * D + d) * N + sg] =
                            d2(std::exp(P.delta[d] * psi(P, sg, kap == 0 ? P.eta[lag] : P.E[lag])));
        }
    // address offsets of the outer digit groups g >= 1 and of the tile-local fibres
    ls.goff.assign((size_t)G * X, 0);
    for (int g = 1; g < G; ++g) {
        const int i0 = g_first(g), nd = g_size(g);
        for (int x = 0; x < (int)ipow(N, nd); ++x) {
            long long o = 0;
            int r = x;
            for (int t = 0; t < nd; ++t) { o += (long long)(r % N) * ipow(N, pos[outer[i0 + t]]); r /= N; }
            ls.goff[(size_t)g * X + x] = o;
        }
    }
    const int qlast = (p0 - 1 + L) % L;  // sub-step 0's 'last' point sigma_{k-1}
    const int ilast = (int)(std::find(outer.begin(), outer.end(), qlast) - outer.begin());
    ls.lofs.assign(T, make_int2(0, -1));
    for (int fl = 0; fl < T; ++fl) {
        long long o = 0;
        int r = fl;
        for (int t = 0; t < v; ++t) { o += (long long)(r % N) * ipow(N, pos[outer[t]]); r /= N; }
        const int lastd = ilast < v ? (int)((fl / ipow(N, ilast)) % N) : -1;
        ls.lofs[fl] = make_int2((int)o, lastd);
    }
    qp::FusedArgs &a = ls.args;
    for (int i = 0; i < S; ++i) a.pw_in[i] = ipow(N, pos[inner[i]]);
    a.n_tiles = (int)ipow(N, hi);
    a.T = T;
    a.G = G;
    a.X = X;
    for (int g = 1; g < G; ++g) {
        a.gdiv[g] = (int)ipow(N, (g - 1) * w);
        a.gmod[g] = (int)ipow(N, g_size(g));
    }
    a.last_div = (ilast >= v && ilast < nout) ? (int)ipow(N, ilast - v) : -1;
    a.fixed_last = -1;  // set per launch when sub-step 0's 'last' slot is a shard slot
    // k_fused3 plain loads: lane map 1 (32 consecutive fibres per warp load) when fibres t, t+1 are adjacent
    a.lane_map = (T >= 64 && ls.lofs[1].x == 1) ? 1 : 0;
    // per-warp TMA staging (k_fused3, unsharded): the view follows from where ring slot 0 sits.
    // View A: slot 0 is the lowest outer slot, the outer slots are two runs of consecutive slots,
    // A = 0 .. p0-1 and B = p0+3 .. L-1; views B/C/D: inner digit 2/1/0 is slot 0 (p0 = L-2/L-1/0)
    ls.tma_a = -1;  // (-1: no TMA view; > 0: view A; 0: view B; -2: view C; -3: view D)
    if (f3 && removed.empty() && T >= 64 && !(P.flags & QP_FLAG_NO_TMA)) {
        if (a.lane_map == 1 && p0 >= 1 && p0 + S <= L) ls.tma_a = p0, ls.tma_b = L - p0 - S;
        else if (p0 == L - 2 && L >= 6) ls.tma_a = 0, ls.tma_b = 0;
        else if (p0 == L - 1 && L >= 6) ls.tma_a = -2, ls.tma_b = 0;
        else if (p0 == 0 && L >= 6) ls.tma_a = -3, ls.tma_b = 0;
    }
    ls.E0r.clear();
    ls.e0r_F = 0;
    if (ls.tma_a != -1) {
        // the stage is read with lane map 0 (the quarters of a super-fibre in one warp); per (round, warp)
        // unit of F = 8 fibres one contiguous block of the group-0 factors [S][2][D][F] and the F
        // tile-local offsets (one bulk copy per unit)
        a.lane_map = 0;
        const int F = 8;
        const int R = T / F, Q = S * 2 * D;
        const size_t blk = (size_t)Q * F + F / 2;
        ls.E0r.assign((size_t)R * blk, make_double2(0.0, 0.0));
        for (int rd = 0; rd < R; ++rd) {
            double2 *b = ls.E0r.data() + rd * blk;
            for (int q = 0; q < Q; ++q) {  // q = (st, kap, d): Etab[st][kap][g = 0][d][rd F + f]
                const int st = q / (2 * D), kap = (q / D) % 2, d = q % D;
                for (int f = 0; f < F; ++f) b[(size_t)q * F + f] = ls.Etab[((((size_t)st * 2 + kap) * G) * D + d) * X + rd * F + f];
            }
            std::memcpy(b + (size_t)Q * F, ls.lofs.data() + (size_t)rd * F, F * sizeof(int2));
        }
        ls.e0r_F = F;
    }
    a.use_tma = 0;
    ls.f4 = false;
    if (f4) {
        // k_fused4: one E0 block per 8-fibre round of a tile: factors [s][kap][c][f] + the 8 lofs (int2)
        if (f4_layout(P, ls, pos, inner, outer) && T % 8 == 0 && T >= 16) {  // >= 2 rounds per tile (slide4.cu ring depth)
            ls.f4 = true;
            const int F = 8, R = T / F, Q = S * 2 * D;
            const size_t blk = (size_t)Q * F + F / 2;
            ls.E0r.assign((size_t)R * blk, make_double2(0.0, 0.0));
            for (int rd = 0; rd < R; ++rd) {
                double2 *b = ls.E0r.data() + rd * blk;
                for (int q = 0; q < Q; ++q) {
                    const int st = q / (2 * D), kap = (q / D) % 2, d = q % D;
                    for (int f = 0; f < F; ++f) b[(size_t)q * F + f] = ls.Etab[((((size_t)st * 2 + kap) * G) * D + d) * X + rd * F + f];
                }
                std::memcpy(b + (size_t)Q * F, ls.lofs.data() + (size_t)rd * F, F * sizeof(int2));
            }
            ls.e0r_F = F;
        }
    }
    ls.f2t = -1;
    const int Lloc = L - (int)removed.size();
    if (f2s && P.sym3 && !(P.flags & QP_FLAG_NO_TMA) && Lloc >= 4 && T % 27 == 0 && T / 27 >= 3) {
        // k_fused2t: one block per 27-fibre unit of a tile: factors [s][kap][d][f] + the 27 lofs (int2).
        // The view follows from the local positions of the inner digits (a shard block's layout has the
        // shard slots removed; the inner slots are never shard slots)
        const int l0 = pos[inner[0]], l1 = pos[inner[1]];
        ls.f2t = (l0 == 0 && l1 == 1) ? 0 : ((l0 == Lloc - 1 && l1 == 0) ? 1 : (l0 == 1 ? 3 : 2));
        ls.f2t_p0 = l0, ls.f2t_L = Lloc;
        const int F = qp::fused2t_unit_fibres(), R = T / F, Q = S * 2 * D;
        const size_t blk = (size_t)qp::fused2t_e0_block();
        ls.E0r.assign((size_t)R * blk, make_double2(0.0, 0.0));
        for (int rd = 0; rd < R; ++rd) {
            double2 *b = ls.E0r.data() + rd * blk;
            for (int q = 0; q < Q; ++q) {
                const int st = q / (2 * D), kap = (q / D) % 2, d = q % D;
                for (int f = 0; f < F; ++f) b[(size_t)q * F + f] = ls.Etab[((((size_t)st * 2 + kap) * G) * D + d) * X + rd * F + f];
            }
            std::memcpy(b + (size_t)Q * F, ls.lofs.data() + (size_t)rd * F, F * sizeof(int2));
        }
        ls.e0r_F = F;
    }
    for (int st = 0; st < qp::kMaxS; ++st)
        for (int kap = 0; kap < 2; ++kap)
            for (int d = 0; d < qp::kMaxD; ++d) a.fixfac[st][kap][d] = make_double2(1.0, 0.0);

}

void compute_layout(qp_plan &P) {
    const int N = P.N;
    size_t off = 0;
    P.off_small = off; off = align256(off + P.small.size() * sizeof(double2));
    auto place = [&](qp_plan::LaunchSet &ls) {
        ls.off_inner = off; off = align256(off + ls.inner.size() * sizeof(double2));
        ls.off_E = off;     off = align256(off + ls.Etab.size() * sizeof(double2));
        ls.off_goff = off;  off = align256(off + ls.goff.size() * sizeof(long long));
        ls.off_lofs = off;  off = align256(off + ls.lofs.size() * sizeof(int2));
        ls.off_E0r = off;   off = align256(off + ls.E0r.size() * sizeof(double2));
    };
    for (auto &ls : P.sets) place(ls);
    for (auto &ls : P.sh.sets) place(ls);
    P.tables_end = off;
    P.off_part = off;  off = align256(off + (size_t)qp::kMaxS * qp::kPartialsMax * N * sizeof(double2));
    P.off_rho = off;   off = align256(off + std::max<size_t>(1, P.out_steps.size()) * N * sizeof(double2));
    P.off_cnt = off;   off = align256(off + 256);
    if (P.persist) {
        P.off_psets = off; off = align256(off + P.sets.size() * sizeof(qp::FusedArgs));
        P.off_pslot = off; off = align256(off + (size_t)(P.n_steps + 1) * sizeof(int));
    }
    P.work_bytes = off;
}

void build_tables(qp_plan &P, int fuse_cap) {
    const int N = P.N, M = P.M, L = P.L, D = P.D;
    // ---- K and self-factor-weighted K'
    P.K.assign(N * N, 0.0);
    for (int a1 = 0; a1 < M; ++a1)
        for (int b1 = 0; b1 < M; ++b1)
            for (int a = 0; a < M; ++a)
                for (int b = 0; b < M; ++b)
                    P.K[(a1 * M + b1) * N + (a * M + b)] = P.U[a1 * M + a] * std::conj(P.U[b1 * M + b]);
    const qp::SmallLayout lay{N, D, L};
    P.small.assign(lay.total(), make_double2(0, 0));
    const cd selfc[2] = {P.self_int, P.self_end};
    for (int kap = 0; kap < 2; ++kap)
        for (int nw = 0; nw < N; ++nw) {
            const cd c = std::exp(dsig(P, nw) * psi(P, nw, selfc[kap]));  // I(new,new; eta_self)
            for (int last = 0; last < N; ++last) P.small[lay.kp(kap) + nw * N + last] = d2(c * P.K[nw * N + last]);
        }
    // ---- beta_d(old) = exp(delta_d psi_L(old)) : variant 0 (k > L), 1 (k == L, partner sigma_0)
    const cd lagL[2][2] = {{P.eta[L], P.E[L]}, {P.E[L], P.TI[L]}};
    for (int var = 0; var < 2; ++var)
        for (int kap = 0; kap < 2; ++kap)
            for (int d = 0; d < D; ++d)
                for (int old = 0; old < N; ++old)
                    P.small[lay.beta(var, kap) + d * N + old] = d2(std::exp(P.delta[d] * psi(P, old, lagL[var][kap])));
    // ---- growth exponent rows psi_{k,j}(sigma), k = 1..L-1, j = 1..k
    for (int k = 1; k < L; ++k)
        for (int j = 1; j <= k; ++j) {
            const cd ep = (j < k) ? P.eta[j] : P.E[k];
            const cd et = (j < k) ? P.E[j] : P.TI[k];
            for (int sg = 0; sg < N; ++sg) {
                P.small[lay.psi(0) + ((size_t)k * L + j) * N + sg] = d2(psi(P, sg, ep));
                P.small[lay.psi(1) + ((size_t)k * L + j) * N + sg] = d2(psi(P, sg, et));
            }
        }
    // ---- fused launch sets: for every start slot p0 and fusion depth S, the super-fibres of the
    //      inner slots p0..p0+S-1 and the factor / address tables of the L-S outer slots
    // fusion depth: three steps per pass for M = 2 (k_fused3), one for M = 3, 4 (k_fused_r); the
    // caller may cap it (qp_problem.fuse_steps)
    P.group_w = (M == 2) ? 4 : (M == 3 ? 3 : 2);
    // M = 2: four fused steps per pass (k_fused4, TMA load and store) when the outer slots hold at
    // least two digits (L >= 6), else three (k_fused3)
    const int s2 = (L >= 6 && !(P.flags & QP_FLAG_NO_TMA)) ? 4 : 3;
    P.Smax = std::max(1, std::min(M == 2 ? s2 : (M == 3 ? 2 : 1), L - 1));
    // persistent path (persist.cu): a small ARDM runs each qp_steps call in one single-CTA launch with
    // everything in shared memory, one step at a time -- there the launch, not the bandwidth, is the
    // cost of a step
    P.persist = !(P.flags & QP_FLAG_NO_PERSIST) && 16.0 * std::pow((double)N, (double)L) <= (double)QP_PERSIST_MAX_BYTES;
    if (P.persist) P.Smax = 1;
    if (fuse_cap > 0) P.Smax = std::min(P.Smax, fuse_cap);
    P.sets.assign((size_t)L * P.Smax, qp_plan::LaunchSet{});
    {  // the L * Smax launch sets are independent (read-only plan, own tables): build them on host threads
        const int nset = L * P.Smax;
        const int nth = (int)std::max(1u, std::min<unsigned>((unsigned)nset, std::min(16u, std::thread::hardware_concurrency())));
        std::atomic<int> next{0};
        auto worker = [&] {
            for (int i = next++; i < nset; i = next++) build_launch_set(P, i / P.Smax, i % P.Smax + 1, {}, P.sets[(size_t)i]);
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
        worker();
        for (auto &th : pool) th.join();
    }
    // ---- A_0(sigma_0) = rho0(sigma_0) I(sigma_0, sigma_0; eta_00 = G(1/2))   (Eq. 13, reading C.3-2)
    P.A0.assign(N, 0.0);
    for (int sg = 0; sg < N; ++sg) P.A0[sg] = P.rho0[sg] * std::exp(dsig(P, sg) * psi(P, sg, P.self_end));
    compute_layout(P);
}

// Capacity (a1): need bytes against the caller's budget (max_bytes > 0), or against the free memory
// of the current CUDA device (max_bytes == 0; no check when no device is visible), or no check
// (max_bytes < 0).
qp_status check_capacity(int64_t max_bytes, double need, const char *what) {
    double budget = -1.0;
    const char *src = "budget";
    if (max_bytes > 0) {
        budget = (double)max_bytes;
    } else if (max_bytes == 0) {
        int n = 0;
        size_t fr = 0, tot = 0;
        if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0 && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
            budget = (double)fr;
            src = "free device memory";
        } else {
            cudaGetLastError();  // no device visible: nothing to check against
        }
    }
    if (budget >= 0.0 && need > budget)
        return err(QP_ERR_CAPACITY, "capacity: need %.0f B (%s) > %s %.0f B", need, what, src, budget);
    return QP_OK;
}

qp_status validate(const qp_problem *pr) {
    if (!pr) return err(QP_ERR_ARG, "arg: problem is NULL");
    const int M = pr->M;
    if (M < 2 || M > qp::kMaxM) return err(QP_ERR_CONFIG, "config: GPU path supports 2 <= M <= %d (got %d)", qp::kMaxM, M);
    if (!pr->s || !pr->H || !pr->rho0) return err(QP_ERR_ARG, "arg: s, H and rho0 are required");
    if (pr->dkmax < 2 || pr->dkmax > qp::kMaxL) return err(QP_ERR_CONFIG, "config: dkmax must be in [2, %d] (got %d)", qp::kMaxL, pr->dkmax);
    if (!(pr->dt > 0.0) || !std::isfinite(pr->dt)) return err(QP_ERR_CONFIG, "config: dt must be finite and > 0");
    if (pr->n_steps < 0) return err(QP_ERR_CONFIG, "config: n_steps must be >= 0");
    double hmax = 0.0, rmax = 0.0;
    cd tr = 0.0;
    for (int i = 0; i < M; ++i) {
        if (!std::isfinite(pr->s[i])) return err(QP_ERR_CONFIG, "config: s[%d] not finite", i);
        for (int j = 0; j < M; ++j) {
            const cd h = {pr->H[i * M + j].re, pr->H[i * M + j].im}, hT = {pr->H[j * M + i].re, pr->H[j * M + i].im};
            const cd r = {pr->rho0[i * M + j].re, pr->rho0[i * M + j].im}, rT = {pr->rho0[j * M + i].re, pr->rho0[j * M + i].im};
            hmax = std::max(hmax, std::abs(h - std::conj(hT)));
            rmax = std::max(rmax, std::abs(r - std::conj(rT)));
        }
        tr += cd(pr->rho0[i * M + i].re, pr->rho0[i * M + i].im);
    }
    if (!(hmax <= 1e-12)) return err(QP_ERR_CONFIG, "config: H not Hermitian (max |H - H^+| = %.3g)", hmax);
    if (!(rmax <= 1e-12)) return err(QP_ERR_CONFIG, "config: rho0 not Hermitian (max |rho0 - rho0^+| = %.3g)", rmax);
    if (!(std::abs(tr - 1.0) <= 1e-12)) return err(QP_ERR_CONFIG, "config: trace(rho0) = %.17g%+.3gi, must be 1", tr.real(), tr.imag());
    switch (pr->kind) {
    case QP_J_ZERO: break;
    case QP_J_OHMIC_EXP: case QP_J_DEBYE: case QP_J_SUPEROHMIC_GAUSS:
        if (!(pr->omega_c > 0.0)) return err(QP_ERR_CONFIG, "config: omega_c must be > 0");
        if (!(pr->kT >= 0.0)) return err(QP_ERR_CONFIG, "config: kT must be >= 0");
        break;
    case QP_J_CALLBACK:
        if (!pr->J || !(pr->J_cutoff > 0.0)) return err(QP_ERR_CONFIG, "config: callback bath needs J and J_cutoff > 0");
        if (!(pr->kT >= 0.0)) return err(QP_ERR_CONFIG, "config: kT must be >= 0");
        break;
    case QP_J_G_TABLE:
        if (!pr->G_in) return err(QP_ERR_CONFIG, "config: G_TABLE bath needs G_in[2*dkmax+3]");
        break;
    case QP_J_ETA_TABLE:
        if (!pr->eta_in) return err(QP_ERR_CONFIG, "config: ETA_TABLE bath needs eta_in[3*dkmax+2]");
        for (int i = 0; i < 3 * pr->dkmax + 2; ++i)
            if (!std::isfinite(pr->eta_in[i].re) || !std::isfinite(pr->eta_in[i].im))
                return err(QP_ERR_CONFIG, "config: eta_in[%d] not finite", i);
        break;
    default: return err(QP_ERR_CONFIG, "config: unknown bath kind %d", pr->kind);
    }
    if (pr->fuse_steps < 0 || pr->fuse_steps > 4) return err(QP_ERR_CONFIG, "config: fuse_steps must be in [0, 4] (got %d)", pr->fuse_steps);
    if (pr->flags & ~(uint32_t)(QP_FLAG_NO_TMA | QP_FLAG_GENERIC_MOMENTS | QP_FLAG_NO_PERSIST))
        return err(QP_ERR_CONFIG, "config: unknown flags 0x%x", pr->flags);
    if (pr->out_steps) {
        if (pr->n_out < 0) return err(QP_ERR_CONFIG, "config: n_out must be >= 0 (got %lld)", (long long)pr->n_out);
        for (int64_t o = 0; o < pr->n_out; ++o) {
            const int64_t k = pr->out_steps[o];
            if (k < 0 || k > pr->n_steps || (o > 0 && k <= pr->out_steps[o - 1]))
                return err(QP_ERR_CONFIG, "config: out_steps must be sorted, unique and within [0, n_steps]");
        }
    }
    // N^L must fit comfortably in int64 and the 32-bit tile indices
    const double ent = std::pow(double(M * M), double(pr->dkmax));
    if (ent > 4.0e12) return err(QP_ERR_CAPACITY, "capacity: need %.4g B for the ARDM (N^L = %.4g entries)", 16.0 * ent, ent);
    return QP_OK;
}

}  // namespace

// ===================================================================================== C ABI
extern "C" {

const char *qp_last_error(void) { return g_err.c_str(); }
const char *qp_version(void) { return "quapi 0.1 sm_100a"; }

qp_status qp_plan_create(const qp_problem *pr, qp_plan **out) {
    if (!out) return err(QP_ERR_ARG, "arg: out is NULL");
    *out = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    qp_status st = validate(pr);
    if (st) return st;
    qp_plan *P = new (std::nothrow) qp_plan();
    if (!P) return err(QP_ERR_CAPACITY, "capacity: host allocation failed");
    P->M = pr->M;
    P->N = pr->M * pr->M;
    P->L = pr->dkmax;
    P->dt = pr->dt;
    P->n_steps = pr->n_steps;
    P->flags = pr->flags;
    if (pr->out_steps) P->out_steps.assign(pr->out_steps, pr->out_steps + pr->n_out);
    else for (int64_t k = 0; k <= pr->n_steps; ++k) P->out_steps.push_back(k);
    P->s.assign(pr->s, pr->s + P->M);
    P->H.resize(P->M * P->M);
    P->rho0.resize(P->M * P->M);
    for (int i = 0; i < P->M * P->M; ++i) {
        P->H[i] = cd(pr->H[i].re, pr->H[i].im);
        P->rho0[i] = cd(pr->rho0[i].re, pr->rho0[i].im);
    }
    std::vector<cd> X(P->M * P->M);
    for (int i = 0; i < P->M * P->M; ++i) X[i] = cd(0.0, -P->dt) * P->H[i];
    P->U = expm_taylor(X, P->M);
    build_classes(*P);
    const auto t1 = std::chrono::steady_clock::now();
    if ((st = compute_eta(*P, *pr))) { delete P; return st; }
    const auto t2 = std::chrono::steady_clock::now();
    build_tables(*P, pr->fuse_steps);
    for (const auto &ls : P->sets)
        if (ls.S == 4 && !ls.f4) {
            const int p0 = ls.p0;
            delete P;
            return err(QP_ERR_CONFIG, "internal: no k_fused4 stage layout for p0 = %d", p0);
        }
    const auto t3 = std::chrono::steady_clock::now();
    P->setup_ms[0] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    P->setup_ms[1] = std::chrono::duration<double, std::milli>(t2 - t1).count();
    P->setup_ms[2] = std::chrono::duration<double, std::milli>(t3 - t2).count();
    P->ardm_entries = ipow(P->N, P->L);
    P->max_bytes = pr->max_bytes;
    const double need = 16.0 * double(P->ardm_entries) + double(P->work_bytes);
    if (pr->max_bytes > 0 && (st = check_capacity(pr->max_bytes, need, "ARDM + workspace"))) {  // explicit budget
        delete P;
        return st;
    }
    P->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = P;
    return QP_OK;
}

void qp_plan_destroy(qp_plan *P) { delete P; }

qp_status qp_plan_check(const qp_plan *P) {
    if (!P) return err(QP_ERR_ARG, "arg: NULL plan");
    const double need = P->sh.on ? 2.0 * 16.0 * double(P->sh.n_own[P->sh.rank] * P->sh.blk) + double(P->work_bytes)
                                 : 16.0 * double(P->ardm_entries) + double(P->work_bytes);
    return check_capacity(P->max_bytes, need, P->sh.on ? "two shard buffers + workspace" : "ARDM + workspace");
}

qp_status qp_plan_query(const qp_plan *P, qp_sizes *o) {
    if (!P || !o) return err(QP_ERR_ARG, "arg: NULL plan or out");
    o->M = P->M; o->N = P->N; o->L = P->L;
    o->ardm_entries = P->ardm_entries;
    o->ardm_bytes = 16 * P->ardm_entries;
    o->work_bytes = (int64_t)P->work_bytes;
    o->pmc_bytes = 64.0 * std::pow(double(P->M), 2.0 * (P->L + 1));
    o->n_out = (int64_t)P->out_steps.size();
    o->n_steps = P->n_steps;
    o->bytes_per_step = 32 * P->ardm_entries;
    o->lattice = P->lattice;
    o->n_classes = P->D;
    o->grid = P->grid[P->Smax];
    o->block = P->block;
    o->tile_fibres = P->sets.empty() ? 0 : P->sets[(size_t)P->Smax - 1].args.T;
    o->fuse_steps = P->Smax;
    o->persistent = (P->persist && (!P->inited || P->small_dyn)) ? 1 : 0;
    o->setup_seconds = P->setup_seconds;
    for (int i = 0; i < 3; ++i) o->setup_ms[i] = P->setup_ms[i];
    o->init_h2d_bytes = (int64_t)(P->tables_end + 2 * P->N * sizeof(double2));
    return QP_OK;
}

qp_status qp_plan_eta(const qp_plan *P, qp_c64 *out, int64_t cap) {
    if (!P || !out) return err(QP_ERR_ARG, "arg: NULL plan or out");
    if (cap < 3 * P->L + 2) return err(QP_ERR_ARG, "arg: eta output needs %d entries", 3 * P->L + 2);
    auto put = [&](int i, cd z) { out[i].re = z.real(); out[i].im = z.imag(); };
    put(0, P->self_int);
    put(1, P->self_end);
    for (int j = 1; j <= P->L; ++j) {
        put(1 + j, P->eta[j]);
        put(1 + P->L + j, P->E[j]);
        put(1 + 2 * P->L + j, P->TI[j]);
    }
    return QP_OK;
}

static qp_status validate_bath(const qp_bath &q, int b) {
    if (q.kind < QP_J_ZERO || q.kind > QP_J_SUPEROHMIC_GAUSS)
        return err(QP_ERR_CONFIG, "config: bath %d: kind %d has no device quadrature (analytic families 0..3 only)", b, q.kind);
    if (q.kind != QP_J_ZERO) {
        if (!(q.omega_c > 0.0) || !std::isfinite(q.omega_c)) return err(QP_ERR_CONFIG, "config: bath %d: omega_c must be > 0", b);
        if (!(q.kT >= 0.0) || !std::isfinite(q.kT)) return err(QP_ERR_CONFIG, "config: bath %d: kT must be >= 0", b);
        if (!std::isfinite(q.coupling)) return err(QP_ERR_CONFIG, "config: bath %d: coupling not finite", b);
    }
    return QP_OK;
}

// enqueue k_eta over B baths (chunks of kEtaBatchMax): d_eta [B][3L+2]
static qp_status enqueue_eta(const qp_bath *baths, int B, double dt, int L, double2 *d_eta, double *d_err, cudaStream_t s) {
    const size_t nc = 3 * (size_t)L + 2;
    static thread_local qp::EtaBatch batch;  // 16 KB kernel parameter block
    for (int b0 = 0; b0 < B; b0 += qp::kEtaBatchMax) {
        const int nb = std::min(B - b0, qp::kEtaBatchMax);
        for (int i = 0; i < nb; ++i) {
            const qp_bath &q = baths[b0 + i];
            batch.b[i] = qp::EtaBath{q.kind, q.coupling, q.omega_c, q.kT};
        }
        const cudaError_t e = qp::launch_eta(batch, nb, L, dt, d_eta + (size_t)b0 * nc, d_err ? d_err + (size_t)b0 * nc : nullptr, s);
        if (e != cudaSuccess) return err(QP_ERR_CUDA, "cuda: eta launch: %s", cudaGetErrorString(e));
    }
    return QP_OK;
}

qp_status qp_eta_device(const qp_bath *baths, int32_t B, double dt, int32_t L, qp_c64 *d_eta, double *d_err,
                        void *stream) {
    if (!baths || !d_eta) return err(QP_ERR_ARG, "arg: NULL baths or d_eta");
    if (B < 1) return err(QP_ERR_ARG, "arg: B must be >= 1 (got %d)", B);
    if (!(dt > 0.0) || !std::isfinite(dt)) return err(QP_ERR_ARG, "arg: dt must be finite and > 0");
    if (L < 1 || L > qp::kMaxL) return err(QP_ERR_ARG, "arg: dkmax must be in [1, %d] (got %d)", qp::kMaxL, L);
    for (int b = 0; b < B; ++b)
        if (qp_status st = validate_bath(baths[b], b)) return st;
    return enqueue_eta(baths, B, dt, L, reinterpret_cast<double2 *>(d_eta), d_err, (cudaStream_t)stream);
}

qp_status qp_plan_propagator(const qp_plan *P, qp_c64 *U) {
    if (!P || !U) return err(QP_ERR_ARG, "arg: NULL plan or out");
    for (int i = 0; i < P->M * P->M; ++i) { U[i].re = P->U[i].real(); U[i].im = P->U[i].imag(); }
    return QP_OK;
}

qp_status qp_init(qp_plan *P, void *d_ardm, void *d_work, void *stream) {
    if (!P || !d_ardm || !d_work) return err(QP_ERR_ARG, "arg: NULL plan or device buffer");
    if ((uintptr_t)d_ardm % 16 || (uintptr_t)d_work % 256) return err(QP_ERR_ARG, "arg: misaligned device buffer");
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    QP_CUDA(cudaGetDevice(&dev));
    QP_CUDA(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, dev));
    char *w = (char *)d_work;
    QP_CUDA(cudaMemcpyAsync(w + P->off_small, P->small.data(), P->small.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    std::vector<const qp_plan::LaunchSet *> all;
    for (const auto &ls : P->sets) all.push_back(&ls);
    for (const auto &ls : P->sh.sets) all.push_back(&ls);
    for (const auto *lsp : all) {
        const auto &ls = *lsp;
        QP_CUDA(cudaMemcpyAsync(w + ls.off_inner, ls.inner.data(), ls.inner.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaMemcpyAsync(w + ls.off_E, ls.Etab.data(), ls.Etab.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaMemcpyAsync(w + ls.off_goff, ls.goff.data(), ls.goff.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaMemcpyAsync(w + ls.off_lofs, ls.lofs.data(), ls.lofs.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
        if (!ls.E0r.empty())
            QP_CUDA(cudaMemcpyAsync(w + ls.off_E0r, ls.E0r.data(), ls.E0r.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    }
    QP_CUDA(cudaMemsetAsync(w + P->off_cnt, 0, 256, s));
    std::vector<double2> a0(P->N);
    for (int i = 0; i < P->N; ++i) a0[i] = d2(P->A0[i]);
    QP_CUDA(cudaMemcpyAsync(d_ardm, a0.data(), P->N * sizeof(double2), cudaMemcpyHostToDevice, s));
    const int64_t slot0 = P->slot_of(0);
    if (slot0 >= 0) {  // rho(t_0) = rho0 exactly (reading C.3-8)
        std::vector<double2> r0(P->N);
        for (int i = 0; i < P->N; ++i) r0[i] = d2(P->rho0[i]);
        QP_CUDA(cudaMemcpyAsync(w + P->off_rho + slot0 * P->N * sizeof(double2), r0.data(), P->N * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
    }
    // the host vectors above are pageable: cudaMemcpyAsync from pageable memory returns after the
    // source has been staged, so they may go out of scope.
    // persistent slide grid of the launch set p0 = 1 (the common view-A path for M = 2), for qp_plan_query
    {
        const qp_plan::LaunchSet &ls = P->sets[(size_t)std::min(1, P->L - 1) * P->Smax + P->Smax - 1];
        qp::FusedArgs a = ls.args;
        a.use_tma = ls.tma_a != -1 || ls.f2t >= 0;
        P->grid[P->Smax] = launch_grid(P, P->Smax, a);
        P->block = P->persist ? qp::kPersistBlock
                   : (P->M == 3 && P->Smax == 2) ? (ls.f2t >= 0 ? qp::fused2t_block() : qp::fused2s_block())
                   : (P->M == 2 && P->Smax == 4) ? qp::fused4_block()
                   : (P->M == 2 && P->Smax == 3) ? qp::fused3_block(a.lane_map, a.use_tma) : qp::fused_r_block(P->M, P->Smax);
    }
    if (P->persist) {  // launch-set arguments (table pointers into this workspace) + readout slot per step
        std::vector<qp::FusedArgs> sets(P->sets.size());
        for (size_t i = 0; i < P->sets.size(); ++i) {
            const qp_plan::LaunchSet &ls = P->sets[i];
            qp::FusedArgs a = ls.args;
            a.A = (double2 *)d_ardm;
            a.small = (const double2 *)(w + P->off_small);
            a.inner = (const double2 *)(w + ls.off_inner);
            a.Etab = (const double2 *)(w + ls.off_E);
            a.goff = (const long long *)(w + ls.off_goff);
            a.lofs = (const int2 *)(w + ls.off_lofs);
            a.partials = (double2 *)(w + P->off_part);
            a.counter = (unsigned *)(w + P->off_cnt);
            a.rho_accumulate = 0;
            sets[i] = a;
        }
        std::vector<int> slot((size_t)P->n_steps + 1);
        for (int64_t k = 0; k <= P->n_steps; ++k) slot[(size_t)k] = (int)P->slot_of(k);
        QP_CUDA(cudaMemcpyAsync(w + P->off_psets, sets.data(), sets.size() * sizeof(qp::FusedArgs), cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaMemcpyAsync(w + P->off_pslot, slot.data(), slot.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        // one CTA when the ARDM, every table and the launch-set arguments fit its shared memory
        const size_t dyn = P->tables_end + 16 * (size_t)P->ardm_entries + P->sets.size() * sizeof(qp::FusedArgs);
        int dev = 0, optin = 0;
        QP_CUDA(cudaGetDevice(&dev));
        QP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        P->small_dyn = (dyn + (size_t)qp::small_static_smem(P->M, P->lattice, P->sym) <= (size_t)optin) ? dyn : 0;
        if (P->small_dyn) P->grid[P->Smax] = 1;
        else P->block = qp::fused_r_block(P->M, 1);  // does not fit this device: one k_fused_r launch per step
    }
    P->next_k = 1;
    P->sh.seg = 0;
    P->inited = true;
    return QP_OK;
}

qp_status qp_steps(qp_plan *P, int64_t k_begin, int64_t k_end, void *d_ardm, void *d_work, void *stream,
                   int64_t *n_launch) {
    if (n_launch) *n_launch = 0;
    if (!P || !d_ardm || !d_work) return err(QP_ERR_ARG, "arg: NULL plan or device buffer");
    if (!P->inited) return err(QP_ERR_ARG, "arg: qp_init must be called before qp_steps");
    if (P->sh.on) return err(QP_ERR_ARG, "arg: sharded plan: use qp_shard_steps");
    if (k_begin != P->next_k || k_end < k_begin || k_end > P->n_steps + 1)
        return err(QP_ERR_ARG, "arg: steps must be enqueued in order: expected k_begin = %lld, k_end <= %lld",
                   (long long)P->next_k, (long long)P->n_steps + 1);
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)d_work;
    double2 *A = (double2 *)d_ardm;
    const double2 *small = (const double2 *)(w + P->off_small);
    double2 *part = (double2 *)(w + P->off_part);
    unsigned *cnt = (unsigned *)(w + P->off_cnt);
    int64_t launched = 0;
    for (int64_t k = k_begin; k < k_end;) {
        cudaError_t e;
        int64_t adv = 1;
        if (k < P->L) {
            const int64_t slot = P->slot_of(k);
            qp::GrowArgs g{};
            g.A = A; g.small = small; g.partials = part; g.counter = cnt;
            g.rho = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * P->N : nullptr;
            g.n_in = ipow(P->N, (int)k);
            g.k = (int)k;
            g.L = P->L;
            for (int d = 0; d < P->D; ++d) g.delta[d] = P->delta[d];
            const int grid = (int)std::min<int64_t>({(g.n_in + 255) / 256, (int64_t)P->sms * 8, (int64_t)qp::kPartialsMax});
            e = qp::launch_grow(P->M, P->lattice, g, std::max(1, grid), s);
        } else if (P->small_dyn) {  // every remaining slide step of this call: one single-CTA launch
            qp::PersistArgs pa{};
            pa.sets = (const qp::FusedArgs *)(w + P->off_psets);
            pa.set_stride = P->Smax;
            pa.small = small;
            pa.A = A;
            pa.slot = (const int *)(w + P->off_pslot);
            pa.rho_base = (double2 *)(w + P->off_rho);
            const qp::SmallLayout lay{P->N, P->D, P->L};
            for (int var = 0; var < 2; ++var)
                for (int kap = 0; kap < 2 && P->sym; ++kap) {  // FusedArgs::sym per beta variant
                    const double2 c = P->small[lay.beta(var, kap) + 0];
                    const double rho = P->small[lay.beta(var, kap) + 1].x;
                    pa.sym[var][kap][0] = c.x;
                    pa.sym[var][kap][1] = c.y;
                    pa.sym[var][kap][2] = 0.5 * (rho + 1.0 / rho);
                    pa.sym[var][kap][3] = 0.5 * (rho - 1.0 / rho);
                }
            pa.k_begin = k;
            pa.k_end = k_end;
            pa.L = P->L;
            pa.wbase = w;
            pa.tables_bytes = (long long)P->tables_end;
            pa.ardm_entries = P->ardm_entries;
            pa.nsets = (int)P->sets.size();
            e = qp::launch_small(P->M, P->lattice, P->sym, pa, P->small_dyn, s);
            adv = k_end - k;
        } else {
            // fusion groups are aligned on absolute k (k - L multiple of Smax), so the floating-point
            // grouping of a step does not depend on how the caller segments qp_steps calls
            const int64_t grp_end = P->L + ((k - P->L) / P->Smax + 1) * P->Smax;
            const int S = (int)std::min<int64_t>(grp_end, k_end) - (int)k;
            const int p0 = (int)(k % P->L);
            const qp_plan::LaunchSet &ls = P->sets[(size_t)p0 * P->Smax + (S - 1)];
            qp::FusedArgs a = ls.args;
            a.A = A;
            a.small = small;
            if (qp_status st = set_tma(*P, ls, a, A, w)) return st;
            a.inner = (const double2 *)(w + ls.off_inner);
            a.Etab = (const double2 *)(w + ls.off_E);
            a.goff = (const long long *)(w + ls.off_goff);
            a.lofs = (const int2 *)(w + ls.off_lofs);
            a.partials = part;
            a.counter = cnt;
            bool ro = false;
            for (int st = 0; st < S; ++st) {
                const int64_t slot = P->slot_of(k + st);
                a.rho[st] = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * P->N : nullptr;
                ro |= slot >= 0;
                const int var = (k + st == P->L) ? 1 : 0;
                const qp::SmallLayout lay{P->N, P->D, P->L};
                a.var[st] = var;
                if (P->sym) {  // class 1 = (0,1): beta_1 = (c, rho, 1/rho, conj c)
                    for (int kap = 0; kap < 2; ++kap) {
                        const double2 c = P->small[lay.beta(var, kap) + 0];
                        const double rho = P->small[lay.beta(var, kap) + 1].x;
                        a.sym[st][kap][0] = c.x;
                        a.sym[st][kap][1] = c.y;
                        a.sym[st][kap][2] = 0.5 * (rho + 1.0 / rho);
                        a.sym[st][kap][3] = 0.5 * (rho - 1.0 / rho);
                    }
                }
            }
            e = launch_slide(*P, S, a, ro, launch_grid(P, S, a), s);
            adv = S;
        }
        if (e != cudaSuccess) return err(QP_ERR_CUDA, "cuda: launch of step %lld failed: %s", (long long)k, cudaGetErrorString(e));
        ++launched;
        k += adv;
        P->next_k = k;
    }
    if (n_launch) *n_launch = launched;
    return QP_OK;
}

qp_status qp_read_rho(const qp_plan *P, const void *d_work, qp_c64 *rho_out, void *stream) {
    if (!P || !d_work || !rho_out) return err(QP_ERR_ARG, "arg: NULL plan, workspace or output");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t n = P->out_steps.size() * P->N;
    if (n == 0) return QP_OK;
    QP_CUDA(cudaMemcpyAsync(rho_out, (const char *)d_work + P->off_rho, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
    QP_CUDA(cudaStreamSynchronize(s));
    return QP_OK;
}

qp_status qp_run(qp_plan *P, void *d_ardm, void *d_work, void *stream, qp_c64 *rho_out) {
    qp_status st;
    if ((st = qp_init(P, d_ardm, d_work, stream))) return st;
    if ((st = qp_steps(P, 1, P->n_steps + 1, d_ardm, d_work, stream, nullptr))) return st;
    return qp_read_rho(P, d_work, rho_out, stream);
}

}  // extern "C"

// ===================================================================================== sharding
// Multi-GPU execution.  G ranks each hold, for the current segment j, the ARDM
// entries whose z shard slots Z_j = {(k_j - 1 - i) mod L, i < z} (the most recently written slots,
// k_j = L + j (L - z)) take one of the rank's owned combos c in [c_lo, c_lo + n_own): one block of
// N^(L-z) entries per combo, the other slots in ascending order.  The L - z steps of a segment never
// contract a shard slot, so they run shard-locally (k_fused with the combo's fixed factors); between
// segments the data is re-sharded on Z_{j+1} (pack -> NCCL all-to-all by the caller -> unpack).
namespace {

void shard_combo_digits(const qp_plan &P, int64_t c, int *dig) {
    for (int i = 0; i < P.sh.z; ++i) { dig[i] = (int)(c % P.N); c /= P.N; }
}

// positions of the non-shard slots (ascending) in a segment's local layout
std::vector<int> local_pos(const qp_plan &P, const std::vector<int> &Z) {
    std::vector<int> pos(P.L, -1);
    for (int q = 0, n = 0; q < P.L; ++q)
        if (std::find(Z.begin(), Z.end(), q) == Z.end()) pos[q] = n++;
    return pos;
}

}  // namespace

extern "C" {

qp_status qp_shard_configure(qp_plan *P, int32_t n_ranks, int32_t rank) {
    if (!P) return err(QP_ERR_ARG, "arg: NULL plan");
    if (n_ranks < 2 || rank < 0 || rank >= n_ranks) return err(QP_ERR_ARG, "arg: need n_ranks >= 2 and 0 <= rank < n_ranks");
    if (P->inited || P->sh.on) return err(QP_ERR_ARG, "arg: qp_shard_configure must be called once, before qp_init");
    const int L = P->L, N = P->N;
    // smallest z with at most 10% load imbalance of the N^z combos over the ranks
    // (segments need 2z <= L - 1 so that consecutive shard-slot sets are disjoint); else the smallest
    // z with N^z >= n_ranks
    int z = 0, zmin = 0;
    for (int zz = 1; 2 * zz <= L - 1; ++zz) {
        const double nz = std::pow((double)N, zz);
        if (nz < n_ranks) continue;
        if (!zmin) zmin = zz;
        if (std::ceil(nz / n_ranks) / (nz / n_ranks) <= 1.1 + 1e-12) { z = zz; break; }
    }
    if (!z) z = zmin;
    if (!z) return err(QP_ERR_CONFIG, "config: cannot shard L = %d over %d ranks (need N^z >= ranks, 2z <= L-1)", L, n_ranks);
    auto &sh = P->sh;
    sh = qp_plan::Shard{};
    sh.on = true;
    sh.G = n_ranks;
    sh.rank = rank;
    sh.z = z;
    sh.seg_len = L - z;
    sh.NZ = ipow(N, z);
    sh.blk = ipow(N, L - z);
    sh.c_lo.resize(n_ranks);
    sh.n_own.resize(n_ranks);
    for (int r = 0; r < n_ranks; ++r) {
        const int64_t base = sh.NZ / n_ranks, extra = sh.NZ % n_ranks;
        sh.n_own[r] = base + (r < extra ? 1 : 0);
        sh.c_lo[r] = r * base + std::min<int64_t>(r, extra);
    }
    // launch sets for every segment start slot of the (periodic) schedule
    std::vector<int> starts;
    for (int64_t j = 0;; ++j) {
        const int zs = (int)(P->seg_begin(j) % L);
        if (std::find(starts.begin(), starts.end(), zs) != starts.end()) break;
        starts.push_back(zs);
    }
    // fusion depth of the segments: the plan's, or 3 when a four-step shard set has no k_fused4 layout
    // (fewer than two outer digits in the local layout)
    sh.Smax = P->Smax;
    for (bool retry = true; retry;) {
        retry = false;
        sh.sets.clear();
        sh.index.clear();
        for (int zs : starts) {
            std::vector<int> Z;
            for (int i = 0; i < z; ++i) Z.push_back(((zs - 1 - i) % L + L) % L);
            std::sort(Z.begin(), Z.end());
            for (int m = 0; m < sh.seg_len && !retry; ++m)
                for (int S = 1; S <= sh.Smax && m + S <= sh.seg_len; ++S) {
                    const int p0 = (zs + m) % L;
                    sh.index[std::make_tuple(zs, p0, S)] = sh.sets.size();
                    sh.sets.emplace_back();
                    build_launch_set(*P, p0, S, Z, sh.sets.back());
                    if (S == 4 && !sh.sets.back().f4) { sh.Smax = 3; retry = true; break; }
                }
        }
    }
    compute_layout(*P);
    // capacity (a1) against an explicit budget: two buffers of this rank's shard (local + exchange) +
    // workspace (qp_plan_check compares with the device's free memory)
    const double need = 2.0 * 16.0 * double(sh.n_own[rank] * sh.blk) + double(P->work_bytes);
    if (P->max_bytes > 0 && check_capacity(P->max_bytes, need, "two shard buffers + workspace")) {
        const qp_status st = QP_ERR_CAPACITY;
        sh = qp_plan::Shard{};
        compute_layout(*P);
        return st;
    }
    return QP_OK;
}

qp_status qp_shard_query(const qp_plan *P, qp_shard_sizes *o) {
    if (!P || !o) return err(QP_ERR_ARG, "arg: NULL plan or out");
    if (!P->sh.on) return err(QP_ERR_ARG, "arg: plan is not sharded (qp_shard_configure)");
    const auto &sh = P->sh;
    o->n_ranks = sh.G;
    o->rank = sh.rank;
    o->shard_slots = sh.z;
    o->segment_steps = sh.seg_len;
    o->local_entries = sh.n_own[sh.rank] * sh.blk;
    int64_t mx = 0;
    for (int r = 0; r < sh.G; ++r) mx = std::max(mx, sh.n_own[r]);
    o->max_local_entries = mx * sh.blk;
    o->exchange_entries = sh.n_own[sh.rank] * sh.blk;  // everything moves (incl. the part kept locally)
    o->xbuf_entries = std::max(o->local_entries, o->exchange_entries);
    o->work_bytes = (int64_t)P->work_bytes;
    return QP_OK;
}

qp_status qp_shard_counts(const qp_plan *P, int64_t *send_counts, int64_t *recv_counts) {
    if (!P || !send_counts || !recv_counts) return err(QP_ERR_ARG, "arg: NULL plan or output");
    if (!P->sh.on) return err(QP_ERR_ARG, "arg: plan is not sharded");
    const auto &sh = P->sh;
    const int64_t rest = ipow(P->N, P->L - 2 * sh.z);
    for (int r = 0; r < sh.G; ++r) {
        send_counts[r] = sh.n_own[sh.rank] * sh.n_own[r] * rest;
        recv_counts[r] = sh.n_own[r] * sh.n_own[sh.rank] * rest;
    }
    return QP_OK;
}

// Re-shard from segment j to j + 1 through the caller's two buffers (local L, exchange X):
//   qp_shard_pack:   L -> X in send order [dst rank][my Z_j block][dst's Z_{j+1} combo][other slots]
//   caller:          all-to-all X -> L (L is free once packed)
//   qp_shard_unpack: L (received, [src rank][src's Z_j combo][my Z_{j+1} block][other]) -> X in the
//                    segment j + 1 layout; the caller then swaps the two buffers (X is the new local).
static qp_status shard_permute(qp_plan *P, bool pack, const void *src, void *dst, cudaStream_t st) {
    const auto &sh = P->sh;
    const std::vector<int> Z0 = P->zset(sh.seg), Z1 = P->zset(sh.seg + 1);
    const std::vector<int> pos = local_pos(*P, pack ? Z0 : Z1);
    const int64_t R = ipow(P->N, P->L - 2 * sh.z), me = sh.rank;
    int64_t off = 0;
    for (int r = 0; r < sh.G; ++r) {
        qp::PermuteArgs a{};
        a.scatter = pack ? 0 : 1;
        a.nd = 0;
        for (int q = 0; q < P->L; ++q)  // the other slots, ascending
            if (std::find(Z0.begin(), Z0.end(), q) == Z0.end() && std::find(Z1.begin(), Z1.end(), q) == Z1.end())
                a.dstr[a.nd++] = ipow(P->N, pos[q]);
        a.ncombo = 2;
        if (pack) {  // gather from local: dst's combos of Z_{j+1} (digits), then my blocks (linear)
            a.crad[0] = (int)sh.n_own[r], a.clo[0] = (int)sh.c_lo[r], a.cnd[0] = sh.z;
            for (int i = 0; i < sh.z; ++i) a.cstr[0][i] = ipow(P->N, pos[Z1[i]]);
            a.crad[1] = (int)sh.n_own[me], a.clo[1] = 0, a.cnd[1] = 0, a.cstr[1][0] = sh.blk;
            a.count = sh.n_own[me] * sh.n_own[r] * R;
            a.src = (const double2 *)src;
            a.dst = (double2 *)dst + off;
        } else {  // scatter into the new local: my new blocks (linear), then src's combos of Z_j (digits)
            a.crad[0] = (int)sh.n_own[me], a.clo[0] = 0, a.cnd[0] = 0, a.cstr[0][0] = sh.blk;
            a.crad[1] = (int)sh.n_own[r], a.clo[1] = (int)sh.c_lo[r], a.cnd[1] = sh.z;
            for (int i = 0; i < sh.z; ++i) a.cstr[1][i] = ipow(P->N, pos[Z0[i]]);
            a.count = sh.n_own[r] * sh.n_own[me] * R;
            a.src = (const double2 *)src + off;
            a.dst = (double2 *)dst;
        }
        QP_CUDA(qp::launch_permute(P->M, a, P->sms, st));
        off += a.count;
    }
    return QP_OK;
}

qp_status qp_shard_pack(qp_plan *P, const void *d_local, void *d_xbuf, void *stream) {
    if (!P || !d_local || !d_xbuf) return err(QP_ERR_ARG, "arg: NULL plan or buffer");
    if (!P->sh.on || !P->inited) return err(QP_ERR_ARG, "arg: plan not sharded / not initialised");
    if (P->next_k != P->seg_begin(P->sh.seg + 1))
        return err(QP_ERR_ARG, "arg: pack at the end of a segment (next step %lld, segment ends at %lld)",
                   (long long)P->next_k, (long long)P->seg_begin(P->sh.seg + 1));
    return shard_permute(P, true, d_local, d_xbuf, (cudaStream_t)stream);
}

qp_status qp_shard_unpack(qp_plan *P, const void *d_recv, void *d_xbuf, void *stream) {
    if (!P || !d_recv || !d_xbuf) return err(QP_ERR_ARG, "arg: NULL plan or buffer");
    if (!P->sh.on || !P->inited) return err(QP_ERR_ARG, "arg: plan not sharded / not initialised");
    if (P->next_k != P->seg_begin(P->sh.seg + 1)) return err(QP_ERR_ARG, "arg: unpack follows a pack");
    if (qp_status st = shard_permute(P, false, d_recv, d_xbuf, (cudaStream_t)stream)) return st;
    P->sh.seg += 1;
    return QP_OK;
}

qp_status qp_shard_steps(qp_plan *P, int64_t k_begin, int64_t k_end, void *d_local, void *d_xbuf, void *d_work,
                         void *stream, int64_t *n_launch) {
    if (n_launch) *n_launch = 0;
    if (!P || !d_local || !d_xbuf || !d_work) return err(QP_ERR_ARG, "arg: NULL plan or buffer");
    auto &sh = P->sh;
    if (!sh.on || !P->inited) return err(QP_ERR_ARG, "arg: plan not sharded (qp_shard_configure) / not initialised (qp_init)");
    const int L = P->L, N = P->N, kb = L - sh.z;
    if (k_begin != P->next_k || k_end < k_begin || k_end > P->n_steps + 1)
        return err(QP_ERR_ARG, "arg: shard steps must be enqueued in order: expected k_begin = %lld", (long long)P->next_k);
    if (k_begin >= L) {
        const int64_t s0 = P->seg_begin(sh.seg), s1 = s0 + sh.seg_len;
        if (k_begin < s0 || k_end > s1)
            return err(QP_ERR_ARG, "arg: slide steps stay within segment [%lld, %lld) (re-shard between segments)",
                       (long long)s0, (long long)s1);
    } else if (k_end > L) {
        return err(QP_ERR_ARG, "arg: growth steps (k < %d) and slide steps in separate calls", L);
    }
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)d_work;
    const double2 *small = (const double2 *)(w + P->off_small);
    double2 *part = (double2 *)(w + P->off_part);
    unsigned *cnt = (unsigned *)(w + P->off_cnt);
    int64_t launched = 0;
    for (int64_t k = k_begin; k < k_end;) {
        if (k < kb) {  // replicated growth on the exchange buffer: N^(k+1) <= N^(L-z) entries
            const int64_t slot = P->slot_of(k);
            qp::GrowArgs g{};
            g.A = (double2 *)d_xbuf; g.small = small; g.partials = part; g.counter = cnt;
            g.rho = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * N : nullptr;
            g.n_in = ipow(N, (int)k);
            g.k = (int)k;
            g.L = L;
            for (int d = 0; d < P->D; ++d) g.delta[d] = P->delta[d];
            const int grid = (int)std::min<int64_t>({(g.n_in + 255) / 256, (int64_t)P->sms * 8, (int64_t)qp::kPartialsMax});
            QP_CUDA(qp::launch_grow(P->M, P->lattice, g, std::max(1, grid), s));
            ++launched;
            ++k;
        } else if (k < L) {  // the z growth steps that add the shard digits: this rank's combos only
            const int64_t slot = P->slot_of(k);
            qp::GrowShardArgs g{};
            g.Abase = (const double2 *)d_xbuf;
            g.local = (double2 *)d_local;
            g.small = small; g.partials = part; g.counter = cnt;
            g.rho = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * N : nullptr;
            g.nb = sh.blk;
            g.L = L, g.z = sh.z, g.step = (int)(k - kb), g.n_own = (int)sh.n_own[sh.rank], g.c_lo = (int)sh.c_lo[sh.rank];
            for (int d = 0; d < P->D; ++d) g.delta[d] = P->delta[d];
            const int grid = (int)std::min<int64_t>({(g.nb + 255) / 256, (int64_t)P->sms * 8, (int64_t)qp::kPartialsMax});
            QP_CUDA(qp::launch_grow_shard(P->M, P->lattice, g, std::max(1, grid), s));
            ++launched;
            ++k;
        } else {  // slide steps of the current segment, one launch per owned block
            const int64_t s0 = P->seg_begin(sh.seg);
            const int64_t grp_end = s0 + ((k - s0) / sh.Smax + 1) * sh.Smax;
            const int S = (int)(std::min<int64_t>({grp_end, k_end, s0 + sh.seg_len}) - k);
            const int p0 = (int)(k % L);
            const std::vector<int> Z = P->zset(sh.seg);
            const int zs = (int)(s0 % L);
            const auto it = sh.index.find(std::make_tuple(zs, p0, S));
            if (it == sh.index.end()) return err(QP_ERR_ARG, "internal: no shard launch set for (%d, %d, %d)", zs, p0, S);
            const qp_plan::LaunchSet &ls = sh.sets[it->second];
            for (int64_t b = 0; b < sh.n_own[sh.rank]; ++b) {
                qp::FusedArgs a = ls.args;
                a.A = (double2 *)d_local + b * sh.blk;
                a.small = small;
                a.inner = (const double2 *)(w + ls.off_inner);
                a.Etab = (const double2 *)(w + ls.off_E);
                a.goff = (const long long *)(w + ls.off_goff);
                a.lofs = (const int2 *)(w + ls.off_lofs);
                a.partials = part;
                a.counter = cnt;
                a.rho_accumulate = b > 0 ? 1 : 0;
                if (qp_status st = set_tma(*P, ls, a, a.A, w)) return st;
                int dig[8];
                shard_combo_digits(*P, sh.c_lo[sh.rank] + b, dig);
                bool ro = false;
                const qp::SmallLayout lay{N, P->D, L};
                for (int st = 0; st < S; ++st) {
                    const int64_t slot = P->slot_of(k + st);
                    a.rho[st] = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * N : nullptr;
                    ro |= slot >= 0;
                    const int var = (k + st == L) ? 1 : 0;
                    a.var[st] = var;
                    if (P->sym)
                        for (int kap = 0; kap < 2; ++kap) {
                            const double2 c = P->small[lay.beta(var, kap) + 0];
                            const double rho = P->small[lay.beta(var, kap) + 1].x;
                            a.sym[st][kap][0] = c.x;
                            a.sym[st][kap][1] = c.y;
                            a.sym[st][kap][2] = 0.5 * (rho + 1.0 / rho);
                            a.sym[st][kap][3] = 0.5 * (rho - 1.0 / rho);
                        }
                    // fixed shard-slot digits: their Eq. 9 factor for this sub-step (propagate / terminal)
                    for (int kap = 0; kap < 2; ++kap) {
                        cd Ps = 0.0;
                        for (int i = 0; i < sh.z; ++i) {
                            const int lag = ((p0 + st - Z[i]) % L + L) % L;
                            Ps += psi(*P, dig[i], kap == 0 ? P->eta[lag] : P->E[lag]);
                        }
                        for (int d = 0; d < P->D; ++d) a.fixfac[st][kap][d] = d2(std::exp(P->delta[d] * Ps));
                    }
                }
                const int qlast = (p0 - 1 + L) % L;
                a.fixed_last = -1;
                for (int i = 0; i < sh.z; ++i)
                    if (Z[i] == qlast) a.fixed_last = dig[i];
                const cudaError_t e = launch_slide(*P, S, a, ro, launch_grid(P, S, a), s);
                if (e != cudaSuccess) return err(QP_ERR_CUDA, "cuda: shard launch of step %lld failed: %s", (long long)k, cudaGetErrorString(e));
                ++launched;
            }
            k += S;
        }
        P->next_k = k;
    }
    if (n_launch) *n_launch = launched;
    return QP_OK;
}

int64_t qp_rho_offset(const qp_plan *P) { return P ? (int64_t)P->off_rho : -1; }

// ===================================================================================== path filtering
// SURVEY 8(f3), reading C.3-15 (ofpf.cu): the ARDM as a compacted (key, value) list of the entries with
// |A|^2 >= theta^2, ping-ponged between two halves of the caller's buffer.
namespace {
struct FilterLayout {
    size_t key[2], val[2], flags, blkcnt, blkbase, tab, ctr, kept, total;
};
FilterLayout filter_layout(const qp_plan *P, int64_t cap, int nblk) {
    FilterLayout f{};
    size_t off = 0;
    for (int h = 0; h < 2; ++h) { f.key[h] = off; off = align256(off + (size_t)cap * 8); }
    for (int h = 0; h < 2; ++h) { f.val[h] = off; off = align256(off + (size_t)cap * 16); }
    f.flags = off;   off = align256(off + (size_t)cap * 2);
    f.blkcnt = off;  off = align256(off + (size_t)nblk * P->N * 4);
    f.blkbase = off; off = align256(off + (size_t)nblk * P->N * 8);
    f.tab = off;     off = align256(off + (size_t)2 * (qp::kMaxL + 1) * P->N * 16);
    f.ctr = off;     off = align256(off + 4 * 8);  // n[0], n[1], overflow
    f.kept = off;    off = align256(off + (size_t)(P->n_steps + 1) * 8);
    f.total = off;
    return f;
}
constexpr int kFilterBlocksPerSM = 4;
}  // namespace

qp_status qp_filter_query(const qp_plan *P, int64_t capacity, int64_t *bytes) {
    if (!P || !bytes || capacity < 1) return err(QP_ERR_ARG, "arg: NULL plan / output or capacity < 1");
    *bytes = (int64_t)filter_layout(P, capacity, 148 * kFilterBlocksPerSM * 2).total;  // room for up to 296 SMs
    return QP_OK;
}

qp_status qp_filter_run(qp_plan *P, double theta, void *d_buf, int64_t buf_bytes, void *d_work, void *stream,
                        qp_c64 *rho_out, int64_t *kept_out) {
    if (!P || !d_buf || !d_work || !rho_out) return err(QP_ERR_ARG, "arg: NULL plan, buffer or output");
    if (!(theta >= 0.0) || !std::isfinite(theta)) return err(QP_ERR_ARG, "arg: theta must be finite and >= 0");
    if (P->sh.on) return err(QP_ERR_ARG, "arg: path filtering runs unsharded");
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    QP_CUDA(cudaGetDevice(&dev));
    QP_CUDA(cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, dev));
    const int nblk = P->sms * kFilterBlocksPerSM;
    // largest capacity that fits the buffer
    // 50 B per list entry (two keys, two values, one flag word) + fixed tables and 256-B alignment slack
    const int64_t fixed = (int64_t)filter_layout(P, 1, nblk).total + 8 * 256;
    int64_t cap = std::max<int64_t>(1, (buf_bytes - fixed) / 50);
    while (cap > 1 && (int64_t)filter_layout(P, cap, nblk).total > buf_bytes) --cap;
    const FilterLayout f = filter_layout(P, cap, nblk);
    if ((int64_t)f.total > buf_bytes) return err(QP_ERR_CAPACITY, "capacity: filter buffer of %lld B too small", (long long)buf_bytes);
    char *b = (char *)d_buf, *w = (char *)d_work;
    const int N = P->N, L = P->L;
    // tables: small (K', beta, growth psi rows) into the workspace, slide partner psi rows into the buffer
    QP_CUDA(cudaMemcpyAsync(w + P->off_small, P->small.data(), P->small.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    std::vector<double2> tab((size_t)2 * (qp::kMaxL + 1) * N, make_double2(0.0, 0.0));
    for (int lag = 1; lag <= L; ++lag)
        for (int sg = 0; sg < N; ++sg) {
            tab[(size_t)(0 * (qp::kMaxL + 1) + lag) * N + sg] = d2(psi(*P, sg, P->eta[lag]));
            tab[(size_t)(1 * (qp::kMaxL + 1) + lag) * N + sg] = d2(psi(*P, sg, P->E[lag]));
        }
    QP_CUDA(cudaMemcpyAsync(b + f.tab, tab.data(), tab.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    QP_CUDA(cudaMemsetAsync(w + P->off_cnt, 0, 256, s));
    QP_CUDA(cudaMemsetAsync(b + f.ctr, 0, 4 * 8, s));
    QP_CUDA(cudaMemsetAsync(b + f.kept, 0, (size_t)(P->n_steps + 1) * 8, s));
    // A_0: its nonzero entries (exact zeros contribute nothing), keys sigma_0
    std::vector<long long> k0;
    std::vector<double2> v0;
    for (int sg = 0; sg < N; ++sg)
        if (P->A0[sg] != cd(0.0, 0.0)) { k0.push_back(sg); v0.push_back(d2(P->A0[sg])); }
    const long long n0 = (long long)k0.size();
    if (n0 > cap) return err(QP_ERR_CAPACITY, "capacity: filter buffer too small");
    if (n0) {
        QP_CUDA(cudaMemcpyAsync(b + f.key[0], k0.data(), n0 * 8, cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaMemcpyAsync(b + f.val[0], v0.data(), n0 * 16, cudaMemcpyHostToDevice, s));
    }
    QP_CUDA(cudaMemcpyAsync(b + f.ctr, &n0, 8, cudaMemcpyHostToDevice, s));
    QP_CUDA(cudaMemcpyAsync(b + f.kept, &n0, 8, cudaMemcpyHostToDevice, s));
    QP_CUDA(cudaStreamSynchronize(s));  // the host staging vectors above go out of scope
    const int64_t slot0 = P->slot_of(0);
    if (slot0 >= 0) {
        std::vector<double2> r0(N);
        for (int i = 0; i < N; ++i) r0[i] = d2(P->rho0[i]);
        QP_CUDA(cudaMemcpyAsync(w + P->off_rho + slot0 * N * sizeof(double2), r0.data(), N * sizeof(double2), cudaMemcpyHostToDevice, s));
        QP_CUDA(cudaStreamSynchronize(s));
    }
    long long *ctr = (long long *)(b + f.ctr);
    for (int64_t k = 1; k <= P->n_steps; ++k) {
        const int h = (int)((k - 1) & 1);
        qp::OfpfArgs a{};
        a.key_in = (const long long *)(b + f.key[h]);
        a.val_in = (const double2 *)(b + f.val[h]);
        a.key_out = (long long *)(b + f.key[h ^ 1]);
        a.val_out = (double2 *)(b + f.val[h ^ 1]);
        a.n_in = ctr + h;
        a.n_out = ctr + (h ^ 1);
        a.flags = (unsigned short *)(b + f.flags);
        a.blkcnt = (int *)(b + f.blkcnt);
        a.blkbase = (long long *)(b + f.blkbase);
        a.kept = (long long *)(b + f.kept) + k;
        a.overflow = (int *)(ctr + 2);
        a.cap = cap;
        a.small = (const double2 *)(w + P->off_small);
        a.tab = (const double2 *)(b + f.tab);
        a.partials = (double2 *)(w + P->off_part);
        a.counter = (unsigned *)(w + P->off_cnt);
        const int64_t slot = P->slot_of(k);
        a.rho = slot >= 0 ? (double2 *)(w + P->off_rho) + slot * N : nullptr;
        a.th2 = theta * theta;
        a.top = ipow(N, L - 1);
        a.grow_w = k < L ? ipow(N, (int)k) : 0;
        a.k = (int)std::min<int64_t>(k, L);
        a.L = L;
        a.slide = k >= L ? 1 : 0;
        a.var = (k == L) ? 1 : 0;
        for (int d = 0; d < P->D; ++d) a.delta[d] = P->delta[d];
        const cudaError_t e = qp::launch_ofpf_step(P->M, P->lattice, a, nblk, s);
        if (e != cudaSuccess) return err(QP_ERR_CUDA, "cuda: filtered step %lld: %s", (long long)k, cudaGetErrorString(e));
    }
    long long hctr[3];
    QP_CUDA(cudaMemcpyAsync(hctr, ctr, 3 * 8, cudaMemcpyDeviceToHost, s));
    std::vector<long long> kept((size_t)P->n_steps + 1);
    QP_CUDA(cudaMemcpyAsync(kept.data(), b + f.kept, kept.size() * 8, cudaMemcpyDeviceToHost, s));
    QP_CUDA(cudaStreamSynchronize(s));
    if (((int *)&hctr[2])[0]) {
        int64_t kk = 0;
        for (size_t i = 0; i < kept.size(); ++i) if (kept[i] > cap) { kk = (int64_t)i; break; }
        return err(QP_ERR_CAPACITY, "capacity: the filtered ARDM exceeded %lld entries at step %lld", (long long)cap, (long long)kk);
    }
    if (kept_out) for (size_t i = 0; i < kept.size(); ++i) kept_out[i] = kept[i];
    return qp_read_rho(P, d_work, rho_out, s);
}

qp_status qp_shard_combine(const qp_plan *P, const void *d_parts, void *d_work, qp_c64 *rho_out, void *stream) {
    if (!P || !d_parts || !d_work || !rho_out) return err(QP_ERR_ARG, "arg: NULL plan, buffer or output");
    if (!P->sh.on) return err(QP_ERR_ARG, "arg: plan is not sharded");
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)d_work;
    const int64_t n_out = (int64_t)P->out_steps.size();
    if (n_out == 0) return QP_OK;
    // out_steps on the device (after the rho block), then the rank-ordered sum into the rho block
    long long *d_steps = (long long *)(w + P->off_cnt + 256);
    QP_CUDA(cudaMemcpyAsync(d_steps, P->out_steps.data(), n_out * sizeof(long long), cudaMemcpyHostToDevice, s));
    QP_CUDA(qp::launch_shard_combine((const double2 *)d_parts, (double2 *)(w + P->off_rho), d_steps, n_out, P->N, P->sh.G,
                                     P->L - P->sh.z, s));
    return qp_read_rho(P, d_work, rho_out, s);
}

}  // extern "C"

// ===================================================================================== batched sweeps
// B problems sharing the bath / grid, each with its own drive amplitude and initial state
// (include/quapi.h).  The shared parts (validation, eta classes, Delta-s classes) come from an
// internal qp_plan of the base problem; the device image holds the per-lag psi rows, the two
// Hamiltonian parts, the drive amplitudes, the initial states and the output map.
struct qp_batch_plan {
    qp_plan *P = nullptr;
    int B = 0;
    std::vector<double2> tab, rho0;
    std::vector<double> f;
    std::vector<int> out_idx;
    std::vector<qp_bath> baths;        // per-problem baths (empty: base's bath for all)
    size_t off_tab = 0, off_f = 0, off_rho0 = 0, off_idx = 0, off_rho = 0, off_eta = 0, off_ptab = 0, work_bytes = 0;
    double setup_seconds = 0.0;
};

extern "C" {

qp_status qp_batch_create(const qp_batch *bt, qp_batch_plan **out) {
    if (!bt || !out) return err(QP_ERR_ARG, "arg: NULL batch or out");
    *out = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (bt->B < 1) return err(QP_ERR_CONFIG, "config: batch size B must be >= 1 (got %d)", bt->B);
    qp_problem base = bt->base;
    const int64_t mb = base.max_bytes;
    base.max_bytes = 0;  // capacity is checked for the whole batch below
    qp_plan *P = nullptr;
    qp_status st = qp_plan_create(&base, &P);
    if (st) return st;
    const int M = P->M, N = P->N, L = P->L;
    auto fail = [&](qp_status code, const char *msg) {
        qp_plan_destroy(P);
        return err(code, "%s", msg);
    };
    if (bt->H1) {
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) {
                const cd h = {bt->H1[i * M + j].re, bt->H1[i * M + j].im}, hT = {bt->H1[j * M + i].re, bt->H1[j * M + i].im};
                if (!(std::abs(h - std::conj(hT)) <= 1e-12) || !std::isfinite(h.real()) || !std::isfinite(h.imag()))
                    return fail(QP_ERR_CONFIG, "config: H1 not Hermitian");
            }
    }
    if (bt->baths)
        for (int b = 0; b < bt->B; ++b)
            if (validate_bath(bt->baths[b], b)) {
                const std::string m = g_err;
                return fail(QP_ERR_CONFIG, m.c_str());
            }
    if (bt->f)
        for (int64_t i = 0; i < (int64_t)bt->B * P->n_steps; ++i)
            if (!std::isfinite(bt->f[i])) return fail(QP_ERR_CONFIG, "config: drive amplitude f not finite");
    if (bt->rho0)
        for (int b = 0; b < bt->B; ++b) {
            const qp_c64 *r = bt->rho0 + (size_t)b * N;
            cd tr = 0.0;
            for (int i = 0; i < M; ++i) {
                for (int j = 0; j < M; ++j) {
                    const cd x = {r[i * M + j].re, r[i * M + j].im}, xT = {r[j * M + i].re, r[j * M + i].im};
                    if (!(std::abs(x - std::conj(xT)) <= 1e-12)) return fail(QP_ERR_CONFIG, "config: a batch rho0 is not Hermitian");
                }
                tr += cd(r[i * M + i].re, r[i * M + i].im);
            }
            if (!(std::abs(tr - 1.0) <= 1e-12)) return fail(QP_ERR_CONFIG, "config: a batch rho0 does not have trace 1");
        }
    const double bytes = 16.0 * bt->B * std::pow((double)N, L);
    if (mb > 0 && bytes > (double)mb) {
        qp_plan_destroy(P);
        return err(QP_ERR_CAPACITY, "capacity: need %.0f B for the batch ARDM, budget %lld B", bytes, (long long)mb);
    }
    auto *bp = new qp_batch_plan;
    bp->P = P;
    bp->B = bt->B;
    // psi rows (lag j = 1..L), self classes, H0, H1
    bp->tab.assign((size_t)(3 * (L + 1) + 2) * N + 2 * M * M, make_double2(0.0, 0.0));
    for (int j = 1; j <= L; ++j)
        for (int sg = 0; sg < N; ++sg) {
            bp->tab[(size_t)j * N + sg] = d2(psi(*P, sg, P->eta[j]));
            bp->tab[(size_t)(L + 1 + j) * N + sg] = d2(psi(*P, sg, P->E[j]));
            bp->tab[(size_t)(2 * (L + 1) + j) * N + sg] = d2(psi(*P, sg, P->TI[j]));
        }
    for (int sg = 0; sg < N; ++sg) {
        bp->tab[(size_t)3 * (L + 1) * N + sg] = d2(psi(*P, sg, P->self_int));
        bp->tab[(size_t)(3 * (L + 1) + 1) * N + sg] = d2(psi(*P, sg, P->self_end));
    }
    const size_t oh = (size_t)(3 * (L + 1) + 2) * N;
    for (int i = 0; i < M * M; ++i) {
        bp->tab[oh + i] = d2(P->H[i]);
        bp->tab[oh + M * M + i] = bt->H1 ? make_double2(bt->H1[i].re, bt->H1[i].im) : make_double2(0.0, 0.0);
    }
    if (bt->f && bt->H1) bp->f.assign(bt->f, bt->f + (size_t)bt->B * P->n_steps);
    bp->rho0.resize((size_t)bt->B * N);
    for (int b = 0; b < bt->B; ++b)
        for (int n = 0; n < N; ++n)
            bp->rho0[(size_t)b * N + n] = bt->rho0 ? make_double2(bt->rho0[(size_t)b * N + n].re, bt->rho0[(size_t)b * N + n].im)
                                                   : d2(P->rho0[n]);
    bp->out_idx.assign((size_t)P->n_steps + 1, -1);
    for (size_t o = 0; o < P->out_steps.size(); ++o) bp->out_idx[(size_t)P->out_steps[o]] = (int)o;
    size_t off = 0;
    bp->off_tab = off;  off = align256(off + bp->tab.size() * sizeof(double2));
    bp->off_f = off;    off = align256(off + bp->f.size() * sizeof(double));
    bp->off_rho0 = off; off = align256(off + bp->rho0.size() * sizeof(double2));
    bp->off_idx = off;  off = align256(off + bp->out_idx.size() * sizeof(int));
    bp->off_rho = off;  off = align256(off + (size_t)bt->B * P->out_steps.size() * N * sizeof(double2));
    if (bt->baths) {  // device eta [B][3L+2] and per-problem psi tables [B][(3(L+1)+2) N]
        bp->baths.assign(bt->baths, bt->baths + bt->B);
        bp->off_eta = off;  off = align256(off + (size_t)bt->B * (3 * L + 2) * sizeof(double2));
        bp->off_ptab = off; off = align256(off + (size_t)bt->B * (3 * (L + 1) + 2) * N * sizeof(double2));
    }
    bp->work_bytes = off;
    bp->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = bp;
    return QP_OK;
}

qp_status qp_batch_query(const qp_batch_plan *bp, qp_batch_sizes *o) {
    if (!bp || !o) return err(QP_ERR_ARG, "arg: NULL batch plan or out");
    const qp_plan *P = bp->P;
    o->B = bp->B;
    o->M = P->M, o->N = P->N, o->L = P->L;
    o->ardm_entries = (int64_t)bp->B * ipow(P->N, P->L);
    o->ardm_bytes = 16 * o->ardm_entries;
    o->work_bytes = (int64_t)bp->work_bytes;
    o->n_out = (int64_t)P->out_steps.size();
    o->n_steps = P->n_steps;
    o->block = qp::kBatchBlock;
    o->setup_seconds = bp->setup_seconds;
    return QP_OK;
}

qp_status qp_batch_run(qp_batch_plan *bp, void *d_ardm, void *d_work, void *stream, qp_c64 *rho_out) {
    if (!bp || !d_ardm || !d_work) return err(QP_ERR_ARG, "arg: NULL batch plan or device buffer");
    const qp_plan *P = bp->P;
    const int N = P->N;
    cudaStream_t s = (cudaStream_t)stream;
    char *w = (char *)d_work;
    QP_CUDA(cudaMemcpyAsync(w + bp->off_tab, bp->tab.data(), bp->tab.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    if (!bp->f.empty())
        QP_CUDA(cudaMemcpyAsync(w + bp->off_f, bp->f.data(), bp->f.size() * sizeof(double), cudaMemcpyHostToDevice, s));
    QP_CUDA(cudaMemcpyAsync(w + bp->off_rho0, bp->rho0.data(), bp->rho0.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    QP_CUDA(cudaMemcpyAsync(w + bp->off_idx, bp->out_idx.data(), bp->out_idx.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    qp::BatchArgs a{};
    a.A = (double2 *)d_ardm;
    a.tab = (const double2 *)(w + bp->off_tab);
    a.f = bp->f.empty() ? nullptr : (const double *)(w + bp->off_f);
    a.rho0 = (const double2 *)(w + bp->off_rho0);
    a.out_idx = (const int *)(w + bp->off_idx);
    a.rho = (double2 *)(w + bp->off_rho);
    a.NL = ipow(N, P->L);
    a.n_steps = P->n_steps;
    a.dt = P->dt;
    a.L = P->L;
    a.n_out = (int)P->out_steps.size();
    a.D = P->D;
    for (int n = 0; n < N; ++n) {
        a.cls[n] = qp::class_of(P->M, P->lattice, n / P->M, n % P->M);
        a.dsig[n] = dsig(*P, n);
    }
    for (int d = 0; d < P->D; ++d) a.delta[d] = P->delta[d];
    if (!bp->baths.empty()) {  // per-problem eta on the device, then psi rows (Eq. 9 exponents) per problem
        double2 *eta = (double2 *)(w + bp->off_eta);
        if (qp_status st = enqueue_eta(bp->baths.data(), bp->B, P->dt, P->L, eta, nullptr, s)) return st;
        double sv[qp::kMaxM] = {0};
        for (int i = 0; i < P->M; ++i) sv[i] = P->s[i];
        a.ptab = (double2 *)(w + bp->off_ptab);
        const cudaError_t ep = qp::launch_psi_tables(P->M, sv, eta, (double2 *)a.ptab, bp->B, P->L, s);
        if (ep != cudaSuccess) return err(QP_ERR_CUDA, "cuda: psi table launch failed: %s", cudaGetErrorString(ep));
    }
    const cudaError_t e = qp::launch_batch(P->M, a, bp->B, s);
    if (e != cudaSuccess) return err(QP_ERR_CUDA, "cuda: batch launch failed: %s", cudaGetErrorString(e));
    if (rho_out) {
        const size_t n = (size_t)bp->B * P->out_steps.size() * N;
        std::vector<double2> h(n);
        QP_CUDA(cudaMemcpyAsync(h.data(), w + bp->off_rho, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
        QP_CUDA(cudaStreamSynchronize(s));
        for (size_t i = 0; i < n; ++i) rho_out[i] = qp_c64{h[i].x, h[i].y};
    }
    return QP_OK;
}

void qp_batch_destroy(qp_batch_plan *bp) {
    if (!bp) return;
    qp_plan_destroy(bp->P);
    delete bp;
}

}  // extern "C"
