// batch.cu -- batched QUAPI sweeps: many small independent problems (the paper's
// use case: rho_11(t) of the driven quantum dot swept over pulse areas) propagated in ONE
// kernel launch.  One CTA owns one problem for the whole run: per step it forms the step's
// propagator pair from H_b(k) = H0 + f_b(k) H1 (Omega(t) of P:288), then performs the growth
// (k < L) or slide (k >= L) update of its ARDM in place and, for output steps, the fused readout
// rho_b(t_k) from A_{k-1} (terminal classes) with a fixed-order block reduction (no atomics: run-to-run
// bit-identical).  The per-problem ARDM (16 N^L bytes) stays L2-resident for the sweep sizes of
// interest; steps are separated by CTA barriers only (no kernel launch per step).
//
// Same mathematics as the single-problem kernels: for a fibre along the contracted
// slot p,
//   out[new] = K'(new, last) exp(Ds(new) Psi(mid)) sum_old exp(Ds(new) psi_L(old)) a[old]
// with exp(delta_d Psi(mid)) a product over the L-1 kept partners.  Per slide step the CTA builds
// digit-group tables in shared memory -- for groups of w consecutive kept slots (w digits of the
// fibre index), the product of their per-lag factors for every digit combination -- so a fibre
// multiplies ceil((L-1)/w) table entries per class instead of L-1 (the single-problem path's
// Etab groups, built per step from the problem's own psi tables).
#include "qp_internal.h"

namespace qp {

// Group width w (digits) of the slide factor tables: the widest w <= 4 with N^w <= 256 whose tables
// (both kinds, D classes, all groups) stay within 48 KB and hold at most a quarter as many entries
// as a step has fibres (the per-step table build stays small against the fibre loop); entries per
// (kind, class): full groups of N^w plus the last group.
__host__ __device__ inline int batch_bw(int M, int L, int D) {
    const int N = M * M;
    long long nf = 1;
    for (int i = 0; i < L - 1; ++i) nf *= N;
    for (int w = 4; w > 1; --w) {
        long long nw = 1;
        for (int i = 0; i < w; ++i) nw *= N;
        if (nw > 256) continue;
        long long tot = 0;
        for (int r = L - 1; r > 0; r -= w) {
            long long e = 1;
            for (int i = 0; i < (r < w ? r : w); ++i) e *= N;
            tot += e;
        }
        if (2LL * D * tot * 16 <= 48 * 1024 && 4 * tot <= nf) return w;
    }
    return 1;
}
__host__ __device__ inline long long batch_gtot(int M, int L, int w) {
    const int N = M * M;
    long long tot = 0;
    for (int r = L - 1; r > 0; r -= w) {
        long long e = 1;
        for (int i = 0; i < (r < w ? r : w); ++i) e *= N;
        tot += e;
    }
    return tot;
}

namespace {

__device__ __forceinline__ double2 bmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 bfma(double2 a, double2 b, double2 c) {
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 badd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 bexp(double2 z) {
    double s, c;
    sincos(z.y, &s, &c);
    const double e = exp(z.x);
    return make_double2(e * c, e * s);
}
__device__ __forceinline__ double2 bscale(double2 a, double r) { return make_double2(a.x * r, a.y * r); }

// U = exp(-i H dt) for a Hermitian M x M matrix H (one thread).  M = 2: closed form through the
// Pauli decomposition H = h0 + h.sigma; M > 2: Taylor series of degree 18 after scaling X = -i H dt
// to ||X||_inf <= 1/2, then squaring.
template <int M>
__device__ void expm_herm(const double2 (&H)[M][M], double dt, double2 (&U)[M][M]) {
    if constexpr (M == 2) {
        const double h0 = 0.5 * (H[0][0].x + H[1][1].x), hz = 0.5 * (H[0][0].x - H[1][1].x);
        const double hx = H[0][1].x, hy = -H[0][1].y;  // H01 = hx - i hy
        const double n = sqrt(hx * hx + hy * hy + hz * hz), th = n * dt;
        double sn, cs, s0, c0;
        sincos(th, &sn, &cs);
        sincos(h0 * dt, &s0, &c0);
        const double r = n > 0.0 ? sn / n : dt;  // sin(n dt)/n
        // exp(-i(h.sigma)dt) = cos(th) - i sin(th)/n (hx sx + hy sy + hz sz)
        const double2 e00 = make_double2(cs, -r * hz), e11 = make_double2(cs, r * hz);
        const double2 e01 = make_double2(-r * hy, -r * hx), e10 = make_double2(r * hy, -r * hx);
        const double2 ph = make_double2(c0, -s0);
        U[0][0] = bmul(ph, e00), U[0][1] = bmul(ph, e01), U[1][0] = bmul(ph, e10), U[1][1] = bmul(ph, e11);
    } else {
        double2 X[M][M];
        double nrm = 0.0;
        for (int i = 0; i < M; ++i) {
            double rs = 0.0;
            for (int j = 0; j < M; ++j) {
                X[i][j] = make_double2(H[i][j].y * dt, -H[i][j].x * dt);  // -i H dt
                rs += hypot(X[i][j].x, X[i][j].y);
            }
            nrm = fmax(nrm, rs);
        }
        int sq = 0;
        while (nrm > 0.5) nrm *= 0.5, ++sq;
        const double sc = ldexp(1.0, -sq);
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) X[i][j] = bscale(X[i][j], sc);
        // Horner: E = I + X/1 (I + X/2 (I + ... (I + X/18)))
        double2 E[M][M];
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) E[i][j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
        for (int t = 18; t >= 1; --t) {
            double2 T[M][M];
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) {
                    double2 acc = make_double2(0.0, 0.0);
                    for (int l = 0; l < M; ++l) acc = bfma(X[i][l], E[l][j], acc);
                    T[i][j] = bscale(acc, 1.0 / t);
                }
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) E[i][j] = make_double2(T[i][j].x + (i == j ? 1.0 : 0.0), T[i][j].y);
        }
        for (int q = 0; q < sq; ++q) {
            double2 T[M][M];
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) {
                    double2 acc = make_double2(0.0, 0.0);
                    for (int l = 0; l < M; ++l) acc = bfma(E[i][l], E[l][j], acc);
                    T[i][j] = acc;
                }
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) E[i][j] = T[i][j];
        }
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < M; ++j) U[i][j] = E[i][j];
    }
}

// SMEM: the problem's whole ARDM lives in shared memory for the run (small L), written back at the end.
template <int M, int BLOCK, bool SMEM, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_batch(const __grid_constant__ BatchArgs a) {
    constexpr int N = M * M, W = BLOCK / 32;
    constexpr int DMX = M * (M - 1);  // largest class count for this M (general s)
    const int b = blockIdx.x, L = a.L, D = a.D;
    // dynamic shared memory: psi_eta, psi_E, psi_TI [L+1][N]; psi_self [2][N]; then the slide factor
    // tables sT[kap][d][j][sigma] = exp(delta_d psi^kap_j(sigma)) (kap 0: eta_j rows, propagate; 1: E_j
    // rows, terminal; j = 0..L-1, row 0 = 1); then (SMEM) the ARDM
    extern __shared__ double2 tabs[];
    const int ntab = (3 * (L + 1) + 2) * N;
    double2 *const pEta = tabs, *const pE = tabs + (L + 1) * N, *const pTI = tabs + 2 * (L + 1) * N,
                   *const pSelf = tabs + 3 * (L + 1) * N;
    double2 *const sT = tabs + ntab;
    const int nT = 2 * D * L * N;
    // slide digit-group tables gT[kap][d][g * N^w + v] (rebuilt every slide step)
    const int bw = batch_bw(M, L, D), G = (L - 1 + bw - 1) / bw;
    const int gtot = (int)batch_gtot(M, L, bw);
    unsigned Nw = 1;
    for (int i = 0; i < bw; ++i) Nw *= N;
    double2 *const gT = sT + nT;
    double2 *const A = SMEM ? gT + 2 * D * gtot : a.A + (size_t)b * a.NL;
    // the steps' propagators, computed for a chunk of CH steps at once (one step per thread) instead of
    // by one thread inside every step
    constexpr int CH = 8192 / (M * M * 16);
    __shared__ double2 sH0[M][M], sH1[M][M], sU[CH][M][M];
    __shared__ double2 sKp[2][N][N];     // K'(new, last) for propagate (0) / terminal (1) self classes
    // exp(delta_d psi_L(old)) of the lag-L partner [variant][kap][d][old]: variant 0 (k > L) propagate
    // eta_L / terminal E_L; variant 1 (k == L, partner sigma_0) propagate E_L / terminal TI_L
    __shared__ double2 sBetaV[2][2][DMX][N];
    __shared__ double2 sSelf[2][N];      // exp(Ds(n) psi_self(n)): interior G(1) / end G(1/2) self factor
    __shared__ double2 red[W][N];
    const double2 *src = a.ptab ? a.ptab + (size_t)b * ntab : a.tab;  // per-problem bath or the shared one
    for (int i = threadIdx.x; i < ntab; i += BLOCK) tabs[i] = src[i];
    if (threadIdx.x < M * M) {
        (&sH0[0][0])[threadIdx.x] = a.tab[ntab + threadIdx.x];
        (&sH1[0][0])[threadIdx.x] = a.tab[ntab + M * M + threadIdx.x];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nT; i += BLOCK) {  // read after the step loop's first barrier
        const int kap = i / (D * L * N), d = (i / (L * N)) % D, j = (i / N) % L, sg = i % N;
        sT[i] = j == 0 ? make_double2(1.0, 0.0) : bexp(bscale((kap == 0 ? pEta : pE)[j * N + sg], a.delta[d]));
    }
    for (int i = threadIdx.x; i < 2 * 2 * D * N; i += BLOCK) {  // step-independent factors, built once
        const int var = i / (2 * D * N), kap = (i / (D * N)) % 2, d = (i / N) % D, old = i % N;
        const double2 ps = kap == 0 ? (var ? pE[L * N + old] : pEta[L * N + old])
                                    : (var ? pTI[L * N + old] : pE[L * N + old]);
        sBetaV[var][kap][d][old] = bexp(bscale(ps, a.delta[d]));
    }
    for (int i = threadIdx.x; i < 2 * N; i += BLOCK) sSelf[i / N][i % N] = bexp(bscale(pSelf[i], a.dsig[i % N]));
    const double2 *r0 = a.rho0 + (size_t)b * N;
    if (threadIdx.x < N) {  // A_0(sigma_0) = rho0(sigma_0) I(sigma_0, sigma_0; eta_00 = G(1/2))
        const int n = threadIdx.x;
        A[n] = bmul(r0[n], bexp(bscale(pSelf[N + n], a.dsig[n])));
        if (a.out_idx[0] >= 0) a.rho[((size_t)b * a.n_out + a.out_idx[0]) * N + n] = r0[n];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool drive = a.f != nullptr;
    // divisions by powers of N: shifts and masks when N is a power of two (M = 2, 4)
    constexpr bool POW2 = (N & (N - 1)) == 0;
    auto udiv = [&](unsigned x, unsigned pw) -> unsigned {
        if constexpr (POW2) return x >> (31 - __clz(pw));
        else return x / pw;
    };
    auto umod = [&](unsigned x, unsigned pw) -> unsigned {
        if constexpr (POW2) return x & (pw - 1);
        else return x % pw;
    };
    for (long long k = 1; k <= a.n_steps; ++k) {
        const bool ro = a.out_idx[k] >= 0;
        if ((k - 1) % CH == 0 && (k == 1 || drive)) {  // propagators of steps k .. k + CH - 1
            const long long kk = k + threadIdx.x;
            if (threadIdx.x < CH && kk <= a.n_steps && (drive || threadIdx.x == 0)) {
                const double fk = drive ? a.f[(size_t)b * a.n_steps + (kk - 1)] : 0.0;
                double2 H[M][M], U[M][M];
                for (int i = 0; i < M; ++i)
                    for (int j = 0; j < M; ++j)
                        H[i][j] = make_double2(sH0[i][j].x + fk * sH1[i][j].x, sH0[i][j].y + fk * sH1[i][j].y);
                expm_herm<M>(H, a.dt, U);
                for (int i = 0; i < M; ++i)
                    for (int j = 0; j < M; ++j) sU[threadIdx.x][i][j] = U[i][j];
            }
        }
        __syncthreads();  // sU ready; previous step's writes visible
        if (k == 1 || drive) {
            const double2(&U)[M][M] = sU[drive ? (int)((k - 1) % CH) : 0];
            for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) {
                const int kap = i / (N * N), nw = (i / N) % N, last = i % N;
                // K(new, last) = U[a, a'] conj(U[b, b']) (Eq. 8), times the self factor of the new point
                const double2 ua = U[nw / M][last / M], ub = U[nw % M][last % M];
                sKp[kap][nw][last] = bmul(bmul(ua, make_double2(ub.x, -ub.y)), sSelf[kap][nw]);
            }
            __syncthreads();
        }
        const double2(*sBeta)[DMX][N] = sBetaV[k == L ? 1 : 0];
        double2 acc[N];
#pragma unroll
        for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
        if (k < L) {  // growth: A_k[x + v N^k] = K'(v, d_{k-1}) exp(Ds(v) Psi_k(x)) A_{k-1}[x]
            long long nin = 1;
            for (int t = 0; t < k; ++t) nin *= N;
            for (long long x = threadIdx.x; x < nin; x += BLOCK) {
                int last = 0;
                double2 Pp = make_double2(0.0, 0.0), Pt = make_double2(0.0, 0.0);
                long long r = x;
                for (int t = 0; t < k; ++t) {  // digit t holds point t, the partner at lag j = k - t
                    const int sg = (int)(r % N), j = k - t;
                    r /= N;
                    if (t == k - 1) last = sg;
                    Pp = badd(Pp, j < k ? pEta[j * N + sg] : pE[k * N + sg]);
                    Pt = badd(Pt, j < k ? pE[j * N + sg] : pTI[k * N + sg]);
                }
                const double2 ax = A[x];
                double2 Ep[DMX] = {}, Et[DMX] = {};
#pragma unroll
                for (int d = 0; d < DMX; ++d) {
                    if (d >= D) break;
                    Ep[d] = bexp(bscale(Pp, a.delta[d]));
                    if (ro) Et[d] = bexp(bscale(Pt, a.delta[d]));
                }
#pragma unroll
                for (int v = N - 1; v >= 0; --v) {  // v = 0 overwrites x itself: last
                    const int c = a.cls[v];
                    double2 fp = make_double2(1.0, 0.0), ft = make_double2(1.0, 0.0);
#pragma unroll
                    for (int d = 0; d < DMX; ++d)  // register-resident select
                        if (c == d + 1) fp = Ep[d], ft = Et[d];
                    if (ro) acc[v] = bfma(bmul(sKp[1][v][last], ft), ax, acc[v]);
                    A[x + v * nin] = bmul(bmul(sKp[0][v][last], fp), ax);
                }
            }
        } else {  // slide on slot p = k mod L: exp(delta_d Psi) as products of digit-group table entries
            const int p = (int)(k % L);
            unsigned Pp_ = 1;
            for (int t = 0; t < p; ++t) Pp_ *= N;
            // the fibre index fi enumerates the kept slots q != p in increasing order (rank r = q or
            // q - 1); the previous point sigma_{k-1} sits in slot p - 1 (rank p - 1), or L - 1 (rank L - 2)
            unsigned Pl = 1;
            for (int t = 0; t < (p >= 1 ? p - 1 : L - 2); ++t) Pl *= N;
            for (int i = threadIdx.x; i < (ro ? 2 : 1) * D * gtot; i += BLOCK) {
                const int kd = i / gtot, e = i % gtot, g = e / (int)Nw, kap = kd / D, d = kd % D;
                unsigned v = (unsigned)(e - g * (int)Nw);
                double2 pr = make_double2(1.0, 0.0);
                for (int j = 0; j < bw && g * bw + j < L - 1; ++j, v /= N) {
                    const int rk = g * bw + j, q = rk < p ? rk : rk + 1;
                    pr = bmul(pr, sT[((kap * D + d) * L + (p - q + L) % L) * N + (int)(v % N)]);  // lag 1..L-1
                }
                gT[i] = pr;
            }
            __syncthreads();
            const unsigned nf = (unsigned)(a.NL / N);  // N^(L-1) < 2^32 for batch problems
            for (unsigned fi = threadIdx.x; fi < nf; fi += BLOCK) {
                const unsigned xb = udiv(fi, Pp_) * Pp_ * N + umod(fi, Pp_);
                const int last = (int)umod(udiv(fi, Pl), (unsigned)N);
                double2 Ep[DMX], Et[DMX];
                {
                    const unsigned v0 = G > 1 ? umod(fi, Nw) : fi;
#pragma unroll
                    for (int d = 0; d < DMX; ++d)
                        if (d < D) {
                            Ep[d] = gT[d * gtot + v0];
                            Et[d] = ro ? gT[(D + d) * gtot + v0] : make_double2(0.0, 0.0);
                        }
                }
                unsigned rem = udiv(fi, Nw);
                for (int g = 1; g < G; ++g, rem = udiv(rem, Nw)) {
                    const int o = g * (int)Nw + (int)(g < G - 1 ? umod(rem, Nw) : rem);
#pragma unroll
                    for (int d = 0; d < DMX; ++d)
                        if (d < D) {
                            Ep[d] = bmul(Ep[d], gT[d * gtot + o]);
                            if (ro) Et[d] = bmul(Et[d], gT[(D + d) * gtot + o]);
                        }
                }
                double2 xo[N];
#pragma unroll
                for (int o = 0; o < N; ++o) xo[o] = A[xb + o * Pp_];
                double2 S0 = make_double2(0.0, 0.0);
#pragma unroll
                for (int o = 0; o < N; ++o) S0 = badd(S0, xo[o]);
                double2 mP[DMX] = {}, mT[DMX] = {};
#pragma unroll
                for (int d = 0; d < DMX; ++d) {
                    if (d >= D) break;
                    double2 m = make_double2(0.0, 0.0);
#pragma unroll
                    for (int o = 0; o < N; ++o) m = bfma(sBeta[0][d][o], xo[o], m);
                    mP[d] = bmul(Ep[d], m);
                    if (ro) {
                        double2 mt = make_double2(0.0, 0.0);
#pragma unroll
                        for (int o = 0; o < N; ++o) mt = bfma(sBeta[1][d][o], xo[o], mt);
                        mT[d] = bmul(Et[d], mt);
                    }
                }
#pragma unroll
                for (int n = 0; n < N; ++n) {
                    const int c = a.cls[n];
                    double2 mp = S0, mt = S0;
#pragma unroll
                    for (int d = 0; d < DMX; ++d)  // register-resident select (no local-memory indexing)
                        if (c == d + 1) mp = mP[d], mt = mT[d];
                    A[xb + n * Pp_] = bmul(sKp[0][n][last], mp);
                    if (ro) acc[n] = bfma(sKp[1][n][last], mt, acc[n]);
                }
            }
        }
        if (ro) {  // fixed-order block reduction of rho_b(t_k)
#pragma unroll
            for (int n = 0; n < N; ++n) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    acc[n].x += __shfl_xor_sync(0xffffffffu, acc[n].x, o);
                    acc[n].y += __shfl_xor_sync(0xffffffffu, acc[n].y, o);
                }
                if (lane == 0) red[warp][n] = acc[n];
            }
            __syncthreads();
            if (threadIdx.x < N) {
                double2 t = red[0][threadIdx.x];
                for (int w = 1; w < W; ++w) t = badd(t, red[w][threadIdx.x]);
                a.rho[((size_t)b * a.n_out + a.out_idx[k]) * N + threadIdx.x] = t;
            }
        }
        __syncthreads();  // step complete before the next step reads A
    }
    if constexpr (SMEM)  // the caller's ARDM buffer holds the final A, as on the global-memory path
        for (long long i = threadIdx.x; i < a.NL; i += BLOCK) a.A[(size_t)b * a.NL + i] = A[i];
}

// psi(sigma', e) = -(e s+(sigma') - conj(e) s-(sigma')) (Eq. 9 summand without the later point's Delta s)
// for every eta class of problem b: rows j = 1..L of psi_eta / psi_E / psi_TI, then psi_self [2][N].
struct PsiArgs {
    double s[kMaxM];
    int M, L;
};
__global__ void k_psi(const PsiArgs p, const double2 *__restrict__ eta, double2 *__restrict__ ptab, int B) {
    const int N = p.M * p.M, L = p.L, nc = 3 * L + 2, ntab = (3 * (L + 1) + 2) * N;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (long long)B * ntab;
         i += (long long)gridDim.x * blockDim.x) {
        const int b = (int)(i / ntab), r = (int)(i % ntab), row = r / N, sg = r % N;
        int c = -1;  // eta class of this row (qp_plan_eta order), -1: unused row 0 of a lag table
        if (row < 3 * (L + 1)) {
            const int g = row / (L + 1), j = row % (L + 1);
            if (j > 0) c = 2 + g * L + (j - 1);
        } else {
            c = row - 3 * (L + 1);  // 0: self interior, 1: self end
        }
        double2 v = make_double2(0.0, 0.0);
        if (c >= 0) {
            const double2 e = eta[(size_t)b * nc + c];
            const double sp = p.s[sg / p.M], sm = p.s[sg % p.M];
            v = make_double2(-(e.x * sp - e.x * sm), -(e.y * sp + e.y * sm));
        }
        ptab[i] = v;
    }
}

constexpr size_t kBatchSmemArdmMax = 100 * 1024;  // ARDM + tables in shared memory up to this size

template <int M, bool SMEM, int MINB>
cudaError_t batch_launch(const BatchArgs &a, int B, size_t dyn, cudaStream_t s) {
    cudaFuncSetAttribute(k_batch<M, kBatchBlock, SMEM, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k_batch<M, kBatchBlock, SMEM, MINB><<<B, kBatchBlock, dyn, s>>>(a);
    return cudaGetLastError();
}

template <int M>
cudaError_t batch_t(const BatchArgs &a, int B, cudaStream_t s) {
    const size_t tab = batch_dyn_smem(M, a.L, a.D);
    const size_t full = tab + (size_t)a.NL * sizeof(double2);
    const bool smem = full <= kBatchSmemArdmMax;
    // M = 2: 3 CTAs (24 warps, 80 registers) per SM for the shared-memory-resident ARDM, 2 CTAs (128
    // registers, no spills) when the ARDM stays in global memory (measured: L = 5 13.8 vs 15.0 ms, L = 7
    // 0.198 vs 0.177 s for 1024 problems x 1000 steps)
    if (M == 2 && smem)
        return smem ? batch_launch<M, true, 3>(a, B, full, s) : batch_launch<M, false, 3>(a, B, tab, s);
    return smem ? batch_launch<M, true, M == 2 ? 2 : 1>(a, B, full, s) : batch_launch<M, false, M == 2 ? 2 : 1>(a, B, tab, s);
}

}  // namespace

size_t batch_dyn_smem(int M, int L, int D) {
    return ((size_t)(3 * (L + 1) + 2) * M * M + (size_t)2 * D * L * M * M + (size_t)2 * D * batch_gtot(M, L, batch_bw(M, L, D))) *
           sizeof(double2);
}

cudaError_t launch_psi_tables(int M, const double (&s)[kMaxM], const double2 *eta, double2 *ptab, int B, int L, cudaStream_t st) {
    PsiArgs p{};
    for (int i = 0; i < kMaxM; ++i) p.s[i] = s[i];
    p.M = M, p.L = L;
    const long long n = (long long)B * (3 * (L + 1) + 2) * M * M;
    const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    k_psi<<<grid, 256, 0, st>>>(p, eta, ptab, B);
    return cudaGetLastError();
}

cudaError_t launch_batch(int M, const BatchArgs &a, int B, cudaStream_t s) {
    switch (M) {
    case 2: return batch_t<2>(a, B, s);
    case 3: return batch_t<3>(a, B, s);
    case 4: return batch_t<4>(a, B, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace qp
