// batch.cu -- batched QUAPI sweeps: many small independent problems (the paper's
// use case: rho_11(t) of the driven quantum dot swept over pulse areas) propagated in ONE
// kernel launch.  One CTA owns one problem for the whole run: per step it forms the step's
// propagator pair from H_b(k) = H0 + f_b(k) H1 (Omega(t) of P:288), then performs the growth
// (k < L) or slide (k >= L) update of its ARDM in place and, for output steps, the fused readout
// rho_b(t_k) from A_{k-1} (terminal classes) with a fixed-order block reduction (no atomics: run-to-run
// bit-identical).  The per-problem ARDM (16 N^L bytes) stays L2-resident for the sweep sizes of
// interest; steps are separated by CTA barriers only (no kernel launch per step).
//
// Same mathematics as kernels.cu: for a fibre along the contracted slot p,
//   out[new] = K'(new, last) exp(Ds(new) Psi(mid)) sum_old exp(Ds(new) psi_L(old)) a[old]
// with the Eq. 9 exponents evaluated directly from the per-lag psi tables (Psi = sum over the kept
// partners, one complex exp per Delta-s class), so no per-launch-set factor tables are needed.
#include "qp_internal.h"

namespace qp {
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

template <int M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_batch(const __grid_constant__ BatchArgs a) {
    constexpr int N = M * M, W = BLOCK / 32, DM = kMaxD;
    const int b = blockIdx.x, L = a.L;
    double2 *const A = a.A + (size_t)b * a.NL;
    extern __shared__ double2 tabs[];  // psi_eta, psi_E, psi_TI [L+1][N]; psi_self [2][N]
    const int ntab = (3 * (L + 1) + 2) * N;
    double2 *const pEta = tabs, *const pE = tabs + (L + 1) * N, *const pTI = tabs + 2 * (L + 1) * N,
                   *const pSelf = tabs + 3 * (L + 1) * N;
    __shared__ double2 sH0[M][M], sH1[M][M], sU[M][M];
    __shared__ double2 sKp[2][N][N];     // K'(new, last) for propagate (0) / terminal (1) self classes
    __shared__ double2 sBeta[2][DM][N];  // exp(delta_d psi_L(old)): propagate / terminal
    __shared__ double2 red[W][N];
    const double2 *src = a.ptab ? a.ptab + (size_t)b * ntab : a.tab;  // per-problem bath or the shared one
    for (int i = threadIdx.x; i < ntab; i += BLOCK) tabs[i] = src[i];
    if (threadIdx.x < M * M) {
        (&sH0[0][0])[threadIdx.x] = a.tab[ntab + threadIdx.x];
        (&sH1[0][0])[threadIdx.x] = a.tab[ntab + M * M + threadIdx.x];
    }
    __syncthreads();
    const double2 *r0 = a.rho0 + (size_t)b * N;
    if (threadIdx.x < N) {  // A_0(sigma_0) = rho0(sigma_0) I(sigma_0, sigma_0; eta_00 = G(1/2))
        const int n = threadIdx.x;
        A[n] = bmul(r0[n], bexp(bscale(pSelf[N + n], a.dsig[n])));
        if (a.out_idx[0] >= 0) a.rho[((size_t)b * a.n_out + a.out_idx[0]) * N + n] = r0[n];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (long long k = 1; k <= a.n_steps; ++k) {
        const bool ro = a.out_idx[k] >= 0;
        if (threadIdx.x == 0 && (k == 1 || a.f != nullptr)) {  // the step's propagator
            const double fk = a.f ? a.f[(size_t)b * a.n_steps + (k - 1)] : 0.0;
            double2 H[M][M], U[M][M];
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) H[i][j] = make_double2(sH0[i][j].x + fk * sH1[i][j].x, sH0[i][j].y + fk * sH1[i][j].y);
            expm_herm<M>(H, a.dt, U);
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j) sU[i][j] = U[i][j];
        }
        __syncthreads();  // sU ready; previous step's writes visible
        for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) {
            const int kap = i / (N * N), nw = (i / N) % N, last = i % N;
            // K(new, last) = U[a, a'] conj(U[b, b']) (Eq. 8), times the self factor of the new point
            const double2 ua = sU[nw / M][last / M], ub = sU[nw % M][last % M];
            const double2 kk = bmul(ua, make_double2(ub.x, -ub.y));
            sKp[kap][nw][last] = bmul(kk, bexp(bscale(pSelf[kap * N + nw], a.dsig[nw])));
        }
        if (k >= L)
            for (int i = threadIdx.x; i < 2 * a.D * N; i += BLOCK) {
                const int kap = i / (a.D * N), d = (i / N) % a.D, old = i % N;
                // lag-L partner sigma_{k-L}: propagate eta_L (E_L at k = L), terminal E_L (TI_L at k = L)
                const double2 ps = kap == 0 ? (k == L ? pE[L * N + old] : pEta[L * N + old])
                                            : (k == L ? pTI[L * N + old] : pE[L * N + old]);
                sBeta[kap][d][old] = bexp(bscale(ps, a.delta[d]));
            }
        __syncthreads();
        double2 acc[N];
#pragma unroll
        for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
        if (k < L) {  // growth: A_k[x + v N^k] = K'(v, d_{k-1}) exp(Ds(v) Psi_k(x)) A_{k-1}[x]
            long long nin = 1;
            for (int t = 0; t < k; ++t) nin *= N;
            for (long long x = threadIdx.x; x < nin; x += BLOCK) {
                int dig[kMaxL];
                long long r = x;
                for (int t = 0; t < k; ++t) dig[t] = (int)(r % N), r /= N;
                const int last = dig[k - 1];
                double2 Pp = make_double2(0.0, 0.0), Pt = make_double2(0.0, 0.0);
                for (int j = 1; j <= k; ++j) {  // partner point k - j in digit k - j
                    const int sg = dig[k - j];
                    Pp = badd(Pp, j < k ? pEta[j * N + sg] : pE[k * N + sg]);
                    Pt = badd(Pt, j < k ? pE[j * N + sg] : pTI[k * N + sg]);
                }
                const double2 ax = A[x];
                double2 Ep[DM], Et[DM];
                for (int d = 0; d < a.D; ++d) {
                    Ep[d] = bexp(bscale(Pp, a.delta[d]));
                    if (ro) Et[d] = bexp(bscale(Pt, a.delta[d]));
                }
                if (ro)
#pragma unroll
                    for (int n = 0; n < N; ++n) {
                        const int c = a.cls[n];
                        acc[n] = bfma(c ? bmul(sKp[1][n][last], Et[c - 1]) : sKp[1][n][last], ax, acc[n]);
                    }
#pragma unroll
                for (int v = N - 1; v >= 0; --v) {  // v = 0 overwrites x itself: last
                    const int c = a.cls[v];
                    A[x + v * nin] = bmul(c ? bmul(sKp[0][v][last], Ep[c - 1]) : sKp[0][v][last], ax);
                }
            }
        } else {  // slide on slot p = k mod L
            const int p = (int)(k % L);
            long long Pp_ = 1;
            for (int t = 0; t < p; ++t) Pp_ *= N;
            const long long nf = a.NL / N;
            for (long long fi = threadIdx.x; fi < nf; fi += BLOCK) {
                const long long xb = (fi % Pp_) + (fi / Pp_) * Pp_ * N;
                int dig[kMaxL];
                long long r = xb;
                for (int t = 0; t < L; ++t) dig[t] = (int)(r % N), r /= N;
                const int last = dig[(p - 1 + L) % L];
                double2 Pp = make_double2(0.0, 0.0), Pt = make_double2(0.0, 0.0);
                for (int q = 0; q < L; ++q) {
                    if (q == p) continue;
                    const int lag = (p - q + L) % L;  // 1..L-1
                    Pp = badd(Pp, pEta[lag * N + dig[q]]);
                    Pt = badd(Pt, pE[lag * N + dig[q]]);
                }
                double2 xo[N];
#pragma unroll
                for (int o = 0; o < N; ++o) xo[o] = A[xb + o * Pp_];
                double2 S0 = make_double2(0.0, 0.0);
#pragma unroll
                for (int o = 0; o < N; ++o) S0 = badd(S0, xo[o]);
                double2 mP[DM], mT[DM];
                for (int d = 0; d < a.D; ++d) {
                    const double2 Ed = bexp(bscale(Pp, a.delta[d]));
                    double2 m = make_double2(0.0, 0.0);
#pragma unroll
                    for (int o = 0; o < N; ++o) m = bfma(sBeta[0][d][o], xo[o], m);
                    mP[d] = bmul(Ed, m);
                    if (ro) {
                        const double2 Td = bexp(bscale(Pt, a.delta[d]));
                        double2 mt = make_double2(0.0, 0.0);
#pragma unroll
                        for (int o = 0; o < N; ++o) mt = bfma(sBeta[1][d][o], xo[o], mt);
                        mT[d] = bmul(Td, mt);
                    }
                }
#pragma unroll
                for (int n = 0; n < N; ++n) {
                    const int c = a.cls[n];
                    A[xb + n * Pp_] = bmul(sKp[0][n][last], c ? mP[c - 1] : S0);
                    if (ro) acc[n] = bfma(sKp[1][n][last], c ? mT[c - 1] : S0, acc[n]);
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

template <int M>
cudaError_t batch_t(const BatchArgs &a, int B, cudaStream_t s) {
    const size_t dyn = batch_dyn_smem(M, a.L);
    cudaFuncSetAttribute(k_batch<M, kBatchBlock>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k_batch<M, kBatchBlock><<<B, kBatchBlock, dyn, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

size_t batch_dyn_smem(int M, int L) { return (size_t)(3 * (L + 1) + 2) * M * M * sizeof(double2); }

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
