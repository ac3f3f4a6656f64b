// slide_r.cu -- k_fused_r: S (1 or 2) consecutive slide steps k..k+S-1 (k >= L) of the iterative
// tensor propagator (the Makri-Makarov scheme the paper accelerates; its "BSXFUN" lines
// P:384) in ONE pass over HBM, in place on the ring-buffer ARDM, with the rho(t_k) readout of every
// requested step ("line 169") fused into the same pass.  Used for M = 3, 4 and
// for the partial fusion groups (S < 3) of M = 2 plans (slide3.cu holds the M = 2, S = 3 kernel).
//
// ARDM layout: N^L complex FP64 entries, flat index x = sum_q d_q N^q; time point t
// lives in digit ("ring slot") q = t mod L, so nothing is ever transposed.  Step k contracts slot
// k mod L (holding sigma_{k-L}) and writes sigma_k into the same slot.  For one fibre (all slots
// except the contracted one fixed) with old values a[old]:
//   out[new] = K'(new, last) * exp(Ds(new) Psi(mid)) * sum_old exp(Ds(new) psi_L(old)) a[old]
// Ds = s+ - s- of the new pair state, K' = self factor x bare propagator pair (Eq. 8),
// Psi(mid) = sum_j psi_j(partner at lag j) the Eq. 9 exponent of the kept partners.  Rows with the
// same Ds share one moment S_d = sum_old beta_d(old) a[old] and one factor E_d = exp(delta_d Psi),
// a product of host-built tables (no transcendental in the kernel).
//
// Step fusion: step k only reads/writes slot p = k mod L, and its factors depend on the other slots
// only through their values, so for every fixed value of the other L-S ("outer") slots the N^S
// entries of the "super-fibre" evolve independently through all S steps.  One thread loads its
// super-fibre once, applies S steps in registers (reading rho of each step from the pre-step
// values) and stores it once: HBM traffic per step drops from 32 B to 32/S B per ARDM entry.
//
// Warps are independent: each warp owns a contiguous, static range of (tile, 32-fibre chunk) units
// (tile = T = N^v outer fibres), builds the tile's factor table KU in its own shared-memory slice
// (warp-synchronous, no CTA barrier in the main loop) and sweeps the tile in chunks of 32 outer
// fibres, lane = outer fibre.  Readout accumulators live in shared memory; the CTA reduction at the
// end is in fixed order (deterministic).
#include "common.cuh"

namespace qp {

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused_r(const __grid_constant__ FusedArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    constexpr int Q = cpow(N, S - 1);    // fibres per super-fibre and sub-step
    constexpr int NS = Q * N;
    constexpr int NK = RO ? 2 : 1;
    constexpr int W = BLOCK / 32;
    static_assert(!SYM || (M == 2 && D == 2), "symmetric moments are the M = 2 s = (+s,-s) case");
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    // dynamic shared memory: readout accumulators [S][N][BLOCK] (RO only)
    extern __shared__ double2 dyn_smem[];
    auto accS = reinterpret_cast<double2(*)[RO ? N : 1][RO ? BLOCK : 1]>(dyn_smem);
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < S * S * 2 * D * N; i += BLOCK) (&sIn[0][0][0][0][0])[i] = a.inner[i];
    __shared__ double2 sBeta[S][2][D][N];  // beta_d(old) of each sub-step (first slide: initial-edge classes)
    for (int i = threadIdx.x; i < S * 2 * D * N; i += BLOCK) {
        const int s_ = i / (2 * D * N), kap = (i / (D * N)) % 2, r_ = i % (D * N);
        (&sBeta[0][0][0][0])[i] = a.small[lay.beta(a.var[s_], kap) + r_];
    }
    if constexpr (RO)
        for (int s = 0; s < S; ++s)
            for (int n = 0; n < N; ++n) accS[s][n][threadIdx.x] = make_double2(0.0, 0.0);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // work unit = (tile, chunk of 32 outer fibres); contiguous, static unit range per warp
    // (deterministic readout order); the warp rebuilds its tile tables when the tile changes
    const int CH = (a.T + 31) >> 5;
    const long long n_units = (long long)a.n_tiles * CH;
    const int gw = (int)blockIdx.x * W + warp, nw_tot = (int)gridDim.x * W;
    const long long per = n_units / nw_tot, rem = n_units % nw_tot;
    const long long u_begin = gw * per + min((long long)gw, rem);
    const long long u_end = u_begin + per + (gw < rem ? 1 : 0);
    constexpr int NKU = S * NK * Q * N * N;
    // KI (tile independent, per CTA): K'_kap(new, last) * prod_{i != s} inner_i(class(new), digit_i(r))
    __shared__ double2 KI[S][NK][Q][N][N];
    // per warp: KU = KI * Ehi(tile) and the tile's base offset / 'last' digit
    __shared__ double2 KU[W][S][NK][Q][N][N];
    __shared__ double2 sEhi[W][S][NK][D];
    __shared__ long long sBase[W];
    __shared__ int sLast[W];
    __syncthreads();
    for (int j = threadIdx.x; j < NKU; j += BLOCK) {
        const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                  s = j / (N * N * Q * NK);
        const int c = class_of(M, LAT, nw / M, nw % M);
        double2 e = sK[kap][nw][last];
        if (c > 0)
            for (int i = 0; i < S; ++i)
                if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
        KI[s][kap][rr][nw][last] = e;
    }
    __syncthreads();
    const double2(&ki)[S][NK][Q][N][N] = KI;
    double2(&ku_w)[S][NK][Q][N][N] = KU[warp];
    int cur_tile = -1;
    long long tbase = 0;
    int last_t = 0;
    for (long long u = u_begin; u < u_end; ++u) {
        const int tau = (int)(u / CH), t = (int)(u % CH) * 32 + lane;
        if (tau != cur_tile) {  // warp-synchronous tile setup
            __syncwarp();       // previous tile's KU no longer in use
            cur_tile = tau;
            if (lane < S * NK * D) {
                const int s = lane / (NK * D), kap = (lane / D) % NK, d = lane % D;
                double2 e = make_double2(1.0, 0.0);
                for (int g = 1; g < a.G; ++g)
                    e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
                sEhi[warp][s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
            }
            if (lane == 31) {
                long long b = 0;
                for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
                sBase[warp] = b;
                sLast[warp] = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
            }
            __syncwarp();
            for (int j = lane; j < NKU; j += 32) {
                const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                          s = j / (N * N * Q * NK);
                const int c = class_of(M, LAT, nw / M, nw % M);
                const double2 e = ki[s][kap][rr][nw][last];
                ku_w[s][kap][rr][nw][last] = c > 0 ? cmul(e, sEhi[warp][s][kap][c - 1]) : e;
            }
            __syncwarp();
            tbase = sBase[warp];
            last_t = sLast[warp];
        }
        if (t >= a.T) continue;
        const int2 lo = __ldg(&a.lofs[t]);
        const long long base = tbase + lo.x;
        double2 x[NS];
#pragma unroll
        for (int e = 0; e < NS; ++e) {
            long long o = base;
#pragma unroll
            for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
            x[e] = __ldcs(a.A + o);
        }
        const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool ro = RO && a.rho[s] != nullptr;
            double2 E0[NK][D];  // outer group-0 factor of this outer fibre
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    E0[kap][d] = (kap == 0 || ro) ? __ldg(&a.Etab[(((size_t)s * 2 + kap) * a.G * D + d) * a.X + t])
                                                  : make_double2(0.0, 0.0);
            double2 acc[RO ? N : 1];
#pragma unroll
            for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < Q; ++r) {
                double2 xf[N];
#pragma unroll
                for (int v = 0; v < N; ++v) xf[v] = x[fib_elem<N, S>(s, r, v)];
                const int last = s == 0 ? last0 : fib_digit<N, S>(s, r, s - 1);
                const double2(&ku)[NK][Q][N][N] = ku_w[s];
                double2 S0, m[NK][D];
                if constexpr (SYM) {
                    const double2 u = cadd(xf[0], xf[3]), w = csub(xf[0], xf[3]);
                    const double2 p = cadd(xf[1], xf[2]), q = csub(xf[1], xf[2]);
                    S0 = cadd(u, p);
#pragma unroll
                    for (int kap = 0; kap < NK; ++kap) {
                        if (kap == 1 && !ro) break;
                        const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2],
                                     sh = a.sym[s][kap][3];
                        const double2 A = make_double2(fma(cr, u.x, ch * p.x), fma(cr, u.y, ch * p.y));
                        const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                        m[kap][0] = cadd(A, Bv);
                        m[kap][D - 1] = csub(A, Bv);
                    }
                } else {
                    S0 = xf[0];
#pragma unroll
                    for (int v = 1; v < N; ++v) S0 = cadd(S0, xf[v]);
#pragma unroll
                    for (int kap = 0; kap < NK; ++kap) {
                        if (kap == 1 && !ro) break;
#pragma unroll
                        for (int d = 0; d < D; ++d) {
                            double2 mm = cmul(sBeta[s][kap][d][0], xf[0]);
#pragma unroll
                            for (int v = 1; v < N; ++v) mm = cfma(sBeta[s][kap][d][v], xf[v], mm);
                            m[kap][d] = mm;
                        }
                    }
                }
                if (ro) {
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const double2 pt = cmul(E0[NK - 1][d], m[NK - 1][d]);
#pragma unroll
                        for (int aa = 0; aa < M; ++aa)
#pragma unroll
                            for (int bb = 0; bb < M; ++bb)
                                if (class_of(M, LAT, aa, bb) == d + 1)
                                    acc[RO ? aa * M + bb : 0] =
                                        cfma(ku[NK - 1][r][aa * M + bb][last], pt, acc[RO ? aa * M + bb : 0]);
                    }
                }
                double2 P[D];
#pragma unroll
                for (int d = 0; d < D; ++d) P[d] = cmul(E0[0][d], m[0][d]);
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int nw = aa * M + bb;
                        const int c = class_of(M, LAT, aa, bb);
                        const double2 o = cmul(ku[0][r][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                        x[fib_elem<N, S>(s, r, nw)] = o;
                        if (ro && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
                    }
            }
            if (ro) {
#pragma unroll
                for (int n = 0; n < N; ++n)
                    accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0] =
                        cadd(accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0], acc[RO ? n : 0]);
            }
        }
#pragma unroll
        for (int e = 0; e < NS; ++e) {
            long long o = base;
#pragma unroll
            for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
            __stcs(a.A + o, x[e]);
        }
    }
    if constexpr (RO) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr) {
                double2 tt[N];
#pragma unroll
                for (int n = 0; n < N; ++n) tt[n] = accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0];
                reduce_finalize<N, BLOCK>(tt, a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                          a.rho_accumulate != 0);
            }
    }
}

// ---------------------------------------------------------------------------------- dispatch
// (M, S) -> block, tile digits v (T = N^v outer fibres per tile), min blocks per SM
#define QP_FUSED_R_CFGS(X) \
    X(2, 1, 256, 4, 2)     \
    X(2, 2, 256, 4, 2)     \
    X(3, 1, 256, 3, 2)     \
    X(4, 1, 64, 2, 4)

namespace {
template <int M, int S, int BLOCK>
constexpr size_t fused_r_dyn_smem(bool ro) {
    return (ro ? (size_t)S * M * M * BLOCK : 0) * 16;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB>
cudaError_t fused_r_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    const size_t dyn = fused_r_dyn_smem<M, S, BLOCK>(ro);
    if (ro) {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true><<<grid, BLOCK, dyn, s>>>(a);
    } else {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false><<<grid, BLOCK, dyn, s>>>(a);
    }
    return cudaGetLastError();
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB>
int fused_r_occ_t() {
    int o1 = 0, o2 = 0;
    const size_t d1 = fused_r_dyn_smem<M, S, BLOCK>(true), d2 = fused_r_dyn_smem<M, S, BLOCK>(false);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d2);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, BLOCK, d2);
    return o1 < o2 ? o1 : o2;
}
}  // namespace

bool fused_r_has(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return true;
    QP_FUSED_R_CFGS(X)
#undef X
    return false;
}
int fused_r_tile_digits(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return V;
    QP_FUSED_R_CFGS(X)
#undef X
    return -1;
}
int fused_r_block(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return B;
    QP_FUSED_R_CFGS(X)
#undef X
    return 0;
}

cudaError_t launch_fused_r(int M, bool lattice, bool sym, int S, const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
#define X(M_, S_, B, V, MB)                                                                       \
    if (M == M_ && S == S_) {                                                                     \
        if (M_ == 2 && sym) return fused_r_t<M_, false, (M_ == 2), S_, B, MB>(a, ro, grid, s);    \
        if (M_ > 2 && lattice) return fused_r_t<M_, (M_ > 2), false, S_, B, MB>(a, ro, grid, s);  \
        return fused_r_t<M_, false, false, S_, B, MB>(a, ro, grid, s);                            \
    }
    QP_FUSED_R_CFGS(X)
#undef X
    return cudaErrorInvalidValue;
}

int fused_r_occupancy(int M, bool lattice, bool sym, int S) {
#define X(M_, S_, B, V, MB)                                                             \
    if (M == M_ && S == S_) {                                                           \
        if (M_ == 2 && sym) return fused_r_occ_t<M_, false, (M_ == 2), S_, B, MB>();    \
        if (M_ > 2 && lattice) return fused_r_occ_t<M_, (M_ > 2), false, S_, B, MB>();  \
        return fused_r_occ_t<M_, false, false, S_, B, MB>();                            \
    }
    QP_FUSED_R_CFGS(X)
#undef X
    return 0;
}

}  // namespace qp
