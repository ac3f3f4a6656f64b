// kernels.cu -- sm_100a kernels of the QUAPI tensor-propagator step (arXiv 1205.6872).
//
// k_fused : S consecutive time steps k..k+S-1 (k >= L) of the iterative tensor propagator (the
//           Makri-Makarov scheme the paper accelerates; the "BSXFUN" lines P:384) in ONE
//           pass over HBM, in place on a ring-buffer ARDM, with the rho(t) readout of every
//           requested step ("line 169") fused into the same pass.
// k_grow  : growth steps 1 <= k < L (no contraction; the tensor gains one digit per step).
//
// ARDM layout: N^L complex FP64 entries, flat index x = sum_q d_q N^q; time point
// t lives in digit ("ring slot") q = t mod L, so nothing is ever transposed.  Step k contracts
// slot k mod L (holding sigma_{k-L}) and writes sigma_k into the same slot.  For one fibre (all
// slots except the contracted one fixed) with old values a[old]:
//   out[new] = K'(new, last) * exp(Ds(new) Psi(mid)) * sum_old exp(Ds(new) psi_L(old)) a[old]
// Ds = s+ - s- of the new pair state, K' = self factor x bare propagator pair (Eq. 8),
// Psi(mid) = sum_j psi_j(partner at lag j) the Eq. 9 exponent of the kept partners.  Rows with the
// same Ds share one moment S_d = sum_old beta_d(old) a[old] and one factor E_d = exp(delta_d Psi),
// a product of host-built tables (no transcendental in the kernel).
//
// Step fusion: step k only reads/writes slot p = k mod L, and its factors depend on the other
// slots only through their values.  Steps k..k+S-1 touch slots p..p+S-1 only, so for every fixed
// value of the other L-S ("outer") slots the N^S entries of the "super-fibre" evolve independently
// through all S steps.  One thread loads its super-fibre once, applies S steps in registers
// (reading rho of each step from the pre-step values) and stores it once: HBM traffic per step
// drops from 32 B to 32/S B per ARDM entry.
#include <cstdlib>

#include "qp_internal.h"

namespace qp {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cexp_(double2 z) {
    double e = exp(z.x), s, c;
    sincos(z.y, &s, &c);
    return make_double2(e * c, e * s);
}

__host__ __device__ constexpr int cpow(int b, int e) { return e == 0 ? 1 : b * cpow(b, e - 1); }

// Fixed-order block reduction of N complex accumulators into partials[blockIdx][N]; the last
// block to finish sums the partials over blocks in fixed order into rho[N] (deterministic:
// the grid and the tile->block assignment are fixed by the plan).
template <int N, int BLOCK>
__device__ __forceinline__ void reduce_finalize(double2 (&acc)[N], double2 *partials, double2 *rho,
                                                unsigned *counter, bool accumulate = false) {
    constexpr int W = BLOCK / 32;
    __shared__ double2 red[W][N];
    __shared__ double2 fin[W];
    __shared__ int is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();  // red/fin may be reused by consecutive calls
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
        double2 s = red[0][threadIdx.x];
        for (int w = 1; w < W; ++w) s = cadd(s, red[w][threadIdx.x]);
        __stcg(&partials[(size_t)blockIdx.x * N + threadIdx.x], s);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (int n = 0; n < N; ++n) {
        double2 s = make_double2(0.0, 0.0);
        for (int b = threadIdx.x; b < (int)gridDim.x; b += BLOCK) s = cadd(s, __ldcg(&partials[(size_t)b * N + n]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
        }
        if (lane == 0) fin[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double2 t = fin[0];
            for (int w = 1; w < W; ++w) t = cadd(t, fin[w]);
            rho[n] = accumulate ? cadd(rho[n], t) : t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *counter = 0u;
}

// --------------------------------------------------------------------------------------------
// Fused slide kernel.  Persistent CTAs over a contiguous, static range of tiles.  Tile tau = TILE
// consecutive outer fibres (the v lowest outer slots vary inside a tile).  Thread (r, t) with
// r = threadIdx.x / TILE, t = threadIdx.x % TILE works on outer fibre t; during sub-step s it holds
// the N entries of the fibre along inner digit s whose other inner digits are the digits of r.
// A warp therefore covers 32 consecutive outer fibres with ONE inner combination r: every table
// index (inner factors, 'last', K' row) is warp-uniform and the 32 lanes read 32 consecutive
// ARDM entries per load.  Between sub-steps the CTA re-distributes entries through shared memory.
// Inner digit i (i < S) is slot (p0 + i) mod L with address stride pw_in[i]; entry e = sum_i d_i N^i
// of outer fibre t lives at tile_base + lofs[t].x + sum_i d_i pw_in[i].
// --------------------------------------------------------------------------------------------
template <int N, int S>
__device__ __forceinline__ int fib_elem(int s, int r, int v) {  // entry of fibre r along digit s, value v
    int e = 0, rr = r, pw = 1;
#pragma unroll
    for (int i = 0; i < S; ++i) {
        int d;
        if (i == s) d = v;
        else { d = rr % N; rr /= N; }
        e += d * pw;
        pw *= N;
    }
    return e;
}
template <int N, int S>
__device__ __forceinline__ int fib_digit(int s, int r, int i) {  // digit i (i != s) of fibre r along s
    int rr = r;
#pragma unroll
    for (int q = 0; q < S; ++q) {
        if (q == s) continue;
        if (q == i) return rr % N;
        rr /= N;
    }
    return 0;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int TILE, int MINB, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused(const __grid_constant__ FusedArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    constexpr int Q = cpow(N, S - 1);    // inner combinations per sub-step (= fibres per super-fibre)
    constexpr int NK = RO ? 2 : 1;
    static_assert(S == 1 || TILE * Q == BLOCK, "fused kernel: one thread per (outer fibre, inner combination)");
    static_assert(S == 1 || TILE % 32 == 0, "fused kernel: warp-uniform inner combination");
    static_assert(!SYM || (M == 2 && D == 2), "symmetric moments are the M = 2 s = (+s,-s) case");
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];           // K'(new, last): [0] propagate, [1] terminal
    __shared__ double2 sIn[S][S][2][D][N];    // inner-slot factors exp(delta_d psi_lag(sigma))
    __shared__ double2 xch[S > 1 ? cpow(N, S) * TILE : 1];  // [entry][outer fibre] exchange buffer
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < S * S * 2 * D * N; i += BLOCK) (&sIn[0][0][0][0][0])[i] = a.inner[i];
    __shared__ double2 sBeta[S][2][D][N];  // beta_d(old) of each sub-step (first slide: initial-edge classes)
    for (int i = threadIdx.x; i < S * 2 * D * N; i += BLOCK) {
        const int s_ = i / (2 * D * N), kap = (i / (D * N)) % 2, r_ = i % (D * N);
        (&sBeta[0][0][0][0])[i] = a.small[lay.beta(a.var[s_], kap) + r_];
    }

    const int r = threadIdx.x / TILE, t = threadIdx.x % TILE;
    const bool valid = t < a.T && r < Q;
    const int2 lo = valid ? a.lofs[t] : make_int2(0, 0);
    long long off_ld = lo.x, off_st = lo.x;  // this thread's fibre along digit 0 (load) / S-1 (store)
#pragma unroll
    for (int i = 1; i < S; ++i) off_ld += (long long)fib_digit<N, S>(0, r, i) * a.pw_in[i];
#pragma unroll
    for (int i = 0; i < S - 1; ++i) off_st += (long long)fib_digit<N, S>(S - 1, r, i) * a.pw_in[i];
    double2 accR[RO ? S : 1][RO ? N : 1];
#pragma unroll
    for (int s = 0; s < (RO ? S : 1); ++s)
#pragma unroll
        for (int n = 0; n < (RO ? N : 1); ++n) accR[s][n] = make_double2(0.0, 0.0);

    // contiguous, static tile range per CTA (deterministic readout order)
    const int per = a.n_tiles / (int)gridDim.x, rem = a.n_tiles % (int)gridDim.x;
    const int t_begin = (int)blockIdx.x * per + min((int)blockIdx.x, rem);
    const int t_end = t_begin + per + ((int)blockIdx.x < rem ? 1 : 0);
    // Tile-uniform data.  Tile-independent part, once per kernel:
    //   KI[s][kap][r][new][last] = K'_kap(new, last) * prod_{i != s} inner_i(class(new), digit_i(r))
    // Per tile (pipelined through rings, one barrier per tile):
    //   stage A (tile i+2): Ehi[s][kap][d] = product of the outer digit-group tables g >= 1, base, last
    //   stage B (tile i+1): KU[s][kap][r][new][last] = KI * Ehi[s][kap][class(new)]
    // so KU holds every factor of output row `new` except the per-fibre outer group 0.
    constexpr int NKU = S * NK * Q * N * N;
    // (for S = 1 there is no inner slot: KI would equal K', so it is not stored)
    __shared__ double2 KI[S > 1 ? S : 1][S > 1 ? NK : 1][S > 1 ? Q : 1][S > 1 ? N : 1][S > 1 ? N : 1];
    __shared__ double2 KU[3][S][NK][Q][N][N];
    __shared__ double2 sEhi[4][S][NK][D];
    __shared__ long long sBase[4];
    __shared__ int sLast[4];
    __syncthreads();  // sK, sIn loaded
    for (int j = threadIdx.x; j < NKU; j += BLOCK) {
        const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                  s = j / (N * N * Q * NK);
        const int c = class_of(M, LAT, nw / M, nw % M);
        double2 e = sK[kap][nw][last];
        if (c > 0)
            for (int i = 0; i < S; ++i)
                if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
        if constexpr (S > 1) KI[S > 1 ? s : 0][S > 1 ? kap : 0][S > 1 ? rr : 0][S > 1 ? nw : 0][S > 1 ? last : 0] = e;
    }
    auto stage_a = [&](int tau, int slot) {
        if ((int)threadIdx.x < S * NK * D) {
            const int s = threadIdx.x / (NK * D), kap = (threadIdx.x / D) % NK, d = threadIdx.x % D;
            double2 e = make_double2(1.0, 0.0);
            for (int g = 1; g < a.G; ++g)
                e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
            sEhi[slot][s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
        }
        if ((int)threadIdx.x == BLOCK - 1) {
            long long b = 0;
            for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
            sBase[slot] = b;
            sLast[slot] = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
        }
    };
    auto stage_b = [&](int aslot, int kslot) {
        for (int j = threadIdx.x; j < NKU; j += BLOCK) {
            const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                      s = j / (N * N * Q * NK);
            const int c = class_of(M, LAT, nw / M, nw % M);
            double2 e;
            if constexpr (S > 1) e = KI[S > 1 ? s : 0][S > 1 ? kap : 0][S > 1 ? rr : 0][S > 1 ? nw : 0][S > 1 ? last : 0];
            else e = sK[kap][nw][last];
            KU[kslot][s][kap][rr][nw][last] = c > 0 ? cmul(e, sEhi[aslot][s][kap][c - 1]) : e;
        }
    };
    if (t_begin < t_end) stage_a(t_begin, 0);
    if (t_begin + 1 < t_end) stage_a(t_begin + 1, 1);
    __syncthreads();
    if (t_begin < t_end) stage_b(0, 0);
    __syncthreads();
    // register prefetch: the loads of tile i+1 are in flight while tile i is computed
    double2 xn[N];
    if (valid && t_begin < t_end) {
#pragma unroll
        for (int v = 0; v < N; ++v) xn[v] = __ldcs(a.A + sBase[0] + off_ld + v * a.pw_in[0]);
    }
    for (int tau = t_begin, it = 0; tau < t_end; ++tau, ++it) {
        const int buf = it % 3, abuf = it % 4;
        double2 xf[N];
#pragma unroll
        for (int v = 0; v < N; ++v) xf[v] = xn[v];
        if (tau + 1 < t_end) stage_b((it + 1) % 4, (it + 1) % 3);
        if (tau + 2 < t_end) stage_a(tau + 2, (it + 2) % 4);
        __syncthreads();
        if (valid && tau + 1 < t_end) {
#pragma unroll
            for (int v = 0; v < N; ++v) xn[v] = __ldcs(a.A + sBase[(it + 1) % 4] + off_ld + v * a.pw_in[0]);
        }
        const long long base = sBase[abuf];
        const int last0 = lo.y >= 0 ? lo.y : sLast[abuf];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s > 0) {  // re-distribute the super-fibres: fibres along digit s-1 -> along digit s
                if (valid) {
#pragma unroll
                    for (int v = 0; v < N; ++v) xch[fib_elem<N, S>(s - 1, r, v) * TILE + t] = xf[v];
                }
                __syncthreads();
                if (valid) {
#pragma unroll
                    for (int v = 0; v < N; ++v) xf[v] = xch[fib_elem<N, S>(s, r, v) * TILE + t];
                }
                __syncthreads();
            }
            if (!valid) continue;
            const bool ro = RO && a.rho[s] != nullptr;
            const int last = s == 0 ? last0 : fib_digit<N, S>(s, r, s - 1);  // warp-uniform for s > 0
            const double2(&ku)[NK][Q][N][N] = KU[buf][s];
            // per-fibre outer group-0 factor of class d, kind kap
            auto e0 = [&](int kap, int d) { return __ldg(&a.Etab[(((size_t)s * 2 + kap) * a.G * D + d) * a.X + t]); };
            // moments m_d = sum_old beta_d(old) x(old) for both kinds, S0 = sum_old x(old)
            double2 S0, m[NK][D];
            if constexpr (SYM) {
                // M = 2 with s = (+s, -s): beta_1 = (c, rho, 1/rho, conj c), beta_2 = 1/beta_1, so with
                // u = x00 + x11, w = x00 - x11, p = x01 + x10, q = x01 - x10:
                //   m_{1,2} = [Re c u + ch p] +- [i Im c w + sh q],  ch/sh = (rho +- 1/rho)/2
                const double2 u = cadd(xf[0], xf[3]), w = make_double2(xf[0].x - xf[3].x, xf[0].y - xf[3].y);
                const double2 p = cadd(xf[1], xf[2]), q = make_double2(xf[1].x - xf[2].x, xf[1].y - xf[2].y);
                S0 = cadd(u, p);
#pragma unroll
                for (int kap = 0; kap < NK; ++kap) {
                    if (kap == 1 && !ro) break;
                    const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2], sh = a.sym[s][kap][3];
                    const double2 A = make_double2(fma(cr, u.x, ch * p.x), fma(cr, u.y, ch * p.y));
                    const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                    m[kap][0] = cadd(A, Bv);
                    m[kap][D - 1] = make_double2(A.x - Bv.x, A.y - Bv.y);
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
            if (ro) {  // rho(t_{k+s}) from the pre-step values, off-diagonal rows (terminal classes)
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const double2 pt = cmul(e0(NK - 1, d), m[NK - 1][d]);
#pragma unroll
                    for (int aa = 0; aa < M; ++aa)
#pragma unroll
                        for (int bb = 0; bb < M; ++bb)
                            if (class_of(M, LAT, aa, bb) == d + 1)
                                accR[RO ? s : 0][RO ? aa * M + bb : 0] =
                                    cfma(ku[NK - 1][r][aa * M + bb][last], pt, accR[RO ? s : 0][RO ? aa * M + bb : 0]);
                }
            }
            double2 P[D];
#pragma unroll
            for (int d = 0; d < D; ++d) P[d] = cmul(e0(0, d), m[0][d]);
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    const int nw = aa * M + bb;
                    const int c = class_of(M, LAT, aa, bb);
                    xf[nw] = cmul(ku[0][r][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                    if (ro && c == 0)  // diagonal rows of rho: the propagated value itself
                        accR[RO ? s : 0][RO ? nw : 0] = cadd(accR[RO ? s : 0][RO ? nw : 0], xf[nw]);
                }
        }
        if (valid) {
#pragma unroll
            for (int v = 0; v < N; ++v) __stcs(a.A + base + off_st + v * a.pw_in[S - 1], xf[v]);
        }
    }
    if constexpr (RO) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr)
                reduce_finalize<N, BLOCK>(accR[RO ? s : 0], a.partials + (size_t)s * kPartialsMax * N, a.rho[s],
                                          a.counter + s, a.rho_accumulate != 0);
    }
}

// --------------------------------------------------------------------------------------------
// Register variant of the fused slide kernel: one thread per outer fibre holds its whole
// super-fibre (N^S entries) in registers, so the S sub-steps need no exchange; 16 independent
// 16-byte loads per thread (M = 2, S = 2) keep HBM busy.  Warps are independent: each warp owns
// a contiguous, static range of tiles (T = N^v outer fibres), builds the tile's factor table KU
// in its own shared-memory slice (warp-synchronous, no CTA barrier in the main loop) and sweeps
// the tile in chunks of 32 outer fibres, lane = outer fibre.  Readout accumulators live in
// shared memory; the CTA reduction at the end is in fixed order (deterministic).
// --------------------------------------------------------------------------------------------
#ifndef QP_L2_AHEAD
#define QP_L2_AHEAD 0
#endif
constexpr long long kL2Ahead = QP_L2_AHEAD;  // units of L2 prefetch distance in k_fused_r

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory");
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool ASYNC, bool RO>
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
    // dynamic shared memory: readout accumulators [S][N][BLOCK] (RO only), then (ASYNC only) a
    // per-warp double buffer [2][NS][32] of super-fibres staged by cp.async one chunk ahead
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
    double2(*stg)[NS][32] = reinterpret_cast<double2(*)[NS][32]>(
        dyn_smem + (RO ? S * N * BLOCK : 0) + (ASYNC ? (size_t)warp * 2 * NS * 32 : 0));
    auto issue = [&](long long u, int b) {  // stage unit u's super-fibres (this lane's) into buffer b
        const int tau = (int)(u / CH), t = (int)(u % CH) * 32 + lane;
        if (t < a.T) {
            long long base = __ldg(&a.lofs[t]).x;
            for (int g = 1; g < a.G; ++g) base += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
#pragma unroll
            for (int e = 0; e < NS; ++e) {
                long long o = base;
#pragma unroll
                for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
                cp_async16(&stg[b][e][lane], a.A + o);
            }
        }
        cp_async_commit();
    };
    if (ASYNC && u_begin < u_end) issue(u_begin, 0);
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
        if (ASYNC) {
            if (u + 1 < u_end) issue(u + 1, (int)((u + 1 - u_begin) & 1));
            else cp_async_commit();
            cp_async_wait<1>();  // this lane's copies of unit u have landed
        } else if (kL2Ahead > 0 && u + kL2Ahead < u_end) {
            // pull unit u+kL2Ahead into L2 (no registers held): its loads later hit L2 instead of HBM
            const long long un = u + kL2Ahead;
            const int taun = (int)(un / CH), tn = (int)(un % CH) * 32 + lane;
            if (tn < a.T) {
                long long base = __ldg(&a.lofs[tn]).x;
                for (int g = 1; g < a.G; ++g) base += __ldg(&a.goff[(size_t)g * a.X + (taun / a.gdiv[g]) % a.gmod[g]]);
#pragma unroll
                for (int e = 0; e < NS; ++e) {
                    long long o = base;
#pragma unroll
                    for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(a.A + o));
                }
            }
        }
        {
            if (t >= a.T) continue;
            const int2 lo = __ldg(&a.lofs[t]);
            const long long base = tbase + lo.x;
            double2 x[NS];
            if (ASYNC) {
                const int b = (int)((u - u_begin) & 1);
#pragma unroll
                for (int e = 0; e < NS; ++e) x[e] = stg[b][e][lane];
            } else {
#pragma unroll
                for (int e = 0; e < NS; ++e) {
                    long long o = base;
#pragma unroll
                    for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
                    x[e] = __ldcs(a.A + o);
                }
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
                        const double2 u = cadd(xf[0], xf[3]), w = make_double2(xf[0].x - xf[3].x, xf[0].y - xf[3].y);
                        const double2 p = cadd(xf[1], xf[2]), q = make_double2(xf[1].x - xf[2].x, xf[1].y - xf[2].y);
                        S0 = cadd(u, p);
#pragma unroll
                        for (int kap = 0; kap < NK; ++kap) {
                            if (kap == 1 && !ro) break;
                            const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2],
                                         sh = a.sym[s][kap][3];
                            const double2 A = make_double2(fma(cr, u.x, ch * p.x), fma(cr, u.y, ch * p.y));
                            const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                            m[kap][0] = cadd(A, Bv);
                            m[kap][D - 1] = make_double2(A.x - Bv.x, A.y - Bv.y);
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
    }
    if (ASYNC) cp_async_wait<0>();
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

// --------------------------------------------------------------------------------------------
// Split-register variant (S = 2, even N): two lanes share one super-fibre, each holding half of it
// (N^2/2 entries: inner digit 1 in its half {p N/2 .. p N/2 + N/2 - 1}).  Sub-step 0 (fibres along
// digit 0) is complete in each lane; the halves are then swapped across the lane pair with warp
// shuffles (lane ^ 16) so that sub-step 1 (fibres along digit 1) is complete too, and each lane
// stores its new half directly.  Half the registers of k_fused_r per lane -> twice the warps per SM
// for the same bytes in flight.  Lane l: outer fibre (l & 15) of the chunk, part p = l >> 4.
// --------------------------------------------------------------------------------------------
template <int M, bool LAT, bool SYM, int BLOCK, int MINB, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused_p2(const __grid_constant__ FusedArgs a) {
    constexpr int N = M * M;
    constexpr int S = 2;
    constexpr int H = N / 2;             // digit-1 values per part
    constexpr int D = n_classes(M, LAT);
    constexpr int Q = N;                 // fibres per super-fibre and sub-step
    constexpr int NK = RO ? 2 : 1;
    constexpr int W = BLOCK / 32;
    static_assert(N % 2 == 0, "split variant needs even N");
    static_assert(!SYM || (M == 2 && D == 2), "symmetric moments are the M = 2 s = (+s,-s) case");
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    extern __shared__ double2 dyn_smem[];  // readout accumulators [S][N][BLOCK] (RO only)
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
    const int part = lane >> 4, sub = lane & 15;
    const int CH = (a.T + 15) >> 4;
    const long long n_units = (long long)a.n_tiles * CH;
    const int gw = (int)blockIdx.x * W + warp, nw_tot = (int)gridDim.x * W;
    const long long per = n_units / nw_tot, rem = n_units % nw_tot;
    const long long u_begin = gw * per + min((long long)gw, rem);
    const long long u_end = u_begin + per + (gw < rem ? 1 : 0);
    constexpr int NKU = S * NK * Q * N * N;
    __shared__ double2 KI[S][NK][Q][N][N];
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
        const int tau = (int)(u / CH), t = (int)(u % CH) * 16 + sub;
        if (tau != cur_tile) {  // warp-synchronous tile setup
            __syncwarp();
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
        const bool valid = t < a.T;
        const int2 lo = valid ? __ldg(&a.lofs[t]) : make_int2(0, 0);
        const long long base = tbase + lo.x;
        // X[i][v]: digit 1 = part*H + i, digit 0 = v
        double2 X[H][N];
        if (valid) {
#pragma unroll
            for (int i = 0; i < H; ++i)
#pragma unroll
                for (int v = 0; v < N; ++v) X[i][v] = __ldcs(a.A + base + (long long)v * a.pw_in[0] + (long long)(part * H + i) * a.pw_in[1]);
        }
        const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == 1) {
                // swap halves across the lane pair: keep digit 0 in {part*H + jj}, all digit-1 values.
                // Send X[i][(1-part)*H + jj] (the partner's digit-0 half), receive the partner's X[i][part*H + jj].
                double2 Y[N][H];  // Y[d1][jj], d0 = part*H + jj
#pragma unroll
                for (int i = 0; i < H; ++i)
#pragma unroll
                    for (int jj = 0; jj < H; ++jj) {
                        const double2 keep = part == 0 ? X[i][jj] : X[i][H + jj];
                        const double2 give = part == 0 ? X[i][H + jj] : X[i][jj];
                        double2 got;
                        got.x = __shfl_xor_sync(0xffffffffu, give.x, 16);
                        got.y = __shfl_xor_sync(0xffffffffu, give.y, 16);
                        // own digit-1 values are part*H + i, the partner's (1-part)*H + i
                        if (part == 0) { Y[i][jj] = keep; Y[H + i][jj] = got; }
                        else { Y[H + i][jj] = keep; Y[i][jj] = got; }
                    }
#pragma unroll
                for (int i = 0; i < H; ++i)
#pragma unroll
                    for (int v = 0; v < N; ++v) X[i][v] = make_double2(0.0, 0.0);
                // re-use X as [jj][d1] storage: X_(jj)[d1]
#pragma unroll
                for (int jj = 0; jj < H; ++jj)
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) X[jj][d1] = Y[d1][jj];
            }
            if (!valid) continue;
            const bool ro = RO && a.rho[s] != nullptr;
            double2 E0[NK][D];
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    E0[kap][d] = (kap == 0 || ro) ? __ldg(&a.Etab[(((size_t)s * 2 + kap) * a.G * D + d) * a.X + t])
                                                  : make_double2(0.0, 0.0);
            double2 acc[RO ? N : 1];
#pragma unroll
            for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
            const double2(&ku)[NK][Q][N][N] = ku_w[s];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                double2(&xf)[N] = X[i];
                // fibre index r = value of the other inner digit; 'last' = digit 0 for sub-step 1
                const int r = part * H + i;
                const int last = s == 0 ? last0 : r;
                double2 S0, m[NK][D];
                if constexpr (SYM) {
                    const double2 uu = cadd(xf[0], xf[3]), w = make_double2(xf[0].x - xf[3].x, xf[0].y - xf[3].y);
                    const double2 p = cadd(xf[1], xf[2]), q = make_double2(xf[1].x - xf[2].x, xf[1].y - xf[2].y);
                    S0 = cadd(uu, p);
#pragma unroll
                    for (int kap = 0; kap < NK; ++kap) {
                        if (kap == 1 && !ro) break;
                        const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2], sh = a.sym[s][kap][3];
                        const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                        const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                        m[kap][0] = cadd(A, Bv);
                        m[kap][D - 1] = make_double2(A.x - Bv.x, A.y - Bv.y);
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
                                    acc[RO ? aa * M + bb : 0] = cfma(ku[NK - 1][r][aa * M + bb][last], pt, acc[RO ? aa * M + bb : 0]);
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
                        xf[nw] = o;
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
        if (valid) {  // X[jj][d1]: digit 0 = part*H + jj
#pragma unroll
            for (int jj = 0; jj < H; ++jj)
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
                    __stcs(a.A + base + (long long)(part * H + jj) * a.pw_in[0] + (long long)d1 * a.pw_in[1], X[jj][d1]);
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

// --------------------------------------------------------------------------------------------
// Three fused steps per HBM pass (M = 2, S = 3): the 64-entry super-fibre of an outer fibre is
// held by 4 lanes of a warp (part j = lane >> 3 holds inner digit 2 = j: 16 entries), so sub-steps
// 0 and 1 (fibres along digits 0 and 1) are lane-local; before sub-step 2 the four lanes transpose
// digit 0 <-> digit 2 through a per-warp shared-memory buffer (two halves of 4 KB) and then hold
// the fibres along digit 2.  Lane l works on outer fibre (l & 7) of the warp's 8; a CTA sweeps a
// tile of T outer fibres in rounds of 8 * W.  Factor tables KU are CTA-wide per tile.
// HBM traffic per step: 32/3 B per ARDM entry.
// --------------------------------------------------------------------------------------------

// KU row swizzle: the 16 entries (new, last) of KU row r are stored at (4 new + last) ^ f(r).  The
// lanes of a warp read rows r = d + 4j (sub-steps 0, 1) or j + 4d (sub-step 2) for their digit-2
// value j; rows are 256 B apart (same banks), so without the swizzle the 4 rows conflict 4-way.
// f(r) = g(r / 4) ^ g(r % 4), g(x) = 4 (x & 1) + x / 2: distinct 16-B bank groups for the 4 rows,
// and at most 2-way for sub-step 0 whose 'last' also varies across lanes.
__device__ __forceinline__ int f3_swizzle(int r) {
    const int hi = r >> 2, lo = r & 3;
    return (((hi & 1) << 2) | (hi >> 1)) ^ (((lo & 1) << 2) | (lo >> 1));
}

// TMA (cp.async.bulk.tensor) + mbarrier helpers for k_fused3's staged loads
__device__ __forceinline__ unsigned smem_addr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar)) : "memory");
}
// 32-byte (256-bit) streaming load / store of two adjacent complex entries (p must be 32-B aligned)
__device__ __forceinline__ void ld2_cs(const double2 *p, double2 &x, double2 &y) {
    asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(x.x), "=d"(x.y), "=d"(y.x), "=d"(y.y) : "l"(p));
}
__device__ __forceinline__ void st2_cs(double2 *p, double2 x, double2 y) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(x.x), "d"(x.y), "d"(y.x), "d"(y.y) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}\n" ::"r"(smem_addr(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const void *tmap, unsigned long long *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %4, %4}], [%5];"
        ::"r"(smem_addr(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(0), "r"(smem_addr(bar)) : "memory");
}

// PFM (next-round prefetch): 0 none, 1 registers, 2 TMA box into a shared-memory stage (lane map 1,
// unsharded layouts: FusedArgs::tmap, dims (run A, run B, d0, d1, d2), see host.cpp)
// VW: the TMA stage view (FusedArgs::tma_swz) fixed at compile time (-1: read a.tma_swz at run time);
// one view per instantiation keeps the other views' stage-read code out of the register allocation.
template <bool SYM, int MAP, int BLOCK, int MINB, int PFM, bool RO, int VW = -1>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused3(const __grid_constant__ FusedArgs a) {
    constexpr int M = 2, N = 4, S = 3, Q = 16, D = 2;
    // PFM 5 (TW): TMA staging per warp -- each warp's 8 fibres of a round are its own box on its own
    // mbarrier, refilled by the warp as soon as its lanes have read it (no CTA barrier per round)
    constexpr bool PF = PFM == 1, TW = PFM == 5, TM = PFM == 2 || TW, CA = PFM == 3, STG = TM || CA;
    constexpr int F = 8 * (BLOCK / 32);  // outer fibres per round
    constexpr int FS = TW ? 8 : F;       // fibres per TMA box / stage read pattern
    constexpr int NK = RO ? 2 : 1;
    constexpr int W = BLOCK / 32;
    constexpr bool LAT = false;
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    __shared__ double2 KU[S][NK][Q][N][N];
    __shared__ double2 sEhi[S][NK][D];
    __shared__ long long sBase;
    __shared__ int sLast;
    // dynamic: (TM) the round's TMA stage [d2][d1][d0][F], then the exchange buffer (W x 16 x 8
    // entries: a quarter of the super-fibre entries of the round's fibres), then the readout
    // accumulators [S][N][BLOCK] (RO only)
    extern __shared__ __align__(1024) double2 dyn_smem_raw[];
    double2 *stage = dyn_smem_raw;
    // TM / CA: per-round outer factors E0 [2 buffers][S][2][D][F] and tile-local offsets [2][F] (copied
    // with the round, double-buffered: read during the round while the next one lands)
    double2 *sE0 = dyn_smem_raw + (STG ? F * 64 : 0);
    int2 *sLo = reinterpret_cast<int2 *>(sE0 + (STG ? 2 * S * 2 * D * F : 0));
    double2 *dyn_smem = sE0 + (STG ? 2 * S * 2 * D * F + F : 0);
    __shared__ __align__(8) unsigned long long sFullW[TW ? BLOCK / 32 : 1];
    unsigned long long &sFull = sFullW[TW ? (threadIdx.x >> 5) : 0];
    auto accS = reinterpret_cast<double2(*)[RO ? N : 1][RO ? BLOCK : 1]>(dyn_smem + W * 16 * 8);
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
    static_assert(MAP == 0 || W % 4 == 0, "lane map 1: groups of 4 warps (one per digit-2 value)");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lane map 0: lane = (j, t8), 8 outer fibres per warp, the 4 quarters of a super-fibre in one warp
    // lane map 1: lane = one of 32 consecutive outer fibres, warp -> j (512 contiguous bytes per load
    //             when the lowest ARDM digit is an outer digit); quarters exchanged across 4 warps
    const int j = MAP == 0 ? lane >> 3 : warp & 3;
    const int fib = MAP == 0 ? warp * 8 + (lane & 7) : (warp >> 2) * 32 + lane;  // fibre within a round
    // map 0: [W][16][8] per warp; map 1: [16][8 W] (same size)
    auto xch_at = [&](int e) -> double2 & {
        return MAP == 0 ? dyn_smem[(warp * 16 + e) * 8 + (lane & 7)] : dyn_smem[e * 8 * W + fib];
    };
    const int per = a.n_tiles / (int)gridDim.x, rem = a.n_tiles % (int)gridDim.x;
    const int t_begin = (int)blockIdx.x * per + min((int)blockIdx.x, rem);
    const int t_end = t_begin + per + ((int)blockIdx.x < rem ? 1 : 0);
    constexpr int NKU = S * NK * Q * N * N;
    const int rounds = (a.T + 8 * W - 1) / (8 * W);

    // one fibre: xf holds the N old values; on return the N new values.  r = inner combination,
    // last = value of the previous time point's slot.  acc: readout of this sub-step.
    auto fibre = [&](double2 (&xf)[N], int s, int r, int last, bool ro, const double2 (&E0)[NK][D],
                     double2 (&acc)[RO ? N : 1]) {
        double2 S0, m[NK][D];
        if constexpr (SYM) {
            const double2 uu = cadd(xf[0], xf[3]), w = make_double2(xf[0].x - xf[3].x, xf[0].y - xf[3].y);
            const double2 p = cadd(xf[1], xf[2]), q = make_double2(xf[1].x - xf[2].x, xf[1].y - xf[2].y);
            S0 = cadd(uu, p);
#pragma unroll
            for (int kap = 0; kap < NK; ++kap) {
                if (kap == 1 && !ro) break;
                const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2], sh = a.sym[s][kap][3];
                const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                m[kap][0] = cadd(A, Bv);
                m[kap][1] = make_double2(A.x - Bv.x, A.y - Bv.y);
            }
        } else {
            S0 = cadd(cadd(xf[0], xf[1]), cadd(xf[2], xf[3]));
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
        const int sw = MAP == 0 ? f3_swizzle(r) : 0;
        const double2 *ku0 = &KU[s][0][r][0][0], *ku1 = &KU[s][NK - 1][r][0][0];
        if (ro) {  // off-diagonal readout without the outer factor E0 (applied once per step below)
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int nw = 0; nw < N; ++nw)
                    if (class_of(M, LAT, nw / M, nw % M) == d + 1)
                        acc[RO ? nw : 0] = cfma(ku1[(nw * N + last) ^ sw], m[NK - 1][d], acc[RO ? nw : 0]);
        }
        double2 P[D];
#pragma unroll
        for (int d = 0; d < D; ++d) P[d] = cmul(E0[0][d], m[0][d]);
#pragma unroll
        for (int nw = 0; nw < N; ++nw) {
            const int c = class_of(M, LAT, nw / M, nw % M);
            const double2 o = cmul(ku0[(nw * N + last) ^ sw], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
            xf[nw] = o;
            if (ro && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
        }
    };

    // tile base offset (outer digit groups >= 1) and one unit's loads: unit = (tile tau, round rd),
    // lane -> outer fibre t = rd 8W + 8 warp + t8 and digit-2 value j; X[d1][d0]
    auto tile_base = [&](int tau) {
        long long b = 0;
        for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
        return b;
    };
    auto load_unit = [&](int tau, int rd, double2 (&Y)[N][N], int2 &lo) {
        const int t = rd * 8 * W + fib;
        if (t < a.T) {
            lo = __ldg(&a.lofs[t]);
            const long long base = tile_base(tau) + lo.x + (long long)j * a.pw_in[2];
            if (a.pw_in[0] == 1) {  // d0 is ring slot 0: entry pairs (d0, d0 + 1) are adjacent, 32-B loads
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; d0 += 2) ld2_cs(a.A + base + d0 + (long long)d1 * a.pw_in[1], Y[d1][d0], Y[d1][d0 + 1]);
            } else if (a.pw_in[1] == 1) {  // d1 is slot 0: pairs (d1, d1 + 1)
#pragma unroll
                for (int d1 = 0; d1 < N; d1 += 2)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) ld2_cs(a.A + base + (long long)d0 * a.pw_in[0] + d1, Y[d1][d0], Y[d1 + 1][d0]);
            } else {
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0)
                        Y[d1][d0] = __ldcs(a.A + base + (long long)d0 * a.pw_in[0] + (long long)d1 * a.pw_in[1]);
            }
        } else {
            lo = make_int2(0, 0);
        }
    };
    double2 Xn[PF ? N : 1][PF ? N : 1];  // PF: the next unit's super-fibre quarter, in flight
    int2 lon = make_int2(0, 0);
    if constexpr (PF)
        if (t_begin < t_end) load_unit(t_begin, 0, Xn, lon);
    // TM: one stage; thread 0 issues the TMA box of unit (tau, rd): outer fibres G = tau T + rd F
    // E0r (TM): the round's factors and offsets are one contiguous block of E0B entries (one bulk copy);
    // the two buffers then are [2][E0B] over the same shared-memory region
    // TW: E0r blocks are per (round, warp) of FS = 8 fibres; warp w's two buffers at sE0 + 2 w E0B
    constexpr int E0B = S * 2 * D * FS + FS / 2;
    const bool e0r = TW || (STG && a.E0r != nullptr);
    const int sfib = TW ? (lane & 7) : fib;  // fibre index within the stage / E0 block
    double2 *const sE0w = TW ? sE0 + (size_t)warp * 2 * E0B : sE0;
    double2 *const stg = TW ? stage + (size_t)warp * FS * 64 : stage;
    auto e0_at = [&](int buf, int q) -> double2 {  // q = (s, kap, d)
        return e0r ? sE0w[buf * E0B + q * FS + sfib] : sE0[(buf * S * 2 * D + q) * F + fib];
    };
    auto lo_at = [&](int buf) -> int2 {
        return e0r ? reinterpret_cast<const int2 *>(sE0w + buf * E0B + S * 2 * D * FS)[sfib] : sLo[buf * F + fib];
    };
    auto tma_issue = [&](int tau, int rd, int buf) {
        const int rw = TW ? rd * (BLOCK / 32) + warp : rd;  // TW: the warp's 8-fibre unit of round rd
        const long long G = (long long)tau * a.T + (long long)rw * FS;
        fence_proxy_async();
        mbar_expect_tx(&sFull, FS * 64 * 16 + S * 2 * D * FS * 16 + FS * 8);
        tma_load_5d(stg, &a.tmap, &sFull, (int)(a.tma_c0m * (G % a.tma_nA)), (int)(a.tma_c1m * (G / a.tma_nA)));
        if (e0r) {
            bulk_g2s(sE0w + buf * E0B, a.E0r + (size_t)rw * E0B, E0B * 16, &sFull);
        } else if constexpr (!TW) {  // per-slice copies: q = (s, kap, d): Etab[s][kap][g = 0][d][t0 ..]
            for (int q = 0; q < S * 2 * D; ++q) {
                const int st = q / (2 * D), kap = (q / D) % 2, d = q % D;
                bulk_g2s(sE0 + ((size_t)buf * S * 2 * D + q) * F,
                         a.Etab + ((((size_t)st * 2 + kap) * a.G) * D + d) * a.X + rd * F, F * 16, &sFull);
            }
            bulk_g2s(sLo + buf * F, a.lofs + rd * F, F * 8, &sFull);
        }
    };
    // CA: every thread copies 16-B chunks of the round with cp.async: chunk q enumerates the round in
    // HBM order (fields sorted by stride: a.stg_lg[i] = log2 radix, a.stg_g[i] global stride, a.stg_s[i]
    // stage stride, field a.stg_fi = the fibre index), so consecutive lanes read consecutive 16 B; the
    // stage position is XOR-swizzled with the fibre's low 3 bits when a.stg_swz (bank-conflict-free reads)
    auto ca_issue = [&](int tau, int rd, int buf) {
        const long long rb = tile_base(tau) + __ldg(&a.lofs[rd * F]).x;
        for (int q = threadIdx.x; q < F * 64; q += BLOCK) {
            int r = q, sp = 0, fv = 0;
            long long go = rb;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int dg = r & ((1 << a.stg_lg[i]) - 1);
                r >>= a.stg_lg[i];
                go += (long long)dg * a.stg_g[i];
                sp += dg * a.stg_s[i];
                if (i == a.stg_fi) fv = dg;
            }
            if (a.stg_swz) sp ^= fv & 7;
            cp_async16(stage + sp, a.A + go);
        }
        for (int q = threadIdx.x; q < S * 2 * D * F; q += BLOCK) {
            const int qq = q / F, f = q % F, st = qq / (2 * D), kap = (qq / D) % 2, d = qq % D;
            cp_async16(sE0 + ((size_t)buf * S * 2 * D + qq) * F + f,
                       a.Etab + ((((size_t)st * 2 + kap) * a.G) * D + d) * a.X + rd * F + f);
        }
        for (int q = threadIdx.x; q < F / 2; q += BLOCK) cp_async16(sLo + buf * F + 2 * q, a.lofs + rd * F + 2 * q);
        cp_async_commit();
    };
    unsigned phase = 0, cur = 0;
    if constexpr (CA)
        if (t_begin < t_end) ca_issue(t_begin, 0, 0);
    if constexpr (TM) {
        if (TW ? lane == 0 : threadIdx.x == 0) {
            mbar_init(&sFull, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if ((TW ? lane == 0 : threadIdx.x == 0) && t_begin < t_end) tma_issue(t_begin, 0, 0);
    }

    for (int tau = t_begin; tau < t_end; ++tau) {
        __syncthreads();  // previous tile's KU no longer in use
        if ((int)threadIdx.x < S * NK * D) {
            const int s = threadIdx.x / (NK * D), kap = (threadIdx.x / D) % NK, d = threadIdx.x % D;
            double2 e = make_double2(1.0, 0.0);
            for (int g = 1; g < a.G; ++g)
                e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
            sEhi[s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
        }
        if ((int)threadIdx.x == BLOCK - 1) {
            long long b = 0;
            for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
            sBase = b;
            sLast = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
        }
        __syncthreads();
        for (int jj = threadIdx.x; jj < NKU; jj += BLOCK) {
            const int last = jj % N, nw = (jj / N) % N, rr = (jj / (N * N)) % Q, kap = (jj / (N * N * Q)) % NK,
                      s = jj / (N * N * Q * NK);
            const int c = class_of(M, LAT, nw / M, nw % M);
            double2 e = sK[kap][nw][last];
            if (c > 0) {
                e = cmul(e, sEhi[s][kap][c - 1]);
                for (int i = 0; i < S; ++i)
                    if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
            }
            (&KU[s][kap][rr][0][0])[(nw * N + last) ^ (MAP == 0 ? f3_swizzle(rr) : 0)] = e;
        }
        __syncthreads();
        const long long tbase = sBase;
        const int last_t = sLast;
        for (int rd = 0; rd < rounds; ++rd) {
            const int t = rd * 8 * W + fib;
            const bool valid = t < a.T;
            int2 lo;
            double2 X[N][N];  // X[d1][d0], d2 = j
            if constexpr (TM) {  // the stage holds this unit (issued one unit ago)
                mbar_wait(&sFull, phase);
                cur = phase;
                phase ^= 1;
                lo = lo_at(cur);
                const int swz = VW >= 0 ? VW : a.tma_swz;
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) {
                        if (swz == 1) {  // view B: row r of 8 entries (fibre parity, d2); chunk XOR (r & 7)
                            const int r = (d1 * N + d0) * (FS / 2) + (sfib >> 1);
                            X[d1][d0] = stg[r * 8 + ((((sfib & 1) << 2) | j) ^ (r & 7))];
                        } else if (swz == 4) {  // view D: 128-B row r = (d2, d1 / 2, f) of entries (d1 & 1, d0)
                            const int r = (j * 2 + (d1 >> 1)) * FS + sfib;
                            X[d1][d0] = stg[r * 8 + ((((d1 & 1) << 2) | d0) ^ (r & 7))];
                        } else if (swz == 3) {  // view D, 64-B rows: row r = (d2, d1, f) of the d0 entries
                            const int r = (j * N + d1) * FS + sfib;
                            X[d1][d0] = stg[r * 4 + (d0 ^ ((r >> 1) & 3))];
                        } else if (swz == 5) {  // view C: 128-B row r = (d0, d2 / 2, f) of entries (d2 & 1, d1)
                            const int r = (d0 * 2 + (j >> 1)) * FS + sfib;
                            X[d1][d0] = stg[r * 8 + ((((j & 1) << 2) | d1) ^ (r & 7))];
                        } else if (swz == 2) {  // view C, fibre-major rows: row r of 8 entries (d2 parity, d1)
                            const int r = d0 * 2 * FS + 2 * sfib + (j >> 1);
                            X[d1][d0] = stg[r * 8 + ((((j & 1) << 2) | d1) ^ (r & 7))];
                        } else {
                            X[d1][d0] = stg[sfib * a.tma_sf + d0 * a.tma_s[0] + d1 * a.tma_s[1] + j * a.tma_s[2]];
                        }
                    }
                const int rn = rd + 1 < rounds ? rd + 1 : 0, taun = rd + 1 < rounds ? tau : tau + 1;
                if constexpr (TW) {
                    __syncwarp();  // the warp's stage is free: refill it with the warp's next unit
                    if (lane == 0 && taun < t_end) tma_issue(taun, rn, phase);
                } else {
                    __syncthreads();  // stage free: refill it with the next unit
                    if (threadIdx.x == 0 && taun < t_end) tma_issue(taun, rn, phase);
                }
            } else if constexpr (CA) {  // the stage holds this unit (copied one unit ago)
                cp_async_wait<0>();
                __syncthreads();
                cur = phase;
                phase ^= 1;
                lo = sLo[cur * F + fib];
                const int sw = a.stg_swz ? (fib & 7) : 0;
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0)
                        X[d1][d0] = stage[(fib * a.tma_sf + d0 * a.tma_s[0] + d1 * a.tma_s[1] + j * a.tma_s[2]) ^ sw];
                __syncthreads();  // stage free: refill it with the next unit
                const int rn = rd + 1 < rounds ? rd + 1 : 0, taun = rd + 1 < rounds ? tau : tau + 1;
                if (taun < t_end) ca_issue(taun, rn, phase);
            } else if constexpr (PF) {  // this unit was loaded one unit ago; issue the next unit's loads now
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) X[d1][d0] = Xn[d1][d0];
                lo = lon;
                const int rn = rd + 1 < rounds ? rd + 1 : 0, taun = rd + 1 < rounds ? tau : tau + 1;
                if (taun < t_end) load_unit(taun, rn, Xn, lon);
            } else {
                load_unit(tau, rd, X, lo);
            }
            const long long base = tbase + lo.x;
            const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == 2) {  // transpose digit 0 <-> digit 2 among the 4 lanes of an outer fibre
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) {  // one digit-1 value at a time (16 entries)
                        if (valid) {
#pragma unroll
                            for (int d0 = 0; d0 < N; ++d0) xch_at(d0 + 4 * j) = X[d1][d0];
                        }
                        if constexpr (MAP == 0) __syncwarp(); else __syncthreads();
                        if (valid) {  // X[d1][d2] := (digit0 = j, digit1 = d1, digit2 = d2)
#pragma unroll
                            for (int d2 = 0; d2 < N; ++d2) X[d1][d2] = xch_at(j + 4 * d2);
                        }
                        if constexpr (MAP == 0) __syncwarp(); else __syncthreads();
                    }
                }
                if (!valid) continue;
                const bool ro = RO && a.rho[s] != nullptr;
                double2 E0[NK][D];  // outer group-0 factor (kap = 1, readout: loaded at the end of the step)
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    E0[0][d] = STG ? e0_at(cur, s * 2 * D + d) : __ldg(&a.Etab[((size_t)s * 2 * a.G * D + d) * a.X + t]);
                    E0[NK - 1][d] = E0[0][d];
                }
                double2 acc[RO ? N : 1];
#pragma unroll
                for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
                if (s == 0) {  // fibres along digit 0: X[d1][.], other digits (d1, d2 = j)
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) fibre(X[d1], 0, d1 + 4 * j, last0, ro, E0, acc);
                } else if (s == 1) {  // along digit 1: X[.][d0], other digits (d0, d2 = j); last = d0
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) {
                        double2 xf[N];
#pragma unroll
                        for (int v = 0; v < N; ++v) xf[v] = X[v][d0];
                        fibre(xf, 1, d0 + 4 * j, d0, ro, E0, acc);
#pragma unroll
                        for (int v = 0; v < N; ++v) X[v][d0] = xf[v];
                    }
                } else {  // along digit 2: X[d1][.], other digits (d0 = j, d1); last = d1
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) fibre(X[d1], 2, j + 4 * d1, d1, ro, E0, acc);
                }
                if (ro) {
                    // the outer factor E0 (fixed for this thread's outer fibre) of the off-diagonal
                    // readout rows, factored out of the sum over its four fibres
#pragma unroll
                    for (int n = 0; n < N; ++n) {
                        const int c = class_of(M, LAT, n / M, n % M);
                        if (c > 0)
                            acc[RO ? n : 0] =
                                cmul(STG ? e0_at(cur, s * 2 * D + D + (c > 0 ? c - 1 : 0))
                                        : __ldg(&a.Etab[(((size_t)s * 2 + 1) * a.G * D + (c > 0 ? c - 1 : 0)) * a.X + t]),
                                     acc[RO ? n : 0]);
                    }
#pragma unroll
                    for (int n = 0; n < N; ++n)
                        accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0] =
                            cadd(accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0], acc[RO ? n : 0]);
                }
            }
            if (valid) {  // X[d1][d2] with digit 0 = j
                const long long b0 = base + (long long)j * a.pw_in[0];
                // store path: which inner digit is ring slot 0 follows from the view when VW is fixed
                // (view B: d2 = slot 0; view C: d1 = slot 0; views A and D: neither)
                const bool st_d2 = VW >= 0 ? VW == 1 : a.pw_in[2] == 1;
                const bool st_d1 = VW >= 0 ? (VW == 2 || VW == 5) : a.pw_in[1] == 1;
                if (st_d2) {  // d2 is ring slot 0: 32-B stores of adjacent pairs
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                        for (int d2 = 0; d2 < N; d2 += 2) st2_cs(a.A + b0 + (long long)d1 * a.pw_in[1] + d2, X[d1][d2], X[d1][d2 + 1]);
                } else if (st_d1) {
#pragma unroll
                    for (int d1 = 0; d1 < N; d1 += 2)
#pragma unroll
                        for (int d2 = 0; d2 < N; ++d2) st2_cs(a.A + b0 + d1 + (long long)d2 * a.pw_in[2], X[d1][d2], X[d1 + 1][d2]);
                } else {
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                        for (int d2 = 0; d2 < N; ++d2)
                            __stcs(a.A + b0 + (long long)d1 * a.pw_in[1] + (long long)d2 * a.pw_in[2], X[d1][d2]);
                }
            }
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

// --------------------------------------------------------------------------------------------
// k_fused3s: shared-memory-resident rounds (TMA view A launch sets).  A round = F = 32 consecutive
// outer fibres x the 64 inner entries, staged by TMA into one of two buffers (the next round lands
// while this one is computed).  The three sub-steps run fibre by fibre on the staged round in place:
// lane = outer fibre, warp = inner combination (warp-uniform KU rows and 'last' for sub-steps 1, 2;
// stage reads/writes are 32 consecutive 16-B words), one CTA barrier between sub-steps; sub-step 2's
// outputs go straight to HBM (32 lanes = 512 contiguous bytes).  No super-fibre in registers and the
// readout accumulators stay in registers: 16 warps per SM instead of 8.
// Stage layout [d2][d1][d0][f] (the view-A box).
// --------------------------------------------------------------------------------------------
template <bool SYM, int BLOCK, bool RO>
__global__ void __launch_bounds__(BLOCK, 2) k_fused3s(const __grid_constant__ FusedArgs a) {
    constexpr int M = 2, N = 4, S = 3, Q = 16, D = 2, F = 32, W = BLOCK / 32, RPW = 16 / W;
    constexpr int NK = RO ? 2 : 1;
    constexpr bool LAT = false;
    static_assert(16 % W == 0, "inner combinations per warp");
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    __shared__ double2 KU[S][NK][Q][N][N];
    __shared__ double2 sEhi[S][NK][D];
    __shared__ double2 sBeta[S][2][D][N];
    __shared__ long long sBase;
    __shared__ int sLast;
    __shared__ __align__(8) unsigned long long sFull[2];
    extern __shared__ __align__(1024) double2 dyn_smem_raw[];
    double2 *const stage0 = dyn_smem_raw;                               // [2][64 F]
    double2 *const sE0 = dyn_smem_raw + 2 * 64 * F;                      // [2][S][2][D][F]
    int2 *const sLo = reinterpret_cast<int2 *>(sE0 + 2 * S * 2 * D * F);  // [2][F]
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < S * S * 2 * D * N; i += BLOCK) (&sIn[0][0][0][0][0])[i] = a.inner[i];
    for (int i = threadIdx.x; i < S * 2 * D * N; i += BLOCK) {
        const int s_ = i / (2 * D * N), kap = (i / (D * N)) % 2, r_ = i % (D * N);
        (&sBeta[0][0][0][0])[i] = a.small[lay.beta(a.var[s_], kap) + r_];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = a.n_tiles / (int)gridDim.x, rem = a.n_tiles % (int)gridDim.x;
    const int t_begin = (int)blockIdx.x * per + min((int)blockIdx.x, rem);
    const int t_end = t_begin + per + ((int)blockIdx.x < rem ? 1 : 0);
    const int rounds = a.T / F;
    constexpr int NKU = S * NK * Q * N * N;
    double2 accR[RO ? S : 1][RO ? N : 1];
#pragma unroll
    for (int s = 0; s < (RO ? S : 1); ++s)
#pragma unroll
        for (int n = 0; n < (RO ? N : 1); ++n) accR[s][n] = make_double2(0.0, 0.0);

    auto issue = [&](int tau, int rd, int b) {  // thread 0: TMA box + E0 / offsets of unit (tau, rd)
        const long long G = (long long)tau * a.T + (long long)rd * F;
        fence_proxy_async();
        mbar_expect_tx(&sFull[b], F * 64 * 16 + S * 2 * D * F * 16 + F * 8);
        tma_load_5d(stage0 + b * 64 * F, &a.tmap, &sFull[b], (int)(a.tma_c0m * (G % a.tma_nA)),
                    (int)(a.tma_c1m * (G / a.tma_nA)));
        for (int q = 0; q < S * 2 * D; ++q) {
            const int st = q / (2 * D), kap = (q / D) % 2, d = q % D;
            bulk_g2s(sE0 + ((size_t)b * S * 2 * D + q) * F, a.Etab + ((((size_t)st * 2 + kap) * a.G) * D + d) * a.X + rd * F,
                     F * 16, &sFull[b]);
        }
        bulk_g2s(sLo + b * F, a.lofs + rd * F, F * 8, &sFull[b]);
    };
    if (threadIdx.x == 0) {
        mbar_init(&sFull[0], 1);
        mbar_init(&sFull[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && t_begin < t_end) {
        issue(t_begin, 0, 0);
        if (rounds > 1) issue(t_begin, 1, 1);
        else if (t_begin + 1 < t_end) issue(t_begin + 1, 0, 1);
    }
    unsigned u = 0;  // unit counter of this CTA
    for (int tau = t_begin; tau < t_end; ++tau) {
        __syncthreads();  // previous tile's KU no longer in use
        if ((int)threadIdx.x < S * NK * D) {
            const int s = threadIdx.x / (NK * D), kap = (threadIdx.x / D) % NK, d = threadIdx.x % D;
            double2 e = make_double2(1.0, 0.0);
            for (int g = 1; g < a.G; ++g)
                e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
            sEhi[s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
        }
        if ((int)threadIdx.x == BLOCK - 1) {
            long long b = 0;
            for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
            sBase = b;
            sLast = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
        }
        __syncthreads();
        for (int jj = threadIdx.x; jj < NKU; jj += BLOCK) {
            const int last = jj % N, nw = (jj / N) % N, rr = (jj / (N * N)) % Q, kap = (jj / (N * N * Q)) % NK,
                      s = jj / (N * N * Q * NK);
            const int c = class_of(M, LAT, nw / M, nw % M);
            double2 e = sK[kap][nw][last];
            if (c > 0) {
                e = cmul(e, sEhi[s][kap][c - 1]);
                for (int i = 0; i < S; ++i)
                    if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
            }
            KU[s][kap][rr][nw][last] = e;
        }
        __syncthreads();
        const long long tbase = sBase;
        const int last_t = sLast;
        for (int rd = 0; rd < rounds; ++rd, ++u) {
            const int b = u & 1;
            mbar_wait(&sFull[b], (u >> 1) & 1);
            double2 *const st = stage0 + b * 64 * F;
            const int2 lo = sLo[b * F + lane];
            const long long gbase = tbase + lo.x;
            const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool ro = RO && a.rho[s] != nullptr;
                double2 E00[D];
#pragma unroll
                for (int d = 0; d < D; ++d) E00[d] = sE0[((b * S + s) * 2 * D + d) * F + lane];
                double2 acc[RO ? N : 1];
#pragma unroll
                for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < RPW; ++i) {
                    const int rr = warp + W * i, lo2 = rr & 3, hi2 = rr >> 2;
                    // entry v of this fibre: stage word e0 + v * ev; KU row r; previous point 'last'
                    int e0, ev, r, last;
                    if (s == 0) e0 = (hi2 * 16 + lo2 * 4) * F, ev = F, r = lo2 + 4 * hi2, last = last0;
                    else if (s == 1) e0 = (hi2 * 16 + lo2) * F, ev = 4 * F, r = lo2 + 4 * hi2, last = lo2;
                    else e0 = (hi2 * 4 + lo2) * F, ev = 16 * F, r = lo2 + 4 * hi2, last = hi2;
                    double2 xf[N];
#pragma unroll
                    for (int v = 0; v < N; ++v) xf[v] = st[e0 + v * ev + lane];
                    double2 S0, m[NK][D];
                    if constexpr (SYM) {
                        const double2 uu = cadd(xf[0], xf[3]), w = make_double2(xf[0].x - xf[3].x, xf[0].y - xf[3].y);
                        const double2 p = cadd(xf[1], xf[2]), q = make_double2(xf[1].x - xf[2].x, xf[1].y - xf[2].y);
                        S0 = cadd(uu, p);
#pragma unroll
                        for (int kap = 0; kap < NK; ++kap) {
                            if (kap == 1 && !ro) break;
                            const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2],
                                         sh = a.sym[s][kap][3];
                            const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                            const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                            m[kap][0] = cadd(A, Bv);
                            m[kap][1] = make_double2(A.x - Bv.x, A.y - Bv.y);
                        }
                    } else {
                        S0 = cadd(cadd(xf[0], xf[1]), cadd(xf[2], xf[3]));
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
                    const double2 *ku0 = &KU[s][0][r][0][0], *ku1 = &KU[s][NK - 1][r][0][0];
                    if (ro) {
#pragma unroll
                        for (int d = 0; d < D; ++d)
#pragma unroll
                            for (int nw = 0; nw < N; ++nw)
                                if (class_of(M, LAT, nw / M, nw % M) == d + 1)
                                    acc[RO ? nw : 0] = cfma(ku1[nw * N + last], m[NK - 1][d], acc[RO ? nw : 0]);
                    }
                    double2 P[D];
#pragma unroll
                    for (int d = 0; d < D; ++d) P[d] = cmul(E00[d], m[0][d]);
#pragma unroll
                    for (int nw = 0; nw < N; ++nw) {
                        const int c = class_of(M, LAT, nw / M, nw % M);
                        const double2 o = cmul(ku0[nw * N + last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                        if (ro && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
                        if (s < 2) st[e0 + nw * ev + lane] = o;
                        else __stcs(a.A + gbase + (long long)lo2 * a.pw_in[0] + (long long)hi2 * a.pw_in[1] +
                                        (long long)nw * a.pw_in[2], o);
                    }
                }
                if (ro) {
#pragma unroll
                    for (int n = 0; n < N; ++n) {
                        const int c = class_of(M, LAT, n / M, n % M);
                        if (c > 0)
                            acc[RO ? n : 0] = cmul(sE0[((b * S + s) * 2 * D + D + (c > 0 ? c - 1 : 0)) * F + lane], acc[RO ? n : 0]);
                        accR[RO ? s : 0][RO ? n : 0] = cadd(accR[RO ? s : 0][RO ? n : 0], acc[RO ? n : 0]);
                    }
                }
                __syncthreads();  // sub-step s complete on the whole round (after s = 2: stage b free)
            }
            if (threadIdx.x == 0) {  // refill buffer b with unit u + 2
                int tn = tau, rn = rd + 2;
                while (rn >= rounds && tn < t_end) rn -= rounds, ++tn;
                if (tn < t_end) issue(tn, rn, b);
            }
        }
    }
    if constexpr (RO) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr)
                reduce_finalize<N, BLOCK>(accR[s], a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                          a.rho_accumulate != 0);
    }
}

// --------------------------------------------------------------------------------------------
// Growth step 1 <= k < L: A_{k-1} (digits 0..k-1) -> A_k (digits 0..k), in place:
//   A_k[x + v N^k] = K'(v, d_{k-1}(x)) exp(Ds(v) Psi_k(x)) A_{k-1}[x],
//   Psi_k(x) = sum_{j=1..k} psi_{k,j}(d_{k-j}(x)),   classes eta_j (j<k), E_k (j=k, partner sigma_0).
// Readout of rho(t_k) (terminal classes E_j, TI_k) from the same A_{k-1}[x].
// Small (total ~N/(N-1) of one slide step over all k): one thread per input entry, direct exp.
// --------------------------------------------------------------------------------------------
template <int M, bool LAT, bool RO>
__global__ void __launch_bounds__(256) k_grow(const __grid_constant__ GrowArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    const SmallLayout lay{N, D, a.L};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sPsi[2][kMaxL][N];  // psi_{k,j}(sigma) for this k, j = 1..k
    for (int i = threadIdx.x; i < 2 * N * N; i += 256) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < 2 * a.k * N; i += 256) {
        const int kap = i / (a.k * N), r = i % (a.k * N), j = 1 + r / N, sg = r % N;
        sPsi[kap][j][sg] = a.small[lay.psi(kap) + ((size_t)a.k * a.L + j) * N + sg];
    }
    __syncthreads();
    double2 acc[N];
#pragma unroll
    for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
    const long long stride = (long long)gridDim.x * 256;
    long long Nk = 1;
    for (int i = 0; i < a.k; ++i) Nk *= N;
    for (long long x = (long long)blockIdx.x * 256 + threadIdx.x; x < a.n_in; x += stride) {
        const double2 in = a.A[x];
        double2 psi[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
        long long r = x;
        int last = 0;
        for (int q = 0; q < a.k; ++q) {  // digit q holds sigma_q, lag j = k - q
            const int dq = (int)(r % N);
            r /= N;
            const int j = a.k - q;
            psi[0] = cadd(psi[0], sPsi[0][j][dq]);
            if (RO) psi[1] = cadd(psi[1], sPsi[1][j][dq]);
            if (q == a.k - 1) last = dq;
        }
        double2 e[D], eT[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            e[d] = cexp_(make_double2(a.delta[d] * psi[0].x, a.delta[d] * psi[0].y));
            if (RO) eT[d] = cexp_(make_double2(a.delta[d] * psi[1].x, a.delta[d] * psi[1].y));
        }
#pragma unroll
        for (int aa = 0; aa < M; ++aa)
#pragma unroll
            for (int bb = 0; bb < M; ++bb) {
                const int nw = aa * M + bb;
                const int c = class_of(M, LAT, aa, bb);
                const double2 fac = c == 0 ? sK[0][nw][last] : cmul(sK[0][nw][last], e[c > 0 ? c - 1 : 0]);
                a.A[x + nw * Nk] = cmul(fac, in);
                if (RO) {
                    const double2 ft = c == 0 ? sK[1][nw][last] : cmul(sK[1][nw][last], eT[c > 0 ? c - 1 : 0]);
                    acc[nw] = cfma(ft, in, acc[nw]);
                }
            }
    }
    if (RO) reduce_finalize<N, 256>(acc, a.partials, a.rho, a.counter);
}

// --------------------------------------------------------------------------------------------
// Launch configuration per M (FusedShape in qp_internal.h) and dispatch.
// --------------------------------------------------------------------------------------------
// (M, S) -> block, tile digits v (TILE = N^v outer fibres; TILE * N^(S-1) = block for S > 1), min blocks/SM
#define QP_FUSED_CFGS(X)         \
    X(2, 1, 256, 4, 256, 3)      \
    X(2, 2, 256, 3, 64, 3)       \
    X(3, 1, 736, 3, 736, 1)      \
    X(4, 1, 256, 2, 256, 2)
// register variant k_fused_r: (M, S, block, v, min blocks, cp.async staging)
#define QP_FUSED_R_CFGS(X)           \
    X(2, 1, 256, 4, 2, false)        \
    X(2, 2, 256, 4, 2, false)        \
    X(3, 1, 256, 3, 2, false)
// split-register variant k_fused_p2 (S = 2 only): (M, S, block, v, min blocks, unused)
#define QP_FUSED_P_CFGS(X)           \
    X(2, 2, 256, 4, 3, false)
#define QP_FUSED_A_CFGS(X)           \
    X(2, 1, 128, 4, 2, true)         \
    X(2, 2, 128, 4, 2, true)         \
    X(3, 1, 128, 3, 2, true)

FusedShape fused_shape(int M) {
    switch (M) {
    case 2: return FusedShape{2, 4};
    case 3: return FusedShape{1, 3};
    default: return FusedShape{1, 2};
    }
}

// kind: 0 = warp-mapped k_fused, 1 = register k_fused_r, 2 = register k_fused_r with cp.async staging
// kind 4: three fused steps per pass (k_fused3, M = 2); S < 3 launches of such a plan use kind 1
static int eff_kind(int M, int S, int kind) { return kind == 4 ? ((M == 2 && S == 3) ? 4 : 1) : kind; }

// k_fused3 launch variants (index, mode, BLOCK, MINB, PFM).  mode = lane map + 2 x TMA staging,
// fixed per launch (FusedArgs::lane_map, use_tma); QUAPI_F3 = index selects a variant of that mode
// for tuning, else the mode's default (no register spills at <= 168 registers).
#define QP_F3_CFGS(X)                                                                              \
    X(0, 0, 256, 2, 0) X(1, 0, 192, 2, 0) X(2, 0, 128, 3, 0) X(3, 1, 128, 3, 0) X(4, 1, 256, 1, 0) \
    X(5, 1, 384, 1, 0) X(6, 1, 128, 2, 1) X(7, 3, 128, 2, 2) X(8, 3, 256, 1, 2) X(9, 2, 128, 2, 2)              \
    X(10, 2, 256, 1, 2) X(11, 4, 128, 2, 3) X(12, 2, 256, 2, 4) X(13, 2, 128, 4, 4) X(14, 2, 128, 2, 5)
static int f3_mode(const FusedArgs &a) { return a.use_tma == 2 ? 4 : (a.lane_map & 1) + (a.use_tma ? 2 : 0); }
static int f3_variant(int mode, bool view_a = true) {
    // mode 2 (TMA, lane map 0): per-warp staging (14) -- measured 1.917-1.946 vs 1.988-2.001 ms mean
    // launch on cfg3 for the CTA-wide stage (9, QUAPI_F3=9)
    const int def = mode == 0 ? 1 : (mode == 1 ? 3 : (mode == 2 ? 14 : (mode == 3 ? 7 : 11)));
    const char *e = std::getenv("QUAPI_F3");
    if (!e) return def;
    const int v = std::atoi(e);
    // k_fused3s (PM 4) assumes the view-A stage layout
#define X(I, MD, B, MB, PM) if (v == I) return (MD == mode && (PM != 4 || view_a)) ? I : def;
    QP_F3_CFGS(X)
#undef X
    return def;
}
int fused3_round_fibres(int mode, bool view_a) {
    const int v = f3_variant(mode, view_a);  // the variant launch_fused will pick for this launch set
#define X(I, MD, B, MB, PM) if (v == I) return PM == 4 ? 32 : (PM == 5 ? 8 : B / 4);
    QP_F3_CFGS(X)
#undef X
    return 32;
}

bool has_reg_variant(int M, int S, int kind) {
    kind = eff_kind(M, S, kind);
    if (kind == 4) return true;
    if (kind == 3) {
#define X(M_, S_, B, V, MB, AS) if (M == M_ && S == S_) return true;
        QP_FUSED_P_CFGS(X)
#undef X
    }
    if (kind == 1) {
#define X(M_, S_, B, V, MB, AS) if (M == M_ && S == S_) return true;
        QP_FUSED_R_CFGS(X)
#undef X
    }
    if (kind == 2) {
#define X(M_, S_, B, V, MB, AS) if (M == M_ && S == S_) return true;
        QP_FUSED_A_CFGS(X)
#undef X
    }
    return false;
}

int fused_tile_digits(int M, int S, int kind) {
    kind = eff_kind(M, S, kind);
    if (kind == 4) return 5;
#define X(M_, S_, B, V, MB, AS) if (M == M_ && S == S_) return V;
    if (kind == 1 && has_reg_variant(M, S, 1)) { QP_FUSED_R_CFGS(X) }
    if (kind == 2 && has_reg_variant(M, S, 2)) { QP_FUSED_A_CFGS(X) }
    if (kind == 3 && has_reg_variant(M, S, 3)) { QP_FUSED_P_CFGS(X) }
#undef X
#define X(M_, S_, B, V, TL, MB) if (M == M_ && S == S_) return V;
    QP_FUSED_CFGS(X)
#undef X
    return -1;
}

int fused_tile_digits_min(int M, int S, int kind) {
    kind = eff_kind(M, S, kind);
    const int N = M * M;
    if (kind == 4) return 3;                   // k_fused3: a round is 8 warps x 8 outer fibres = 64
    if (kind == 0) return fused_tile_digits(M, S, kind);  // k_fused: compile-time TILE
    if (kind == 3) return N >= 16 ? 1 : 2;     // k_fused_p2: chunks of 16 outer fibres
    return N >= 9 ? 2 : 3;                     // k_fused_r (+async): chunks of 32 outer fibres
}

int fused_block(int M, int S, int kind) {
    kind = eff_kind(M, S, kind);
    if (kind == 4) {
#define X(I, MD, B, MB, PM) if (f3_variant(0) == I) return B;
        QP_F3_CFGS(X)
#undef X
    }
#define X(M_, S_, B, V, MB, AS) if (M == M_ && S == S_) return B;
    if (kind == 1 && has_reg_variant(M, S, 1)) { QP_FUSED_R_CFGS(X) }
    if (kind == 2 && has_reg_variant(M, S, 2)) { QP_FUSED_A_CFGS(X) }
    if (kind == 3 && has_reg_variant(M, S, 3)) { QP_FUSED_P_CFGS(X) }
#undef X
#define X(M_, S_, B, V, TL, MB) if (M == M_ && S == S_) return B;
    QP_FUSED_CFGS(X)
#undef X
    return 0;
}

template <int M, int S, int BLOCK, bool ASYNC>
static constexpr size_t fused_r_dyn_smem(bool ro) {
    return ((ro ? (size_t)S * M * M * BLOCK : 0) + (ASYNC ? (size_t)(BLOCK / 32) * 2 * cpow(M * M, S) * 32 : 0)) * 16;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool ASYNC>
static cudaError_t fused_r_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    const size_t dyn = fused_r_dyn_smem<M, S, BLOCK, ASYNC>(ro);
    if (ro) {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, true><<<grid, BLOCK, dyn, s>>>(a);
    } else {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, false><<<grid, BLOCK, dyn, s>>>(a);
    }
    return cudaGetLastError();
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool ASYNC>
static int fused_r_occ_t() {
    int o1 = 0, o2 = 0;
    const size_t d1 = fused_r_dyn_smem<M, S, BLOCK, ASYNC>(true), d2 = fused_r_dyn_smem<M, S, BLOCK, ASYNC>(false);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d2);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, ASYNC, false>, BLOCK, d2);
    return o1 < o2 ? o1 : o2;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool ASYNC>
static cudaError_t fused_p_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    const size_t dyn = ro ? (size_t)S * M * M * BLOCK * 16 : 0;
    if (ro) {
        cudaFuncSetAttribute(k_fused_p2<M, LAT, SYM, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_p2<M, LAT, SYM, BLOCK, MINB, true><<<grid, BLOCK, dyn, s>>>(a);
    } else {
        k_fused_p2<M, LAT, SYM, BLOCK, MINB, false><<<grid, BLOCK, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool ASYNC>
static int fused_p_occ_t() {
    int o1 = 0, o2 = 0;
    const size_t d1 = (size_t)S * M * M * BLOCK * 16;
    cudaFuncSetAttribute(k_fused_p2<M, LAT, SYM, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused_p2<M, LAT, SYM, BLOCK, MINB, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused_p2<M, LAT, SYM, BLOCK, MINB, false>, BLOCK, 0);
    return o1 < o2 ? o1 : o2;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int TILE, int MINB>
static cudaError_t fused_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    if (ro) k_fused<M, LAT, SYM, S, BLOCK, TILE, MINB, true><<<grid, BLOCK, 0, s>>>(a);
    else k_fused<M, LAT, SYM, S, BLOCK, TILE, MINB, false><<<grid, BLOCK, 0, s>>>(a);
    return cudaGetLastError();
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int TILE, int MINB>
static int fused_occ_t() {
    int o1 = 0, o2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused<M, LAT, SYM, S, BLOCK, TILE, MINB, true>, BLOCK, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused<M, LAT, SYM, S, BLOCK, TILE, MINB, false>, BLOCK, 0);
    return o1 < o2 ? o1 : o2;
}

// M = 2: the lattice and general class maps give the same classes; the host uses LAT = false.
static size_t fused3_dyn(int block, bool ro, int pfm) {
    const size_t F = block / 4;
    return ((pfm >= 2 ? F * 64 + 2 * 3 * 2 * 2 * F + F : 0) + (size_t)(block / 32) * 16 * 8 + (ro ? (size_t)3 * 4 * block : 0)) * 16;
}

static constexpr size_t fused3s_dyn() { return (size_t)(2 * 64 * 32 + 2 * 3 * 2 * 2 * 32 + 32) * 16; }

template <bool SYM, int MAP, int BLOCK, int MINB, int PF>
static cudaError_t fused3_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    if constexpr (PF == 4) {
        const size_t dyn = fused3s_dyn();
        if (ro) {
            cudaFuncSetAttribute(k_fused3s<SYM, BLOCK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            k_fused3s<SYM, BLOCK, true><<<grid, BLOCK, dyn, s>>>(a);
        } else {
            cudaFuncSetAttribute(k_fused3s<SYM, BLOCK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            k_fused3s<SYM, BLOCK, false><<<grid, BLOCK, dyn, s>>>(a);
        }
        return cudaGetLastError();
    }
    const size_t dyn = fused3_dyn(BLOCK, ro, PF);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        kern<<<grid, BLOCK, dyn, s>>>(a);
    };
    // the default TMA variant (lane map 0, 128 threads) gets one instantiation per stage view
    // (the default per-warp variant only: instantiating the CTA-stage variant per view as well costs a
    // minute of build time for a non-default path)
    constexpr bool spec = PF == 5 && MAP == 0 && BLOCK == 128 && MINB == 2;
    if (spec && a.use_tma == 1) {
        switch (a.tma_swz) {
        case 0: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 0 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 0 : -1>); break;
        case 1: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 1 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 1 : -1>); break;
        case 2: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 2 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 2 : -1>); break;
        case 3: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 3 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 3 : -1>); break;
        case 5: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 5 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 5 : -1>); break;
        default: ro ? go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true, spec ? 4 : -1>) : go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false, spec ? 4 : -1>); break;
        }
        return cudaGetLastError();
    }
    if (ro) go(k_fused3<SYM, MAP, BLOCK, MINB, PF, true>);
    else go(k_fused3<SYM, MAP, BLOCK, MINB, PF, false>);
    return cudaGetLastError();
}

template <bool SYM, int MAP, int BLOCK, int MINB, int PF>
static int fused3_occ_t() {
    int o1 = 0, o2 = 0;
    if constexpr (PF == 4) {
        const size_t dyn = fused3s_dyn();
        cudaFuncSetAttribute(k_fused3s<SYM, BLOCK, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(k_fused3s<SYM, BLOCK, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused3s<SYM, BLOCK, true>, BLOCK, dyn);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused3s<SYM, BLOCK, false>, BLOCK, dyn);
        return o1 < o2 ? o1 : o2;
    }
    const size_t d1 = fused3_dyn(BLOCK, true, PF), d2 = fused3_dyn(BLOCK, false, PF);
    cudaFuncSetAttribute(k_fused3<SYM, MAP, BLOCK, MINB, PF, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaFuncSetAttribute(k_fused3<SYM, MAP, BLOCK, MINB, PF, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d2);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused3<SYM, MAP, BLOCK, MINB, PF, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused3<SYM, MAP, BLOCK, MINB, PF, false>, BLOCK, d2);
    return o1 < o2 ? o1 : o2;
}

cudaError_t launch_fused(int M, bool lattice, bool sym, int kind, int S, const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    kind = eff_kind(M, S, kind);
    if (kind == 4) {
#define X(I, MD, B, MB, PF)                                                                          \
        if (f3_variant(f3_mode(a), a.tma_sf == 1) == I)                                                                 \
            return sym ? fused3_t<true, (MD & 1), B, MB, PF>(a, ro, grid, s) : fused3_t<false, (MD & 1), B, MB, PF>(a, ro, grid, s);
        QP_F3_CFGS(X)
#undef X
    }
#define X(M_, S_, B, V, MB, AS)                                                                   \
    if (M == M_ && S == S_) {                                                                     \
        if (M_ == 2 && sym) return fused_r_t<M_, false, (M_ == 2), S_, B, MB, AS>(a, ro, grid, s);\
        if (M_ > 2 && lattice) return fused_r_t<M_, (M_ > 2), false, S_, B, MB, AS>(a, ro, grid, s); \
        return fused_r_t<M_, false, false, S_, B, MB, AS>(a, ro, grid, s);                        \
    }
    if (kind == 1) { QP_FUSED_R_CFGS(X) }
    if (kind == 2) { QP_FUSED_A_CFGS(X) }
#undef X
#define X(M_, S_, B, V, MB, AS)                                                                   \
    if (M == M_ && S == S_) {                                                                     \
        if (M_ == 2 && sym) return fused_p_t<M_, false, (M_ == 2), S_, B, MB, AS>(a, ro, grid, s);\
        return fused_p_t<M_, false, false, S_, B, MB, AS>(a, ro, grid, s);                        \
    }
    if (kind == 3) { QP_FUSED_P_CFGS(X) }
#undef X
#define X(M_, S_, B, V, TL, MB)                                                                   \
    if (M == M_ && S == S_) {                                                                     \
        if (M_ == 2 && sym) return fused_t<M_, false, (M_ == 2), S_, B, TL, MB>(a, ro, grid, s);   \
        if (M_ > 2 && lattice) return fused_t<M_, (M_ > 2), false, S_, B, TL, MB>(a, ro, grid, s); \
        return fused_t<M_, false, false, S_, B, TL, MB>(a, ro, grid, s);                           \
    }
    QP_FUSED_CFGS(X)
#undef X
    return cudaErrorInvalidValue;
}

int fused_occupancy(int M, bool lattice, bool sym, int kind, int S, int mode) {
    kind = eff_kind(M, S, kind);
    if (kind == 4) {
#define X(I, MD, B, MB, PF) \
        if (f3_variant(mode) == I) return sym ? fused3_occ_t<true, (MD & 1), B, MB, PF>() : fused3_occ_t<false, (MD & 1), B, MB, PF>();
        QP_F3_CFGS(X)
#undef X
    }
#define X(M_, S_, B, V, MB, AS)                                                             \
    if (M == M_ && S == S_) {                                                               \
        if (M_ == 2 && sym) return fused_r_occ_t<M_, false, (M_ == 2), S_, B, MB, AS>();     \
        if (M_ > 2 && lattice) return fused_r_occ_t<M_, (M_ > 2), false, S_, B, MB, AS>();   \
        return fused_r_occ_t<M_, false, false, S_, B, MB, AS>();                             \
    }
    if (kind == 1) { QP_FUSED_R_CFGS(X) }
    if (kind == 2) { QP_FUSED_A_CFGS(X) }
#undef X
#define X(M_, S_, B, V, MB, AS)                                                             \
    if (M == M_ && S == S_) {                                                               \
        if (M_ == 2 && sym) return fused_p_occ_t<M_, false, (M_ == 2), S_, B, MB, AS>();     \
        return fused_p_occ_t<M_, false, false, S_, B, MB, AS>();                             \
    }
    if (kind == 3) { QP_FUSED_P_CFGS(X) }
#undef X
#define X(M_, S_, B, V, TL, MB)                                                         \
    if (M == M_ && S == S_) {                                                           \
        if (M_ == 2 && sym) return fused_occ_t<M_, false, (M_ == 2), S_, B, TL, MB>();   \
        if (M_ > 2 && lattice) return fused_occ_t<M_, (M_ > 2), false, S_, B, TL, MB>(); \
        return fused_occ_t<M_, false, false, S_, B, TL, MB>();                           \
    }
    QP_FUSED_CFGS(X)
#undef X
    return 0;
}

template <int M, bool LAT>
static cudaError_t grow_t(const GrowArgs &a, int grid, cudaStream_t s) {
    if (a.rho) k_grow<M, LAT, true><<<grid, 256, 0, s>>>(a);
    else k_grow<M, LAT, false><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_grow(int M, bool lattice, const GrowArgs &a, int grid, cudaStream_t s) {
    switch (M) {
    case 2: return grow_t<2, false>(a, grid, s);
    case 3: return lattice ? grow_t<3, true>(a, grid, s) : grow_t<3, false>(a, grid, s);
    case 4: return lattice ? grow_t<4, true>(a, grid, s) : grow_t<4, false>(a, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace qp

// ============================================================================================
// Re-shard data movement (multi-GPU path): one generic digit-permutation copy.
// The dense side index i is a mixed-radix number over `nf` fields (innermost first); field f has
// radix rad[f] and contributes to the strided side's address either linearly (ncd[f] == 0:
// value * str[f][0]) or as a combo of ncd[f] base-N digits of (lo[f] + value) with strides
// str[f][0..ncd-1].  gather: dst[i] = src[addr(i)];  scatter: dst[addr(i)] = src[i].
// ============================================================================================
namespace qp {

template <int N>
__global__ void __launch_bounds__(256) k_permute(const PermuteArgs a) {
    const long long stride = (long long)gridDim.x * 256;
    for (long long i = (long long)blockIdx.x * 256 + threadIdx.x; i < a.count; i += stride) {
        long long rest = i, addr = a.base;
        for (int f = 0; f < a.nf; ++f) {
            const long long v = rest % a.rad[f];
            rest /= a.rad[f];
            if (a.ncd[f] == 0) {
                addr += v * a.str[f][0];
            } else {
                long long c = a.lo[f] + v;
                for (int j = 0; j < a.ncd[f]; ++j) {
                    addr += (c % N) * a.str[f][j];
                    c /= N;
                }
            }
        }
        if (a.scatter) a.dst[addr] = __ldcs(a.src + i);
        else a.dst[i] = __ldcs(a.src + addr);
    }
}

cudaError_t launch_permute(int M, const PermuteArgs &a, int sms, cudaStream_t s) {
    if (a.count <= 0) return cudaSuccess;
    const int grid = (int)std::min<long long>((a.count + 255) / 256, (long long)sms * 16);
    switch (M) {
    case 2: k_permute<4><<<grid, 256, 0, s>>>(a); break;
    case 3: k_permute<9><<<grid, 256, 0, s>>>(a); break;
    case 4: k_permute<16><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace qp
