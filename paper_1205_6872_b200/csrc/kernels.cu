// kernels.cu -- sm_100a kernels of the QUAPI tensor-propagator step (arXiv 1205.6872).
//
// k_slide : one time step k >= L of the iterative tensor propagator (Makri-Makarov scheme the
//           paper accelerates, "BSXFUN" lines), in place on a ring-buffer ARDM,
//           with the rho(t_k) readout ("line 169") fused into the same pass.
// k_grow  : growth steps 1 <= k < L (no contraction; the tensor gains one digit per step).
//
// ARDM layout: A has N^L complex FP64 entries, flat index x = sum_q d_q N^q.
// Time point t lives in digit q = t mod L ("ring slot"), so no data is ever transposed.
// Step k (k >= L) contracts slot p = k mod L (holding sigma_{k-L}) and writes sigma_k into the
// same slot.  For one fibre (all digits except p fixed = "mid") with old values a[old]:
//   out[new] = K'(new, last) * exp(Ds(new) Psi(mid)) * sum_old exp(Ds(new) psi_L(old)) a[old]
// where Ds = s+ - s- of the new pair state, K' = self factor * bare propagator pair (Eq. 8),
// Psi(mid) = sum_j psi_j(digit at lag j) the Eq. 9 exponent of the kept partners and psi_L the
// lag-L (summed) partner.  Rows with the same Ds share one "moment" S_d = sum_old beta_d(old) a[old]
// and one factor E_d = exp(delta_d Psi): E_d is a product of per-digit-group tables (host-built),
// one uniform factor per tile times one per-fibre factor.  No transcendental in the slide kernel.
// The readout of rho(t_k) uses the same loaded fibre with the terminal classes (E_j, TI) and
// accumulates sum over all mid of K'_term * E^T_d * S^T_d (diagonal rows: the propagated value).
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

// Fixed-order block reduction of N complex accumulators into partials[blockIdx][N]; the last
// block to finish sums the partials over blocks in fixed order into rho[N] (deterministic:
// the grid and the tile->block assignment are fixed by the plan).
template <int N, int BLOCK>
__device__ __forceinline__ void reduce_finalize(double2 (&acc)[N], double2 *partials, double2 *rho,
                                                unsigned *counter) {
    constexpr int W = BLOCK / 32;
    __shared__ double2 red[W][N];
    __shared__ double2 fin[W];
    __shared__ int is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
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
            rho[n] = t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *counter = 0u;
}

// --------------------------------------------------------------------------------------------
// Slide step (k >= L), persistent over tiles.  Tile tau = T consecutive fibres (the v lowest
// "mid" digits vary inside a tile).  Thread t owns fibres f = t + j*BLOCK (j < F) of every tile
// it visits; it issues all F*N 16-byte loads of a tile before any arithmetic.  With PREF the
// loads of the thread's next tile are issued before the current tile is computed and stored
// (register double buffering), so HBM requests stay in flight through the FP64 work.
// --------------------------------------------------------------------------------------------
__device__ __forceinline__ long long tile_base(const SlideArgs &a, int tau) {
    return a.p_ge_v ? (long long)(tau % a.Qlo) * a.T + (long long)(tau / a.Qlo) * a.pw_p1
                    : (long long)tau * a.tile_stride;
}

template <int M, bool LAT, int BLOCK, int F, int MINB, bool PREF, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_slide(const __grid_constant__ SlideArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    constexpr int NK = RO ? 2 : 1;
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];   // K'(new, last): [0] propagate, [1] terminal (readout)
    __shared__ double2 sB[2][D][N];   // beta_d(old):   [0] propagate, [1] terminal
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < 2 * D * N; i += BLOCK) (&sB[0][0][0])[i] = a.small[lay.beta(a.variant, 0) + i];

    int off[F], lastlo[F];
    bool valid[F];
#pragma unroll
    for (int j = 0; j < F; ++j) {
        const int fl = threadIdx.x + j * BLOCK;
        valid[j] = fl < a.T;
        const int2 o = valid[j] ? a.lofs[fl] : make_int2(0, 0);
        off[j] = o.x;
        lastlo[j] = o.y;
    }
    double2 acc[RO ? N : 1];
#pragma unroll
    for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
    __syncthreads();

    double2 x[F][N], xn[PREF ? F : 1][N];
    auto load = [&](int tau, double2 (&dst)[PREF ? F : 1][N], int jj) {
        const double2 *src = a.A + tile_base(a, tau) + off[jj];
#pragma unroll
        for (int v = 0; v < N; ++v) dst[PREF ? jj : 0][v] = __ldcs(src + v * a.pw_p);
    };
    int tau = blockIdx.x;
    if (PREF && tau < a.n_tiles) {
#pragma unroll
        for (int j = 0; j < F; ++j)
            if (valid[j]) load(tau, xn, j);
    }
    for (; tau < a.n_tiles; tau += gridDim.x) {
        if (PREF) {
#pragma unroll
            for (int j = 0; j < F; ++j)
#pragma unroll
                for (int v = 0; v < N; ++v) x[j][v] = xn[PREF ? j : 0][v];
            const int tn = tau + gridDim.x;
            if (tn < a.n_tiles) {
#pragma unroll
                for (int j = 0; j < F; ++j)
                    if (valid[j]) load(tn, xn, j);
            }
        } else {
            const long long b0 = tile_base(a, tau);
#pragma unroll
            for (int j = 0; j < F; ++j)
                if (valid[j]) {
                    const double2 *src = a.A + b0 + off[j];
#pragma unroll
                    for (int v = 0; v < N; ++v) x[j][v] = __ldcs(src + v * a.pw_p);
                }
        }
        const long long base = tile_base(a, tau);
        // tile-uniform factors: product of the group tables g >= 1
        double2 Et[NK][D];
#pragma unroll
        for (int kap = 0; kap < NK; ++kap)
#pragma unroll
            for (int d = 0; d < D; ++d) Et[kap][d] = make_double2(1.0, 0.0);
        for (int g = 1; g < a.G; ++g) {
            const int idx = (tau / a.gdiv[g]) % a.gmod[g];
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    Et[kap][d] = cmul(Et[kap][d], __ldg(&a.Etab[((size_t)(kap * a.G + g) * D + d) * a.X + idx]));
        }
        const int last_t = a.last_div > 0 ? (tau / a.last_div) % N : 0;
#pragma unroll
        for (int j = 0; j < F; ++j) {
            if (!valid[j]) continue;
            const int fl = threadIdx.x + j * BLOCK;
            const int last = lastlo[j] >= 0 ? lastlo[j] : last_t;
            double2 S0 = x[j][0];
#pragma unroll
            for (int v = 1; v < N; ++v) S0 = cadd(S0, x[j][v]);
            double2 P[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                double2 s = cmul(sB[0][d][0], x[j][0]);
#pragma unroll
                for (int v = 1; v < N; ++v) s = cfma(sB[0][d][v], x[j][v], s);
                const double2 e = cmul(Et[0][d], __ldg(&a.Etab[(size_t)d * a.X + fl]));
                P[d] = cmul(e, s);
            }
            double2 *dst = a.A + base + off[j];
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    const int nw = aa * M + bb;
                    const int c = class_of(M, LAT, aa, bb);
                    const double2 o = cmul(sK[0][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                    __stcs(dst + nw * a.pw_p, o);
                    if (RO && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
                }
            if (RO) {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double2 s = cmul(sB[1][d][0], x[j][0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) s = cfma(sB[1][d][v], x[j][v], s);
                    const double2 e =
                        cmul(Et[NK - 1][d], __ldg(&a.Etab[((size_t)(1 * a.G + 0) * D + d) * a.X + fl]));
                    P[d] = cmul(e, s);
                }
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int nw = aa * M + bb;
                        const int c = class_of(M, LAT, aa, bb);
                        if (c != 0) acc[RO ? nw : 0] = cfma(sK[1][nw][last], P[c > 0 ? c - 1 : 0], acc[RO ? nw : 0]);
                    }
            }
        }
    }
    if constexpr (RO) reduce_finalize<N, BLOCK>(acc, a.partials, a.rho, a.counter);
}

// --------------------------------------------------------------------------------------------
// TMA-staged slide step.  Persistent CTAs stream tiles through an S-stage shared-memory ring:
// thread 0 issues 1-D bulk copies (cp.async.bulk, TMA engine) global -> smem completing on a
// per-stage mbarrier, all threads compute their fibres in smem and overwrite them in place, and
// thread 0 writes the stage back with a bulk smem -> global copy.  Up to S-1 tiles of loads are in
// flight per CTA independently of the register budget.  Tile = N segments of T contiguous entries
// (contracted digit p above the tile digits) or one contiguous block of N*T entries (p below).
// --------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int NPEND> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NPEND) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void tma_load_tile(const SlideArgs &a, double2 *stage, int tau, uint64_t *bar) {
    const long long base = tile_base(a, tau);
    const unsigned seg = (unsigned)a.T * 16u;
    mbar_expect_tx(bar, seg * N);
    if (a.p_ge_v) {
#pragma unroll
        for (int v = 0; v < N; ++v) bulk_g2s(stage + v * a.T, a.A + base + v * a.pw_p, seg, bar);
    } else {
        bulk_g2s(stage, a.A + base, seg * N, bar);
    }
}

template <int N>
__device__ __forceinline__ void tma_store_tile(const SlideArgs &a, const double2 *stage, int tau) {
    const long long base = tile_base(a, tau);
    const unsigned seg = (unsigned)a.T * 16u;
    if (a.p_ge_v) {
#pragma unroll
        for (int v = 0; v < N; ++v) bulk_s2g(a.A + base + v * a.pw_p, stage + v * a.T, seg);
    } else {
        bulk_s2g(a.A + base, stage, seg * N);
    }
    bulk_commit();
}

template <int M, bool LAT, int BLOCK, int F, int S, bool RO>
__global__ void __launch_bounds__(BLOCK, 1) k_slide_tma(const __grid_constant__ SlideArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    constexpr int NK = RO ? 2 : 1;
    const SmallLayout lay{N, D, 0};
    extern __shared__ __align__(128) double2 ring[];  // [S][N*T]
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sB[2][D][N];
    __shared__ __align__(8) uint64_t full[S];
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < 2 * D * N; i += BLOCK) (&sB[0][0][0])[i] = a.small[lay.beta(a.variant, 0) + i];
    const int stage_elems = N * a.T;
    // my tiles: tau_i = blockIdx.x + i * gridDim.x, i < n_my
    const int n_my = a.n_tiles > (int)blockIdx.x ? (a.n_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (threadIdx.x == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < S - 1 && i < n_my; ++i)
            tma_load_tile<N>(a, ring + (size_t)i * stage_elems, blockIdx.x + i * gridDim.x, &full[i]);
    }
    int off[F], lastlo[F];
    bool valid[F];
#pragma unroll
    for (int j = 0; j < F; ++j) {
        const int fl = threadIdx.x + j * BLOCK;
        valid[j] = fl < a.T;
        const int2 o = valid[j] ? a.lofs[fl] : make_int2(0, 0);
        off[j] = o.x;
        lastlo[j] = o.y;
    }
    const int sstride = a.p_ge_v ? a.T : (int)a.pw_p;  // smem distance between the N values of a fibre
    double2 acc[RO ? N : 1];
#pragma unroll
    for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
    __syncthreads();

    for (int i = 0; i < n_my; ++i) {
        const int st = i % S;
        const int tau = blockIdx.x + i * gridDim.x;
        double2 *stage = ring + (size_t)st * stage_elems;
        double2 Et[NK][D];
#pragma unroll
        for (int kap = 0; kap < NK; ++kap)
#pragma unroll
            for (int d = 0; d < D; ++d) Et[kap][d] = make_double2(1.0, 0.0);
        for (int g = 1; g < a.G; ++g) {
            const int idx = (tau / a.gdiv[g]) % a.gmod[g];
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    Et[kap][d] = cmul(Et[kap][d], __ldg(&a.Etab[((size_t)(kap * a.G + g) * D + d) * a.X + idx]));
        }
        const int last_t = a.last_div > 0 ? (tau / a.last_div) % N : 0;
        mbar_wait(&full[st], (unsigned)(i / S) & 1u);
#pragma unroll
        for (int j = 0; j < F; ++j) {
            if (!valid[j]) continue;
            const int fl = threadIdx.x + j * BLOCK;
            const int last = lastlo[j] >= 0 ? lastlo[j] : last_t;
            double2 *xp = stage + off[j];
            double2 x[N];
#pragma unroll
            for (int v = 0; v < N; ++v) x[v] = xp[v * sstride];
            double2 S0 = x[0];
#pragma unroll
            for (int v = 1; v < N; ++v) S0 = cadd(S0, x[v]);
            double2 P[D];
#pragma unroll
            for (int d = 0; d < D; ++d) {
                double2 sacc = cmul(sB[0][d][0], x[0]);
#pragma unroll
                for (int v = 1; v < N; ++v) sacc = cfma(sB[0][d][v], x[v], sacc);
                P[d] = cmul(cmul(Et[0][d], __ldg(&a.Etab[(size_t)d * a.X + fl])), sacc);
            }
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    const int nw = aa * M + bb;
                    const int c = class_of(M, LAT, aa, bb);
                    const double2 o = cmul(sK[0][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                    xp[nw * sstride] = o;
                    if (RO && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
                }
            if (RO) {
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double2 sacc = cmul(sB[1][d][0], x[0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) sacc = cfma(sB[1][d][v], x[v], sacc);
                    P[d] = cmul(cmul(Et[NK - 1][d], __ldg(&a.Etab[((size_t)(1 * a.G + 0) * D + d) * a.X + fl])), sacc);
                }
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int nw = aa * M + bb;
                        const int c = class_of(M, LAT, aa, bb);
                        if (c != 0) acc[RO ? nw : 0] = cfma(sK[1][nw][last], P[c > 0 ? c - 1 : 0], acc[RO ? nw : 0]);
                    }
            }
        }
        fence_async_smem();  // make this thread's smem writes visible to the TMA (async proxy)
        __syncthreads();
        if (threadIdx.x == 0) {
            tma_store_tile<N>(a, stage, tau);
            // refill the stage of tile i-1 (its store was the previous bulk group) with tile i-1+S
            if (i + S - 1 < n_my) {
                const int rs = (i + S - 1) % S;
                if (i >= 1) bulk_wait_read<1>();
                tma_load_tile<N>(a, ring + (size_t)rs * stage_elems, blockIdx.x + (i + S - 1) * gridDim.x, &full[rs]);
            }
        }
    }
    if (threadIdx.x == 0) bulk_wait_all();
    if constexpr (RO) reduce_finalize<N, BLOCK>(acc, a.partials, a.rho, a.counter);
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
// Slide-kernel variants (tile shape and pipelining); the plan picks one per M (env override
// QUAPI_SLIDE_VARIANT=<id> for tuning).  v = tile digits (T = N^v), w = hi-group digits.
// --------------------------------------------------------------------------------------------
// Variant registry.  R(id, M, block, F, v, w, minBlocks, prefetch): register-path k_slide;
// T(id, M, block, F, v, w, stages): TMA-staged k_slide_tma (smem = stages * N^(v+1) * 16 B).
#define QP_REG_VARIANTS(R)              \
    R(0, 2, 256, 4, 5, 6, 1, false)     \
    R(1, 2, 256, 1, 4, 6, 3, false)     \
    R(2, 2, 256, 1, 4, 6, 2, true)      \
    R(3, 2, 128, 2, 4, 6, 4, false)     \
    R(10, 3, 384, 2, 3, 3, 1, false)    \
    R(11, 3, 768, 1, 3, 3, 1, false)    \
    R(12, 3, 768, 1, 3, 3, 1, true)     \
    R(20, 4, 256, 1, 2, 3, 2, false)
#define QP_TMA_VARIANTS(T)              \
    T(5, 2, 256, 1, 4, 6, 4)            \
    T(6, 2, 256, 1, 4, 6, 3)            \
    T(7, 2, 256, 4, 5, 6, 3)            \
    T(8, 2, 128, 2, 4, 6, 4)            \
    T(13, 3, 256, 3, 3, 3, 2)           \
    T(14, 3, 384, 2, 3, 3, 2)

static const SlideVariant kVariants[] = {
#define R(id, M, B, F, V, W, MB, PF) {id, M, B, F, V, W, MB, PF ? 1 : 0, 0},
#define T(id, M, B, F, V, W, ST) {id, M, B, F, V, W, 1, 0, ST},
    QP_REG_VARIANTS(R) QP_TMA_VARIANTS(T)
#undef R
#undef T
};

const SlideVariant *find_variant(int id) {
    for (const auto &v : kVariants)
        if (v.id == id) return &v;
    return nullptr;
}

int default_variant(int M) { return M == 2 ? 3 : (M == 3 ? 11 : 20); }

template <int M, bool LAT, int BLOCK, int F, int MINB, bool PREF>
static cudaError_t slide_t(const SlideArgs &a, int grid, cudaStream_t s) {
    if (a.rho) k_slide<M, LAT, BLOCK, F, MINB, PREF, true><<<grid, BLOCK, 0, s>>>(a);
    else k_slide<M, LAT, BLOCK, F, MINB, PREF, false><<<grid, BLOCK, 0, s>>>(a);
    return cudaGetLastError();
}

template <int M, bool LAT, int BLOCK, int F, int MINB, bool PREF>
static int occ_t() {
    int o1 = 0, o2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_slide<M, LAT, BLOCK, F, MINB, PREF, true>, BLOCK, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_slide<M, LAT, BLOCK, F, MINB, PREF, false>, BLOCK, 0);
    return o1 < o2 ? o1 : o2;
}

template <int M, bool LAT, int BLOCK, int F, int S>
static size_t tma_smem(int T) { return (size_t)S * M * M * T * 16; }

template <int M, bool LAT, int BLOCK, int F, int S>
static cudaError_t slide_tma_t(const SlideArgs &a, int grid, cudaStream_t s) {
    const size_t sm = tma_smem<M, LAT, BLOCK, F, S>(a.T);
    if (a.rho) {
        cudaFuncSetAttribute(k_slide_tma<M, LAT, BLOCK, F, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_slide_tma<M, LAT, BLOCK, F, S, true><<<grid, BLOCK, sm, s>>>(a);
    } else {
        cudaFuncSetAttribute(k_slide_tma<M, LAT, BLOCK, F, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_slide_tma<M, LAT, BLOCK, F, S, false><<<grid, BLOCK, sm, s>>>(a);
    }
    return cudaGetLastError();
}

template <int M, bool LAT, int BLOCK, int F, int S>
static int occ_tma_t(int T) {
    const size_t sm = tma_smem<M, LAT, BLOCK, F, S>(T);
    int o1 = 0, o2 = 0;
    cudaFuncSetAttribute(k_slide_tma<M, LAT, BLOCK, F, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_slide_tma<M, LAT, BLOCK, F, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_slide_tma<M, LAT, BLOCK, F, S, true>, BLOCK, sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_slide_tma<M, LAT, BLOCK, F, S, false>, BLOCK, sm);
    return o1 < o2 ? o1 : o2;
}

// M = 2: the lattice and general class maps are the same set of classes; the host uses LAT = false.
cudaError_t launch_slide(int variant, bool lattice, const SlideArgs &a, int grid, cudaStream_t s) {
#define R(id, M, B, F, V, W, MB, PF)                                               \
    if (variant == id) {                                                            \
        if (M > 2 && lattice) return slide_t<M, (M > 2), B, F, MB, PF>(a, grid, s); \
        return slide_t<M, false, B, F, MB, PF>(a, grid, s);                         \
    }
#define T(id, M, B, F, V, W, ST)                                                   \
    if (variant == id) {                                                            \
        if (M > 2 && lattice) return slide_tma_t<M, (M > 2), B, F, ST>(a, grid, s); \
        return slide_tma_t<M, false, B, F, ST>(a, grid, s);                         \
    }
    QP_REG_VARIANTS(R)
    QP_TMA_VARIANTS(T)
#undef R
#undef T
    return cudaErrorInvalidValue;
}

int slide_occupancy(int variant, bool lattice, int T) {
#define R(id, M, B, F, V, W, MB, PF)                                   \
    if (variant == id) {                                                \
        if (M > 2 && lattice) return occ_t<M, (M > 2), B, F, MB, PF>(); \
        return occ_t<M, false, B, F, MB, PF>();                         \
    }
#define T(id, M, B, F, V, W, ST)                                           \
    if (variant == id) {                                                    \
        if (M > 2 && lattice) return occ_tma_t<M, (M > 2), B, F, ST>(T_); \
        return occ_tma_t<M, false, B, F, ST>(T_);                          \
    }
    const int T_ = T;
    QP_REG_VARIANTS(R)
    QP_TMA_VARIANTS(T)
#undef R
#undef T
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
