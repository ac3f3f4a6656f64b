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
// it visits; it issues all F*N 16-byte loads of a tile before any arithmetic.
// --------------------------------------------------------------------------------------------
template <int M, bool LAT, int BLOCK, int F, bool RO>
__global__ void __launch_bounds__(BLOCK) k_slide(const __grid_constant__ SlideArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
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
    double2 acc[N];
#pragma unroll
    for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
    __syncthreads();

    const double2 *__restrict__ E0 = a.Etab;  // group 0, kappa 0: [d][X]
    for (int tau = blockIdx.x; tau < a.n_tiles; tau += gridDim.x) {
        const long long base = a.p_ge_v ? (long long)(tau % a.Qlo) * a.T + (long long)(tau / a.Qlo) * a.pw_p1
                                        : (long long)tau * a.tile_stride;
        // tile-uniform factors: product of the group tables g >= 1
        double2 Et[RO ? 2 : 1][D];
#pragma unroll
        for (int kap = 0; kap < (RO ? 2 : 1); ++kap)
#pragma unroll
            for (int d = 0; d < D; ++d) Et[kap][d] = make_double2(1.0, 0.0);
        for (int g = 1; g < a.G; ++g) {
            const int idx = (tau / a.gdiv[g]) % a.gmod[g];
#pragma unroll
            for (int kap = 0; kap < (RO ? 2 : 1); ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    Et[kap][d] = cmul(Et[kap][d], __ldg(&a.Etab[((size_t)(kap * a.G + g) * D + d) * a.X + idx]));
        }
        const int last_t = a.last_div > 0 ? (tau / a.last_div) % N : 0;

        double2 x[F][N];
#pragma unroll
        for (int j = 0; j < F; ++j)
            if (valid[j]) {
                const double2 *src = a.A + base + off[j];
#pragma unroll
                for (int v = 0; v < N; ++v) x[j][v] = __ldcs(src + v * a.pw_p);
            }
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
                const double2 e = cmul(Et[0][d], __ldg(&E0[(size_t)d * a.X + fl]));
                P[d] = cmul(e, s);
            }
            double2 *dst = a.A + base + off[j];
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    constexpr int dummy = 0;
                    (void)dummy;
                    const int nw = aa * M + bb;
                    const int c = class_of(M, LAT, aa, bb);
                    const double2 o = cmul(sK[0][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                    __stcs(dst + nw * a.pw_p, o);
                    if (RO && c == 0) acc[nw] = cadd(acc[nw], o);
                }
            if (RO) {
                double2 PT[D];
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double2 s = cmul(sB[1][d][0], x[j][0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) s = cfma(sB[1][d][v], x[j][v], s);
                    const double2 e =
                        cmul(Et[RO ? 1 : 0][d], __ldg(&a.Etab[((size_t)(1 * a.G + 0) * D + d) * a.X + fl]));
                    PT[d] = cmul(e, s);
                }
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int nw = aa * M + bb;
                        const int c = class_of(M, LAT, aa, bb);
                        if (c != 0) acc[nw] = cfma(sK[1][nw][last], PT[c - 1], acc[nw]);
                    }
            }
        }
    }
    if (RO) reduce_finalize<N, BLOCK>(acc, a.partials, a.rho, a.counter);
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
// launch configuration per M:  block, fibres per thread, tile digits v (T = N^v), group digits w
// --------------------------------------------------------------------------------------------
template <int M> struct Shape;
template <> struct Shape<2> { static constexpr int block = 256, F = 4, v = 5, w = 6; };   // T = 1024
template <> struct Shape<3> { static constexpr int block = 384, F = 2, v = 3, w = 3; };   // T = 729
template <> struct Shape<4> { static constexpr int block = 256, F = 1, v = 2, w = 3; };   // T = 256

void slide_shape(int M, int *block, int *F, int *v, int *w) {
    switch (M) {
    case 2: *block = Shape<2>::block; *F = Shape<2>::F; *v = Shape<2>::v; *w = Shape<2>::w; break;
    case 3: *block = Shape<3>::block; *F = Shape<3>::F; *v = Shape<3>::v; *w = Shape<3>::w; break;
    default: *block = Shape<4>::block; *F = Shape<4>::F; *v = Shape<4>::v; *w = Shape<4>::w; break;
    }
}

template <int M, bool LAT>
static cudaError_t slide_t(const SlideArgs &a, int grid, cudaStream_t s) {
    using S = Shape<M>;
    if (a.rho) k_slide<M, LAT, S::block, S::F, true><<<grid, S::block, 0, s>>>(a);
    else k_slide<M, LAT, S::block, S::F, false><<<grid, S::block, 0, s>>>(a);
    return cudaGetLastError();
}

template <int M, bool LAT>
static cudaError_t grow_t(const GrowArgs &a, int grid, cudaStream_t s) {
    if (a.rho) k_grow<M, LAT, true><<<grid, 256, 0, s>>>(a);
    else k_grow<M, LAT, false><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_slide(int M, bool lattice, const SlideArgs &a, int grid, cudaStream_t s) {
    switch (M) {
    case 2: return slide_t<2, false>(a, grid, s);  // M = 2: both class maps coincide
    case 3: return lattice ? slide_t<3, true>(a, grid, s) : slide_t<3, false>(a, grid, s);
    case 4: return lattice ? slide_t<4, true>(a, grid, s) : slide_t<4, false>(a, grid, s);
    default: return cudaErrorInvalidValue;
    }
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
