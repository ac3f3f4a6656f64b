// grow.cu -- growth steps 1 <= k < L of the iterative tensor propagator (k_grow) and the generic
// digit-permutation copy of the multi-GPU re-shard (k_permute).
#include "common.cuh"

namespace qp {

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

// ============================================================================================
// Re-shard data movement (multi-GPU path): one generic digit-permutation copy.
// The dense side index i is a mixed-radix number over `nf` fields (innermost first); field f has
// radix rad[f] and contributes to the strided side's address either linearly (ncd[f] == 0:
// value * str[f][0]) or as a combo of ncd[f] base-N digits of (lo[f] + value) with strides
// str[f][0..ncd-1].  gather: dst[i] = src[addr(i)];  scatter: dst[addr(i)] = src[i].
// ============================================================================================

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
