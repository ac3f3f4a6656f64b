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

// --------------------------------------------------------------------------------------------
// Sharded growth (multi-GPU): the last z growth steps k = L-z .. L-1 add the z digits
// that are the shard slots of segment 0, so a rank only produces the entries of its own combos c
// (digits c_0..c_{z-1} of slots L-z..L-1).  Every launch reads the replicated A_{L-z-1} (N^(L-z)
// entries, grown in the exchange buffer) and recomputes the chain of growth factors of the combo
// prefix: step i (k = L-z+i) reduces the readout rho(t_k) from A_{k-1} -- for i = 0 the replicated
// tensor (every rank holds the complete sum), for i >= 1 the entries with prefix (c_0..c_{i-1}),
// counted on the rank owning the combo c = prefix (the smallest combo with that prefix) -- and the
// last step writes the rank's blocks: local[c - c_lo][x] = A_{L-1}[x, c].  No rank ever holds N^L.
// --------------------------------------------------------------------------------------------
template <int M, bool LAT, bool RO>
__global__ void __launch_bounds__(256) k_grow_shard(const __grid_constant__ GrowShardArgs a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    const SmallLayout lay{N, D, a.L};
    __shared__ double2 sK[2][N][N];
    for (int i = threadIdx.x; i < 2 * N * N; i += 256) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    __syncthreads();
    const int L = a.L, z = a.z, i = a.step, kb = L - z;  // this launch: step k = kb + i
    double2 acc[N];
#pragma unroll
    for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
    const long long stride = (long long)gridDim.x * 256;
    for (long long x = (long long)blockIdx.x * 256 + threadIdx.x; x < a.nb; x += stride) {
        const double2 base = a.Abase[x];
        int dx[kMaxL];  // digits of x (positions 0 .. kb-1)
        {
            long long r = x;
            for (int q = 0; q < kb; ++q) { dx[q] = (int)(r % N); r /= N; }
        }
        // Psi_k (kap 0: propagate, 1: terminal) over the partners at lags j = 1..k: position k - j
        auto psi_of = [&](int k, int kap, const int *dc) {
            double2 p = make_double2(0.0, 0.0);
            for (int j = 1; j <= k; ++j) {
                const int q = k - j;
                const int d = q < kb ? dx[q] : dc[q - kb];
                p = cadd(p, __ldg(&a.small[lay.psi(kap) + ((size_t)k * L + j) * N + d]));
            }
            return p;
        };
        // A_{kb-1+m}[x, c_0..c_{m-1}]: the growth chain of steps kb .. kb+m-1
        auto chain = [&](const int *dc, int m) {
            double2 v = base;
            for (int t = 0; t < m; ++t) {
                const int k = kb + t, nw = dc[t], last = t == 0 ? dx[kb - 1] : dc[t - 1];
                const int c = class_of(M, LAT, nw / M, nw % M);
                double2 f = sK[0][nw][last];
                if (c > 0) {
                    const double2 p = psi_of(k, 0, dc);
                    f = cmul(f, cexp_(make_double2(a.delta[c - 1] * p.x, a.delta[c - 1] * p.y)));
                }
                v = cmul(f, v);
            }
            return v;
        };
        auto readout = [&](const int *dc, double2 v) {  // rho(t_k) contribution of A_{k-1} entry v
            const int k = kb + i, last = i == 0 ? dx[kb - 1] : dc[i - 1];
            const double2 p = psi_of(k, 1, dc);
            double2 e[D];
#pragma unroll
            for (int d = 0; d < D; ++d) e[d] = cexp_(make_double2(a.delta[d] * p.x, a.delta[d] * p.y));
#pragma unroll
            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                for (int bb = 0; bb < M; ++bb) {
                    const int nw = aa * M + bb, c = class_of(M, LAT, aa, bb);
                    const double2 ft = c == 0 ? sK[1][nw][last] : cmul(sK[1][nw][last], e[c > 0 ? c - 1 : 0]);
                    acc[nw] = cfma(ft, v, acc[nw]);
                }
        };
        int dc[4];
        if (RO) {
            if (i == 0) {
                readout(dc, base);
            } else {
                long long np = 1;
                for (int t = 0; t < i; ++t) np *= N;
                for (int c = a.c_lo; c < a.c_lo + a.n_own && c < np; ++c) {
                    int r = c;
                    for (int t = 0; t < z; ++t) { dc[t] = r % N; r /= N; }
                    readout(dc, chain(dc, i));
                }
            }
        }
        if (i == z - 1)
            for (int b = 0; b < a.n_own; ++b) {
                int r = a.c_lo + b;
                for (int t = 0; t < z; ++t) { dc[t] = r % N; r /= N; }
                a.local[(long long)b * a.nb + x] = chain(dc, z);
            }
    }
    if (RO) reduce_finalize<N, 256>(acc, a.partials, a.rho, a.counter);
}

template <int M, bool LAT>
static cudaError_t grow_shard_t(const GrowShardArgs &a, int grid, cudaStream_t s) {
    if (a.rho) k_grow_shard<M, LAT, true><<<grid, 256, 0, s>>>(a);
    else k_grow_shard<M, LAT, false><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_grow_shard(int M, bool lattice, const GrowShardArgs &a, int grid, cudaStream_t s) {
    switch (M) {
    case 2: return grow_shard_t<2, false>(a, grid, s);
    case 3: return lattice ? grow_shard_t<3, true>(a, grid, s) : grow_shard_t<3, false>(a, grid, s);
    case 4: return lattice ? grow_shard_t<4, true>(a, grid, s) : grow_shard_t<4, false>(a, grid, s);
    default: return cudaErrorInvalidValue;
    }
}

// Cross-rank readout (multi-GPU): parts[g][o][n] are the ranks' rho(t_k) of output o in rank order
// (gathered by the caller); rho[o][n] = parts[0][o][n] for outputs complete on every rank (step
// k <= L - z: replicated growth), else the sum over g = 0..G-1 in rank order (deterministic).
__global__ void k_shard_combine(const double2 *parts, double2 *rho, const long long *steps, long long n_out, int N,
                                int G, long long k_rep) {
    const long long n = n_out * N;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        double2 s = parts[t];
        if (steps[t / N] > k_rep)
            for (int g = 1; g < G; ++g) s = cadd(s, parts[(long long)g * n + t]);
        rho[t] = s;
    }
}

cudaError_t launch_shard_combine(const double2 *parts, double2 *rho, const long long *steps, long long n_out, int N, int G,
                                 long long k_rep, cudaStream_t s) {
    if (n_out <= 0) return cudaSuccess;
    const int grid = (int)std::min<long long>((n_out * N + 255) / 256, 1024);
    k_shard_combine<<<grid, 256, 0, s>>>(parts, rho, steps, n_out, N, G, k_rep);
    return cudaGetLastError();
}

// ============================================================================================
// Re-shard data movement (multi-GPU path): one digit-permutation copy.  The dense
// side index i is a mixed-radix number: nd base-N digit fields (innermost first, division by the
// compile-time N), then up to two combo fields of radix crad[c] whose value v is either a linear
// field (cnd = 0: v * cstr[c][0]) or the base-N digits of (clo + v) with strides cstr[c][0..cnd-1].
// gather: dst[i] = src[addr(i)];  scatter: dst[addr(i)] = src[i].  No runtime 64-bit division.
// ============================================================================================

// One thread per row = the N entries of the innermost digit field: the dense side is contiguous
// (32-byte vector accesses), the strided side steps by dstr[0] (also 32-byte pairs when dstr[0] == 1);
// the row's strided address is decomposed once per N entries.
template <int N>
__global__ void __launch_bounds__(256) k_permute(const __grid_constant__ PermuteArgs a) {
    const long long rows = a.count / N;
    const long long stride = (long long)gridDim.x * 256;
    const long long s0 = a.dstr[0];
    for (long long row = (long long)blockIdx.x * 256 + threadIdx.x; row < rows; row += stride) {
        long long addr = 0;
        unsigned long long rest = (unsigned long long)row;
        for (int f = 1; f < a.nd; ++f) {
            const unsigned long long q = rest / N;  // compile-time N: multiply-high / shift
            addr += (long long)(rest - q * N) * a.dstr[f];
            rest = q;
        }
        unsigned r32 = (unsigned)rest;  // combo fields: < 2^32 (checked on the host)
        for (int c = 0; c < a.ncombo; ++c) {
            const unsigned v = r32 % (unsigned)a.crad[c];
            r32 /= (unsigned)a.crad[c];
            if (a.cnd[c] == 0) {
                addr += (long long)v * a.cstr[c][0];
            } else {
                unsigned cc = (unsigned)a.clo[c] + v;
                for (int t = 0; t < a.cnd[c]; ++t) {
                    addr += (long long)(cc % N) * a.cstr[c][t];
                    cc /= N;
                }
            }
        }
        const long long dense = row * N;
        if constexpr (N % 2 == 0) {
            if (s0 == 1) {  // both sides contiguous along the row
                const double2 *src = a.src + (a.scatter ? dense : addr);
                double2 *dst = a.dst + (a.scatter ? addr : dense);
#pragma unroll
                for (int v = 0; v < N; v += 2) {
                    double2 x, y;
                    ld2_cs(src + v, x, y);
                    st2_cs(dst + v, x, y);
                }
                continue;
            }
            double2 buf[N];
            if (a.scatter) {
#pragma unroll
                for (int v = 0; v < N; v += 2) ld2_cs(a.src + dense + v, buf[v], buf[v + 1]);
#pragma unroll
                for (int v = 0; v < N; ++v) __stcs(a.dst + addr + v * s0, buf[v]);
            } else {
#pragma unroll
                for (int v = 0; v < N; ++v) buf[v] = __ldcs(a.src + addr + v * s0);
#pragma unroll
                for (int v = 0; v < N; v += 2) st2_cs(a.dst + dense + v, buf[v], buf[v + 1]);
            }
        } else {
#pragma unroll
            for (int v = 0; v < N; ++v) {
                if (a.scatter) __stcs(a.dst + addr + v * s0, __ldcs(a.src + dense + v));
                else __stcs(a.dst + dense + v, __ldcs(a.src + addr + v * s0));
            }
        }
    }
}

cudaError_t launch_permute(int M, const PermuteArgs &a, int sms, cudaStream_t s) {
    if (a.count <= 0) return cudaSuccess;
    if (a.nd < 1 || a.count % (M * M)) return cudaErrorInvalidValue;  // rows of the innermost digit field
    const int grid = (int)std::min<long long>((a.count / (M * M) + 255) / 256, (long long)sms * 16);
    switch (M) {
    case 2: k_permute<4><<<grid, 256, 0, s>>>(a); break;
    case 3: k_permute<9><<<grid, 256, 0, s>>>(a); break;
    case 4: k_permute<16><<<grid, 256, 0, s>>>(a); break;
    default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace qp
