// ofpf.cu -- path-filtered propagation: Sim's on-the-fly filtering of paths, which the
// paper cites as the way to cut the memory of the tensor propagator, notes its program
// does not do and invites.  Reading C.3-15: after every step
// k >= 1 the entries of A_k with |A|^2 < theta^2 are dropped; rho(t_k) is read from A_{k-1}.
//
// The ARDM is a compacted list of (key, value) of the surviving entries, sorted by key.  Before step
// k the key puts the digit the step works on in the right place:
//   growth k < L : key = x = sum_{q<k} sigma_q N^q; the step appends digit k (most significant);
//   slide  k >= L: key = sum_i d_i N^i with d_i the value of ring slot (k + i) mod L, i.e. the point
//                  sigma_{k-L+i} (partner at lag L - i); d_0 is summed out, the new point becomes
//                  digit L-1: new key = key / N + new N^(L-1).
// A group is one entry (growth) or the <= N entries of one fibre (same key / N, slide).  Every group
// yields N outputs, one per value `new` of the added digit, in key order inside each value, so bucketing
// the outputs by `new` (most significant digit of the new key) keeps the list sorted.  A step is
//   A: count   -- per group the outputs and their keep flags, per block and bucket the count of
//                 survivors; the fused readout rho(t_k) (fixed-order block reduction);
//   B: scan    -- bucket-major exclusive scan of the block counts (one CTA): output offsets;
//   C: scatter -- recompute the outputs (same arithmetic), write the survivors at their offsets.
// Every block owns a contiguous chunk of the list (the grid is fixed by the plan), so the output
// order and the readout are deterministic.  HBM traffic per step ~ 2 x 24 B per kept entry.
#include "common.cuh"

namespace qp {

namespace {
constexpr int kOfpfBlock = 256;

struct Group {       // the entries of one group, missing values are 0
    double2 v[kMaxN];
    long long gkey;  // key / N (slide) or key (growth)
};

template <int M, bool LAT>
struct OfpfMath {
    static constexpr int N = M * M, D = n_classes(M, LAT);
    // outputs out[new] (kap 0) and the readout terms (kap 1) of one group at step k
    __device__ static void eval(const OfpfArgs &a, const Group &g, double2 (&out)[N], double2 (&ro)[N], bool want_ro) {
        const SmallLayout lay{N, D, a.L};
        double2 psi0 = make_double2(0.0, 0.0), psi1 = psi0;
        int last;
        long long r = g.gkey;
        if (a.slide) {  // gkey digit i (i = 0..L-2) is the point at lag L - 1 - i
            for (int i = 0; i < a.L - 1; ++i) {
                const int d = (int)(r % N);
                r /= N;
                const int lag = a.L - 1 - i;
                psi0 = cadd(psi0, __ldg(&a.tab[(0 * (kMaxL + 1) + lag) * N + d]));
                psi1 = cadd(psi1, __ldg(&a.tab[(1 * (kMaxL + 1) + lag) * N + d]));
                if (i == a.L - 2) last = d;
            }
        } else {  // growth k: digit q holds sigma_q, lag k - q
            for (int q = 0; q < a.k; ++q) {
                const int d = (int)(r % N);
                r /= N;
                const int j = a.k - q;
                psi0 = cadd(psi0, __ldg(&a.small[lay.psi(0) + ((size_t)a.k * a.L + j) * N + d]));
                psi1 = cadd(psi1, __ldg(&a.small[lay.psi(1) + ((size_t)a.k * a.L + j) * N + d]));
                if (q == a.k - 1) last = d;
            }
        }
        double2 e0[D], e1[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            e0[d] = cexp_(make_double2(a.delta[d] * psi0.x, a.delta[d] * psi0.y));
            e1[d] = want_ro ? cexp_(make_double2(a.delta[d] * psi1.x, a.delta[d] * psi1.y)) : make_double2(0.0, 0.0);
        }
        // moments of the contracted digit (slide) or the single value (growth)
        double2 S0 = make_double2(0.0, 0.0), m0[D], m1[D];
        if (a.slide) {
#pragma unroll
            for (int v = 0; v < N; ++v) S0 = cadd(S0, g.v[v]);
#pragma unroll
            for (int d = 0; d < D; ++d) {
                double2 x0 = make_double2(0.0, 0.0), x1 = x0;
#pragma unroll
                for (int v = 0; v < N; ++v) {
                    x0 = cfma(__ldg(&a.small[lay.beta(a.var, 0) + d * N + v]), g.v[v], x0);
                    if (want_ro) x1 = cfma(__ldg(&a.small[lay.beta(a.var, 1) + d * N + v]), g.v[v], x1);
                }
                m0[d] = x0, m1[d] = x1;
            }
        } else {
            S0 = g.v[0];
#pragma unroll
            for (int d = 0; d < D; ++d) m0[d] = m1[d] = g.v[0];
        }
#pragma unroll
        for (int aa = 0; aa < M; ++aa)
#pragma unroll
            for (int bb = 0; bb < M; ++bb) {
                const int nw = aa * M + bb, c = class_of(M, LAT, aa, bb);
                const double2 k0 = __ldg(&a.small[lay.kp(0) + nw * N + last]);
                out[nw] = cmul(k0, c == 0 ? S0 : cmul(e0[c > 0 ? c - 1 : 0], m0[c > 0 ? c - 1 : 0]));
                if (want_ro) {
                    const double2 k1 = __ldg(&a.small[lay.kp(1) + nw * N + last]);
                    ro[nw] = cmul(k1, c == 0 ? S0 : cmul(e1[c > 0 ? c - 1 : 0], m1[c > 0 ? c - 1 : 0]));
                }
            }
    }
};

__device__ __forceinline__ bool keep(double2 z, double th2) {  // |z|^2 >= theta^2, no FMA (oracle: -ffp-contract=off)
    return __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y)) >= th2;
}

// the group headed by list entry i (or none: i is not a head)
template <int N>
__device__ __forceinline__ bool load_group(const OfpfArgs &a, long long i, long long n, Group &g) {
    const long long key = a.key_in[i];
    const long long gk = a.slide ? key / N : key;
    if (i > 0) {
        const long long kp = a.key_in[i - 1];
        if ((a.slide ? kp / N : kp) == gk) return false;
    }
#pragma unroll
    for (int v = 0; v < N; ++v) g.v[v] = make_double2(0.0, 0.0);
    g.gkey = gk;
    if (!a.slide) {
        g.v[0] = a.val_in[i];
        return true;
    }
    for (long long j = i; j < n && j < i + N; ++j) {
        const long long kj = a.key_in[j];
        if (kj / N != gk) break;
        g.v[kj % N] = a.val_in[j];
    }
    return true;
}

__device__ __forceinline__ void chunk_of(long long n, long long &lo, long long &hi) {
    const long long ch = (n + gridDim.x - 1) / gridDim.x;
    lo = min(n, (long long)blockIdx.x * ch);
    hi = min(n, lo + ch);
}
}  // namespace

// A: outputs' keep flags, per-block bucket counts, readout
template <int M, bool LAT, bool RO>
__global__ void __launch_bounds__(kOfpfBlock) k_ofpf_count(const __grid_constant__ OfpfArgs a) {
    constexpr int N = M * M;
    __shared__ int cnt[N];
    if (*a.overflow) return;  // an earlier step overflowed: nothing to do (uniform over the grid)
    if (threadIdx.x < N) cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long n = *a.n_in;
    long long lo, hi;
    chunk_of(n, lo, hi);
    double2 acc[N];
#pragma unroll
    for (int v = 0; v < N; ++v) acc[v] = make_double2(0.0, 0.0);
    for (long long i = lo + threadIdx.x; i < hi; i += kOfpfBlock) {
        Group g;
        unsigned fl = 0;
        if (load_group<N>(a, i, n, g)) {
            double2 out[N], ro[N];
            OfpfMath<M, LAT>::eval(a, g, out, ro, RO);
#pragma unroll
            for (int v = 0; v < N; ++v) {
                if (keep(out[v], a.th2)) fl |= 1u << v;
                if (RO) acc[v] = cadd(acc[v], ro[v]);
            }
        }
        a.flags[i] = (unsigned short)fl;
#pragma unroll
        for (int v = 0; v < N; ++v)
            if (fl >> v & 1u) atomicAdd(&cnt[v], 1);  // integer counts: order-independent
    }
    __syncthreads();
    if (threadIdx.x < N) a.blkcnt[(size_t)blockIdx.x * N + threadIdx.x] = cnt[threadIdx.x];
    if (RO) reduce_finalize<N, kOfpfBlock>(acc, a.partials, a.rho, a.counter);
}

// B: bucket-major exclusive scan of the block counts (one CTA)
__global__ void k_ofpf_scan(const int *blkcnt, long long *blkbase, int nblk, int N, long long *n_out, long long cap,
                            long long *kept, int *overflow) {
    __shared__ long long tot[kMaxN];
    if ((int)threadIdx.x < N) {
        long long s = 0;
        for (int b = 0; b < nblk; ++b) s += blkcnt[(size_t)b * N + threadIdx.x];
        tot[threadIdx.x] = s;
    }
    __syncthreads();
    if ((int)threadIdx.x < N) {
        long long run = 0;
        for (int v = 0; v < (int)threadIdx.x; ++v) run += tot[v];
        for (int b = 0; b < nblk; ++b) {
            blkbase[(size_t)b * N + threadIdx.x] = run;
            run += blkcnt[(size_t)b * N + threadIdx.x];
        }
    }
    if (threadIdx.x == 0) {
        long long s = 0;
        for (int v = 0; v < N; ++v) s += tot[v];
        *kept = s;
        if (s > cap || *overflow) {  // the list outgrew the buffer: the run stops here (host reports the step)
            *overflow = 1;
            s = 0;
        }
        *n_out = s;
    }
}

// C: survivors to their offsets, in order
template <int M, bool LAT>
__global__ void __launch_bounds__(kOfpfBlock) k_ofpf_scatter(const __grid_constant__ OfpfArgs a) {
    constexpr int N = M * M, W = kOfpfBlock / 32;
    __shared__ long long run[N];
    __shared__ int wsum[W][N];
    if (*a.overflow) return;
    const long long n = *a.n_in;
    long long lo, hi;
    chunk_of(n, lo, hi);
    if (threadIdx.x < N) run[threadIdx.x] = a.blkbase[(size_t)blockIdx.x * N + threadIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long topw = a.slide ? a.top : a.grow_w;  // N^(L-1) (slide) or N^k (growth): weight of the new digit
    for (long long base = lo; base < hi; base += kOfpfBlock) {
        const long long i = base + threadIdx.x;
        unsigned fl = 0;
        Group g;
        double2 out[N], ro[N];
        if (i < hi) {
            fl = a.flags[i];
            if (fl) {
                load_group<N>(a, i, n, g);
                OfpfMath<M, LAT>::eval(a, g, out, ro, false);
            }
        }
        unsigned below[N];
#pragma unroll
        for (int v = 0; v < N; ++v) {
            const unsigned bal = __ballot_sync(0xffffffffu, (fl >> v) & 1u);
            below[v] = __popc(bal & ((1u << lane) - 1u));
            if (lane == 0) wsum[warp][v] = __popc(bal);
        }
        __syncthreads();
        if (i < hi && fl) {
#pragma unroll
            for (int v = 0; v < N; ++v)
                if (fl >> v & 1u) {
                    long long pos = run[v] + below[v];
                    for (int w = 0; w < warp; ++w) pos += wsum[w][v];
                    a.key_out[pos] = g.gkey + (long long)v * topw;
                    a.val_out[pos] = out[v];
                }
        }
        __syncthreads();
        if (threadIdx.x < N) {
            long long t = 0;
            for (int w = 0; w < W; ++w) t += wsum[w][threadIdx.x];
            run[threadIdx.x] += t;
        }
        __syncthreads();
    }
}

namespace {
template <int M, bool LAT>
cudaError_t ofpf_t(const OfpfArgs &a, int nblk, cudaStream_t s) {
    constexpr int N = M * M;
    if (a.rho) k_ofpf_count<M, LAT, true><<<nblk, kOfpfBlock, 0, s>>>(a);
    else k_ofpf_count<M, LAT, false><<<nblk, kOfpfBlock, 0, s>>>(a);
    k_ofpf_scan<<<1, 32, 0, s>>>(a.blkcnt, a.blkbase, nblk, N, a.n_out, a.cap, a.kept, a.overflow);
    k_ofpf_scatter<M, LAT><<<nblk, kOfpfBlock, 0, s>>>(a);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_ofpf_step(int M, bool lattice, const OfpfArgs &a, int nblk, cudaStream_t s) {
    switch (M) {
    case 2: return ofpf_t<2, false>(a, nblk, s);
    case 3: return lattice ? ofpf_t<3, true>(a, nblk, s) : ofpf_t<3, false>(a, nblk, s);
    case 4: return lattice ? ofpf_t<4, true>(a, nblk, s) : ofpf_t<4, false>(a, nblk, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace qp
