// common.cuh -- device helpers shared by the sm_100a slide / growth / re-shard kernels
// (slide_r.cu, slide3.cu, grow.cu): complex FP64 arithmetic, the fixed-order readout reduction,
// super-fibre index helpers and the TMA / mbarrier / 256-bit load-store PTX wrappers.
#pragma once
#include "qp_internal.h"

namespace qp {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // a*b + c
    return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cexp_(double2 z) {
    double e = exp(z.x), s, c;
    sincos(z.y, &s, &c);
    return make_double2(e * c, e * s);
}

__host__ __device__ constexpr int cpow(int b, int e) { return e == 0 ? 1 : b * cpow(b, e - 1); }

// Fixed-order CTA reduction of N complex per-thread values into partials[blockIdx][N] (shuffle tree
// per warp, then the warps in order).
// dst: this CTA's row (partials + blockIdx.x * N), or rho itself when the grid is one CTA.
template <int N, int BLOCK>
__device__ __forceinline__ void reduce_block_to(double2 (&acc)[N], double2 *dst) {
    constexpr int W = BLOCK / 32;
    __shared__ double2 red[W][N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();  // red may be reused by consecutive calls
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
        __stcg(&dst[threadIdx.x], s);
    }
}

// One CTA sums partials[0..nblk)[N] in fixed order into rho[N] (accumulate: rho[n] += sum).  Thread t
// takes the blocks b = t, t + BLOCK, ... with all N loads of a block (and of 4 blocks) in flight, then
// the per-thread sums go through the CTA tree of reduce_block_to's shape.
template <int N, int BLOCK>
__device__ __forceinline__ void reduce_partials_sum(const double2 *partials, int nblk, double2 *rho, bool accumulate) {
    constexpr int W = BLOCK / 32;
    __shared__ double2 red2[W][N];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double2 s[N];
#pragma unroll
    for (int n = 0; n < N; ++n) s[n] = make_double2(0.0, 0.0);
    int b = threadIdx.x;
    for (; b + 3 * BLOCK < nblk; b += 4 * BLOCK) {
        double2 v[4][N];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int n = 0; n < N; ++n) v[i][n] = __ldcg(&partials[(size_t)(b + i * BLOCK) * N + n]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int n = 0; n < N; ++n) s[n] = cadd(s[n], v[i][n]);
    }
    for (; b < nblk; b += BLOCK)
#pragma unroll
        for (int n = 0; n < N; ++n) s[n] = cadd(s[n], __ldcg(&partials[(size_t)b * N + n]));
    __syncthreads();  // red2 may be reused by consecutive calls
#pragma unroll
    for (int n = 0; n < N; ++n) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s[n].x += __shfl_xor_sync(0xffffffffu, s[n].x, o);
            s[n].y += __shfl_xor_sync(0xffffffffu, s[n].y, o);
        }
        if (lane == 0) red2[warp][n] = s[n];
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double2 t = red2[0][threadIdx.x];
        for (int w = 1; w < W; ++w) t = cadd(t, red2[w][threadIdx.x]);
        rho[threadIdx.x] = accumulate ? cadd(rho[threadIdx.x], t) : t;
    }
}

// Fixed-order reduction of N complex per-thread values over the grid: block partials, then the last
// CTA to finish sums them (deterministic: the grid and the tile -> CTA assignment are fixed by the
// plan).  accumulate: rho[n] += sum.
template <int N, int BLOCK>
__device__ __forceinline__ void reduce_finalize(double2 (&acc)[N], double2 *partials, double2 *rho,
                                                unsigned *counter, bool accumulate = false) {
    __shared__ int is_last;
    reduce_block_to<N, BLOCK>(acc, partials + (size_t)blockIdx.x * N);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    reduce_partials_sum<N, BLOCK>(partials, (int)gridDim.x, rho, accumulate);
    if (threadIdx.x == 0) *counter = 0u;
}

// Fixed-order grid reduction of NV complex values per thread in ONE pass (several readouts of one
// launch together): shuffle tree per warp, warps in order into partials[blockIdx][NV], one counter;
// the last CTA to finish sums the block rows in block order (b = t, t + BLOCK, ... per thread, then the
// same trees) and calls put(v, total) for v < NV.  red: shared scratch of (BLOCK / 32) * NV entries.
template <int NV, int BLOCK, class Put>
__device__ __forceinline__ void grid_sum_multi(double2 (&v)[NV], double2 *red, double2 *partials, unsigned *counter, Put put) {
    constexpr int W = BLOCK / 32;
    __shared__ int is_last_m;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto tree = [&]() {  // v -> red[warp][n] (lane 0), fixed shuffle order
#pragma unroll
        for (int n = 0; n < NV; ++n) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v[n].x += __shfl_xor_sync(0xffffffffu, v[n].x, o);
                v[n].y += __shfl_xor_sync(0xffffffffu, v[n].y, o);
            }
            if (lane == 0) red[warp * NV + n] = v[n];
        }
        __syncthreads();
    };
    auto warps_sum = [&](int t) {
        double2 s = red[t];
        for (int w = 1; w < W; ++w) s = cadd(s, red[w * NV + t]);
        return s;
    };
    __syncthreads();  // red may alias memory the caller used
    tree();
    if (threadIdx.x < NV) __stcg(&partials[(size_t)blockIdx.x * NV + threadIdx.x], warps_sum(threadIdx.x));
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last_m = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last_m) return;
    __threadfence();
#pragma unroll
    for (int n = 0; n < NV; ++n) v[n] = make_double2(0.0, 0.0);
    for (int b = threadIdx.x; b < (int)gridDim.x; b += BLOCK)
#pragma unroll
        for (int n = 0; n < NV; ++n) v[n] = cadd(v[n], __ldcg(&partials[(size_t)b * NV + n]));
    __syncthreads();  // red: every thread has read its block sums above
    tree();
    if (threadIdx.x < NV) put(threadIdx.x, warps_sum(threadIdx.x));
    if (threadIdx.x == 0) *counter = 0u;
}

// Super-fibre index helpers.  A super-fibre holds the N^S entries of the S inner digits of one
// outer fibre, entry e = sum_i d_i N^i.  During sub-step s a "fibre" is the N entries along inner
// digit s; r enumerates the other S-1 inner digits (ascending, digit s skipped).
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

// ---- cp.async (LDGSTS) 16-byte copies global -> shared
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NPEND> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(NPEND) : "memory");
}

// ---- TMA (cp.async.bulk / cp.async.bulk.tensor) + mbarrier + 256-bit streaming access (sm_100a PTX)
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

}  // namespace qp
