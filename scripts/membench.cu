// membench.cu -- calibration microbenchmarks for the slide kernel's roofline (not product code).
//   copy      : B = A            (the MEASURED_PEAKS "hbm copy" pattern, 16-B vectors)
//   inplace   : A = c * A        (in-place read-modify-write, what k_slide does per element)
//   fibre p   : the k_slide access pattern (N=4 values at stride 4^p per thread) with a
//               trivial complex scale, no factor tables -- the memory-only ceiling per ring slot
//   dfma      : FP64 FMA issue rate (independent chains), for the FP64 ridge point
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench scripts/membench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_copy(const double2 *__restrict__ a, double2 *__restrict__ b, long long n) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    for (; i + 3 * st < n; i += 4 * st) {
        double2 x0 = a[i], x1 = a[i + st], x2 = a[i + 2 * st], x3 = a[i + 3 * st];
        b[i] = x0; b[i + st] = x1; b[i + 2 * st] = x2; b[i + 3 * st] = x3;
    }
    for (; i < n; i += st) b[i] = a[i];
}

__global__ void k_inplace(double2 *a, long long n, double c) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
    for (; i + 3 * st < n; i += 4 * st) {
        double2 x0 = __ldcs(a + i), x1 = __ldcs(a + i + st), x2 = __ldcs(a + i + 2 * st), x3 = __ldcs(a + i + 3 * st);
        __stcs(a + i, make_double2(c * x0.x, c * x0.y));
        __stcs(a + i + st, make_double2(c * x1.x, c * x1.y));
        __stcs(a + i + 2 * st, make_double2(c * x2.x, c * x2.y));
        __stcs(a + i + 3 * st, make_double2(c * x3.x, c * x3.y));
    }
    for (; i < n; i += st) { double2 x = a[i]; a[i] = make_double2(c * x.x, c * x.y); }
}

// fibre pattern: fibre f -> lo = f mod 4^p, hi = f / 4^p; entries lo + v 4^p + hi 4^(p+1)
template <int F>
__global__ void k_fibre(double2 *a, long long nfib, int p, double c) {
    const long long pw = 1LL << (2 * p);
    long long f0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x), st = (long long)gridDim.x * blockDim.x;
    for (long long f = f0; f < nfib; f += F * st) {
        double2 x[F][4];
        long long base[F];
#pragma unroll
        for (int j = 0; j < F; ++j) {
            long long g = f + j * st;
            base[j] = (g & (pw - 1)) + (g >> (2 * p)) * (pw << 2);
            if (g < nfib)
#pragma unroll
                for (int v = 0; v < 4; ++v) x[j][v] = __ldcs(a + base[j] + v * pw);
        }
#pragma unroll
        for (int j = 0; j < F; ++j) {
            long long g = f + j * st;
            if (g < nfib) {
                double2 s = make_double2(x[j][0].x + x[j][1].x + x[j][2].x + x[j][3].x, x[j][0].y + x[j][1].y + x[j][2].y + x[j][3].y);
#pragma unroll
                for (int v = 0; v < 4; ++v) __stcs(a + base[j] + v * pw, make_double2(c * s.x + x[j][v].x, c * s.y + x[j][v].y));
            }
        }
    }
}

__global__ void k_dfma(double *out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long n = 1LL << 28;  // 4^14 complex = 4.3 GB
    double2 *a, *b;
    CK(cudaMalloc(&a, n * 16));
    CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    CK(cudaMemset(b, 0, n * 16));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn, int reps) {
        fn();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms / reps;
    };
    for (int occ : {4, 8, 16}) {
        float ms = timeit([&] { k_copy<<<sms * occ, 256>>>(a, b, n); }, 10);
        printf("copy     grid=%d*%d: %.3f ms  %.1f GB/s\n", sms, occ, ms, 2.0 * n * 16 / ms / 1e6);
    }
    for (int occ : {4, 8, 16}) {
        float ms = timeit([&] { k_inplace<<<sms * occ, 256>>>(a, n, 0.5); }, 10);
        printf("inplace  grid=%d*%d: %.3f ms  %.1f GB/s\n", sms, occ, ms, 2.0 * n * 16 / ms / 1e6);
    }
    for (int p : {0, 1, 2, 3, 6, 13}) {
        for (int occ : {4, 8}) {
            float ms = timeit([&] { k_fibre<2><<<sms * occ, 256>>>(a, n / 4, p, 0.1); }, 10);
            printf("fibre p=%2d F=2 grid=%d*%d: %.3f ms  %.1f GB/s\n", p, sms, occ, ms, 2.0 * n * 16 / ms / 1e6);
        }
        float ms = timeit([&] { k_fibre<4><<<sms * 4, 256>>>(a, n / 4, p, 0.1); }, 10);
        printf("fibre p=%2d F=4 grid=%d*4: %.3f ms  %.1f GB/s\n", p, sms, ms, 2.0 * n * 16 / ms / 1e6);
    }
    double *o;
    CK(cudaMalloc(&o, sms * 8 * 256 * 8));
    const int iters = 1 << 16;
    float ms = timeit([&] { k_dfma<<<sms * 8, 256>>>(o, iters); }, 3);
    const double fl = 2.0 * 8 * iters * (double)sms * 8 * 256;
    printf("dfma: %.3f ms  %.2f TFLOP/s FP64 (%.1f DFMA/clk/SM at 1.965 GHz)\n", ms, fl / ms / 1e9,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    return 0;
}
