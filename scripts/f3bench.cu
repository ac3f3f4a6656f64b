// f3bench.cu -- access-pattern microbenchmark for k_fused3 (not product code).
// Reproduces k_fused3's HBM access pattern on a 4^14 complex FP64 array: three inner digits at ring
// positions p, p+1, p+2 (mod 14), tiles of 4^5 outer fibres (lowest outer digits), one round =
// 8 W outer fibres, lane (j, t8) loads the 16 entries (d0, d1) with digit 2 = j, then `work`
// dependent FP64 FMAs per entry (a stand-in for the three fused steps), then stores them back.
// Prints GB/s (2 x 16 B per entry) per (p, work, block).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f3bench scripts/f3bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("cuda %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

struct Args {
    double2 *A;
    const int *lofs;          // [T] tile-local offsets
    const long long *toff;    // [n_tiles] tile offsets
    long long pw0, pw1, pw2;  // inner strides
    int T, n_tiles, work, mode, inter;
};

template <int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_pat(const Args a) {
    constexpr int W = BLOCK / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, j = lane >> 3, t8 = lane & 7;
    const int per = a.n_tiles / gridDim.x, rem = a.n_tiles % gridDim.x;
    const int tb = blockIdx.x * per + min((int)blockIdx.x, rem), te = tb + per + ((int)blockIdx.x < rem);
    const int rounds = (a.T + 8 * W - 1) / (8 * W);
    const int nmine = a.inter ? (a.n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : te - tb;
    for (int it_ = 0; it_ < nmine; ++it_) {
        const int tau = a.inter ? blockIdx.x + it_ * gridDim.x : tb + it_;
        const long long tbase = a.toff[tau];
        for (int rd = 0; rd < rounds; ++rd) {
            // mode 0: lane = (j, t8), 8 fibres per warp; mode 1: lane = t (32 fibres), warp -> j
            const int t = a.mode == 0 ? rd * 8 * W + warp * 8 + t8 : rd * 8 * W + (warp >> 2) * 32 + lane;
            const int jj = a.mode == 0 ? j : (warp & 3);
            if (t >= a.T) continue;
            const long long base = tbase + a.lofs[t] + jj * a.pw2;
            double2 X[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) X[e] = __ldcs(a.A + base + (e & 3) * a.pw0 + (e >> 2) * a.pw1);
            for (int it = 0; it < a.work; ++it)
#pragma unroll
                for (int e = 0; e < 16; ++e) X[e] = make_double2(fma(X[e].x, 0.999, 1e-9), fma(X[e].y, 0.999, -1e-9));
#pragma unroll
            for (int e = 0; e < 16; ++e) __stcs(a.A + base + (e & 3) * a.pw0 + (e >> 2) * a.pw1, X[e]);
        }
    }
}

static long long ipow4(int e) { return 1LL << (2 * e); }

int main(int argc, char **argv) {
    const int L = 14;
    const long long n = ipow4(L);
    double2 *A;
    CK(cudaMalloc(&A, n * 16));
    CK(cudaMemset(A, 0, n * 16));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int *dl;
    long long *dt;
    CK(cudaMalloc(&dl, 1024 * 4));
    CK(cudaMalloc(&dt, 4096 * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int p = 0; p < 14; ++p) {
        int in[3] = {p % L, (p + 1) % L, (p + 2) % L};
        std::vector<int> outer;
        for (int q = 0; q < L; ++q)
            if (q != in[0] && q != in[1] && q != in[2]) outer.push_back(q);
        std::vector<int> lofs(1024);
        std::vector<long long> toff(4096);
        for (int t = 0; t < 1024; ++t) {
            long long o = 0;
            for (int d = 0; d < 5; ++d) o += (long long)((t >> (2 * d)) & 3) * ipow4(outer[d]);
            lofs[t] = (int)o;
        }
        for (int x = 0; x < 4096; ++x) {
            long long o = 0;
            for (int d = 0; d < 6; ++d) o += (long long)((x >> (2 * d)) & 3) * ipow4(outer[5 + d]);
            toff[x] = o;
        }
        CK(cudaMemcpy(dl, lofs.data(), 1024 * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dt, toff.data(), 4096 * 8, cudaMemcpyHostToDevice));
        Args a{A, dl, dt, ipow4(in[0]), ipow4(in[1]), ipow4(in[2]), 1024, 4096, 0, 0, 0};
        for (int cfg : {0, 1, 2, 3}) {
            a.mode = cfg & 1;
            a.inter = cfg >> 1;
            const int work = 0;
            auto run = [&](auto kern, int block, int occ) {
                kern<<<sms * occ, block>>>(a);
                CK(cudaDeviceSynchronize());
                cudaEventRecord(e0);
                for (int r = 0; r < 5; ++r) kern<<<sms * occ, block>>>(a);
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                ms /= 5;
                printf("p=%2d work=%2d mode=%d inter=%d block=%d x%d: %.3f ms  %.0f GB/s\n", p, work, a.mode, a.inter, block, occ, ms, 2.0 * n * 16 / ms / 1e6);
            };
            run(k_pat<256, 2>, 256, 2);
        }
    }
    return 0;
}
