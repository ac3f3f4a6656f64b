// qp_internal.h -- structures shared by the host setup (host.cpp) and the sm_100a kernels
// (kernels.cu).  Not part of the public ABI (include/quapi.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qp {

constexpr int kMaxM = 4;
constexpr int kMaxN = kMaxM * kMaxM;
constexpr int kMaxD = kMaxM * (kMaxM - 1);
constexpr int kMaxL = 40;
constexpr int kMaxGroups = 8;
constexpr int kPartialsMax = 4096;  // max CTAs contributing readout partials

// Number of nonzero Delta-s classes used by the kernels.
//   lattice (s_a = s_0 + a u):  class of (a,b) is a-b in {+-1..+-(M-1)}   -> D = 2(M-1)
//   general:                    every ordered off-diagonal pair (a,b)       -> D = M(M-1)
__host__ __device__ constexpr int n_classes(int M, bool lattice) { return lattice ? 2 * (M - 1) : M * (M - 1); }

// Class index of pair state sigma = (a, b): 0 for a == b (Delta s = 0 rows share the plain sum),
// else 1..D.  Must agree with the host's delta[] table (host.cpp: build_classes).
__host__ __device__ constexpr int class_of(int M, bool lattice, int a, int b) {
    return a == b ? 0
                  : (lattice ? (a > b ? a - b : (M - 1) + (b - a))
                             : 1 + a * (M - 1) + (b < a ? b : b - 1));
}

// Offsets (in double2 units) inside the per-plan "small" table block.
struct SmallLayout {
    int N, D, L;
    __host__ __device__ int kp(int kappa) const { return kappa * N * N; }                 // [2][N][N]: K'(new,last)
    __host__ __device__ int beta(int variant, int kappa) const {                          // [2][2][D][N]
        return 2 * N * N + (variant * 2 + kappa) * D * N;
    }
    __host__ __device__ int psi(int kappa) const { return 2 * N * N + 4 * D * N + kappa * L * L * N; }  // [2][L][L][N]
    __host__ __device__ int total() const { return 2 * N * N + 4 * D * N + 2 * L * L * N; }
};

// Per-launch arguments of the slide step (k >= L).  All tables are device pointers into d_work.
struct SlideArgs {
    double2 *A;              // ARDM, N^L entries, in place
    const double2 *small;    // SmallLayout block
    const double2 *Etab;     // E tables for this p: [kappa][g][d][X]
    const int2 *lofs;        // [T]: x = in-tile element offset of fibre f_local, y = 'last' digit or -1
    double2 *partials;       // [grid][N] readout block partials
    double2 *rho;            // [N] readout destination, nullptr => no readout this step
    unsigned *counter;       // last-block-done counter (reset by the last block)
    long long pw_p;          // N^p: stride of the contracted digit
    long long pw_p1;         // N^(p+1)
    long long tile_stride;   // p <  v: N^(v+1) elements per tile
    int n_tiles;             // N^(L-1-v)
    int T;                   // fibres per tile = N^v
    int p_ge_v;              // 1 if every tile digit lies below p
    int Qlo;                 // p >= v: N^(p-v) tiles share one hi block
    int G;                   // number of digit groups (group 0 = tile-local digits)
    int X;                   // entries per group table (padded)
    int gdiv[kMaxGroups];    // group g >= 1: index = (tau / gdiv[g]) % gmod[g]
    int gmod[kMaxGroups];
    int last_div;            // 'last' digit is a tile digit: (tau / last_div) % N; else -1
    int variant;             // 0 steady (k > L), 1 first slide (k == L)
};

// Per-launch arguments of the growth step k (1 <= k < L): A_{k-1} (N^k) -> A_k (N^(k+1)).
struct GrowArgs {
    double2 *A;
    const double2 *small;
    double2 *partials;
    double2 *rho;
    unsigned *counter;
    long long n_in;          // N^k
    int k;
    int L;
    double delta[kMaxD];     // Delta s of each class (index d-1)
};

// Slide-kernel variant: launch shape and pipelining (kernels.cu registry).
struct SlideVariant {
    int id, M, block, F, v, w, minb, prefetch, stages;  // stages > 0 => TMA-staged kernel
};
const SlideVariant *find_variant(int id);
int default_variant(int M);
// Launchers (kernels.cu).  Return cudaError_t of the launch.
cudaError_t launch_slide(int variant, bool lattice, const SlideArgs &a, int grid, cudaStream_t s);
int slide_occupancy(int variant, bool lattice, int T);  // resident CTAs per SM (needs a device)
cudaError_t launch_grow(int M, bool lattice, const GrowArgs &a, int grid, cudaStream_t s);

}  // namespace qp
