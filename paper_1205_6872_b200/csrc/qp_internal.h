// qp_internal.h -- structures shared by the host setup (host.cpp) and the sm_100a kernels
// (slide_r.cu, slide3.cu, grow.cu, batch.cu, eta.cu).  Not part of the public ABI (include/quapi.h).
#pragma once
#include <cuda.h>  // CUtensorMap (the encode entry point is fetched at run time; no -lcuda)
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

constexpr int kMaxS = 4;  // max steps fused into one launch (FusedArgs arrays)

// Per-launch arguments of the fused slide kernel: steps k..k+S-1 (k >= L) on the super-fibres of
// inner slots p0..p0+S-1 (mod L).  All tables are device pointers into d_work.
struct FusedArgs {
    double2 *A;              // ARDM, N^L entries, in place
    const double2 *small;    // SmallLayout block (K', beta)
    const double2 *inner;    // [S][S][2][D][N]: inner-slot factors per sub-step
    const double2 *Etab;     // [S][2][G][D][X]: outer digit-group factor tables per sub-step
    const double2 *E0r;      // k_fused3 TMA rounds: per round the group-0 factors [S][2][D][F] then the F
                             // tile-local offsets (int2), contiguous: one bulk copy per round; or nullptr
    const long long *goff;   // [G][X]: address offset of outer digit group g >= 1
    const int2 *lofs;        // [T]: x = address offset of tile-local fibre t, y = 'last' digit of sub-step 0 or -1
    double2 *partials;       // [kMaxS][kPartialsMax][N] readout block partials
    unsigned *counter;       // [kMaxS] last-block-done counters
    double2 *rho[kMaxS];     // readout destination per sub-step, nullptr => none
    long long pw_in[kMaxS];  // N^(slot of inner digit i)
    int n_tiles;             // N^(L-S-v)
    int T;                   // outer fibres per tile = N^v (<= block)
    int G;                   // digit groups (group 0 = tile-local)
    int X;                   // entries per group table (padded)
    int gdiv[kMaxGroups];    // group g >= 1: index = (tau / gdiv[g]) % gmod[g]
    int gmod[kMaxGroups];
    int last_div;            // sub-step 0 'last' digit is a tile digit: (tau / last_div) % N; else -1
    int fixed_last;          // sub-step 0 'last' slot is a (fixed) shard slot: its value; else -1
    int rho_accumulate;      // 1: rho[n] += sum (several shard blocks contribute to one step)
    int lane_map;            // k_fused3 plain loads: 1 when tile fibres t, t+1 are adjacent in HBM (slide3.cu)
    int use_tma;             // k_fused3: rounds staged per warp by TMA through `tmap` (unsharded launch sets)
    int tma_view;            // k_fused3 stage view: 0 = A, 1 = B, 2 = C, 3 = D (slide3.cu, host.cpp encode_f3_tmap)
    long long tma_nA;        // outer fibres in run A (slots 0 .. p0-1) of the TMA view (view B: 2, views C/D: 1)
    int tma_c0m;             // TMA coordinate 0 = tma_c0m x (G mod tma_nA) doubles, coordinate 1 = G / tma_nA
    int tma_nA_log2;         // log2(tma_nA) when tma_nA is a power of two (always for M = 2), else -1
    alignas(64) CUtensorMap tmap;   // k_fused3 / k_fused4 load map
    alignas(64) CUtensorMap tmapS;  // k_fused4 store map
    // k_fused4 stage layouts (slide4.cu, host.cpp f4_layout): smem bit position (16-B units) of each
    // box bit: 2 i + b = bit b of inner digit i, 8..10 = bits of the round's fibre index
    int f4_lpos[11], f4_spos[11];
    int f4_q1swap, f4_q2swap;  // lane mappings: phase 1 q = d2 + 4 d3 (0) or d3 + 4 d2 (1); phase 2 q = d0 + 4 d1 / d1 + 4 d0
    int f4_colregion;          // 1: the 8 fibres of a round are the 16-B chunks of each 128-B stage row (slot 0 outer)
    int f4_swz;                // 1: both maps use the 128-B swizzle (128-B inner box rows), 0: dense stage
    int f4_layout;             // k_fused4 instantiation with these layouts compiled in (1..3), 0: run-time layout
    int f4_cdimA[2], f4_cdimB[2];  // per map (load, store): box dims whose coordinate is tma_c0m (G mod tma_nA) / G / tma_nA
    int var[kMaxS];          // beta variant per sub-step: 1 for the first slide step k == L (initial-edge
                             // classes of the partner sigma_0), else 0 (SmallLayout::beta)
    // M = 2, s = (+s, -s): beta_1 = (c, rho, 1/rho, conj c); {Re c, Im c, (rho+1/rho)/2, (rho-1/rho)/2}
    double sym[kMaxS][2][4];
    // sharded layouts: factor of the fixed shard-slot digits of this block, per sub-step / kind / class
    double2 fixfac[kMaxS][2][kMaxD];
};


// Digit-permutation copy for the re-shard (grow.cu: k_permute): nd base-N digit fields, then up to
// two combo fields (radix crad, value lo + v as cnd base-N digits, or cnd = 0: linear stride).
constexpr int kMaxFields = kMaxL + 4;
struct PermuteArgs {
    double2 *dst;
    const double2 *src;
    long long count;         // dense-side entries
    int scatter;             // 0: dst[i] = src[addr(i)], 1: dst[addr(i)] = src[i]
    int nd;                  // digit fields, innermost first
    long long dstr[kMaxFields];
    int ncombo;
    int crad[2], clo[2], cnd[2];
    long long cstr[2][4];
};
cudaError_t launch_permute(int M, const PermuteArgs &a, int sms, cudaStream_t s);

// Sharded growth (grow.cu: k_grow_shard): step k = L - z + step from the replicated A_{L-z-1}.
struct GrowShardArgs {
    const double2 *Abase;    // A_{L-z-1}: N^(L-z) entries
    double2 *local;          // [n_own][N^(L-z)] (written by the last step)
    const double2 *small;
    double2 *partials;
    double2 *rho;            // readout of step k, or nullptr
    unsigned *counter;
    long long nb;            // N^(L-z)
    int L, z, step, n_own, c_lo;
    double delta[kMaxD];
};
cudaError_t launch_grow_shard(int M, bool lattice, const GrowShardArgs &a, int grid, cudaStream_t s);
cudaError_t launch_shard_combine(const double2 *parts, double2 *rho, const long long *steps, long long n_out, int N, int G,
                                 long long k_rep, cudaStream_t s);

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
cudaError_t launch_grow(int M, bool lattice, const GrowArgs &a, int grid, cudaStream_t s);

// Slide kernels.  k_fused_r (slide_r.cu): S <= 2 steps per pass, one thread per super-fibre, for
// (M, S) in {(2,1), (2,2), (3,1), (4,1)}.  k_fused3 (slide3.cu): M = 2, S = 3.
bool fused_r_has(int M, int S);
int fused_r_tile_digits(int M, int S);   // preferred v: T = N^v outer fibres per tile
int fused_r_block(int M, int S);
int fused_r_occupancy(int M, bool lattice, bool sym, int S);  // resident CTAs per SM (needs a device)
cudaError_t launch_fused_r(int M, bool lattice, bool sym, int S, const FusedArgs &a, bool ro, int grid, cudaStream_t s);
constexpr int kFused3TileDigits = 5, kFused3TileDigitsMin = 3;  // a round is 8 fibres x W warps
int fused3_block(int lane_map, bool tma);
int fused3_round_fibres(int lane_map, bool tma);  // outer fibres per round (8 per warp)
int fused3_occupancy(bool sym, int lane_map, bool tma);
cudaError_t launch_fused3(bool sym, const FusedArgs &a, bool ro, int grid, cudaStream_t s);
// k_fused2s (slide2.cu): M = 3, S = 2, shared-memory-staged units of 32 outer fibres
// k_small (persist.cu): all slide steps of one qp_steps call on a small ARDM in ONE launch of one
// CTA, the ARDM and every factor table staged in its shared memory, one step at a time.
struct PersistArgs {
    const FusedArgs *sets;   // device copy of the plan's launch-set arguments, index p0 * set_stride
    int set_stride;          // plan Smax (the S = 1 set of start slot p0 is sets[p0 * set_stride])
    double2 *A;              // ARDM
    const int *slot;         // [n_steps + 1]: readout slot of step k, -1 none
    double2 *rho_base;       // readout array [n_out][N]
    const double2 *small;    // SmallLayout block (K', beta)
    double sym[2][2][4];     // symmetric-moment constants per beta variant (FusedArgs::sym)
    long long k_begin, k_end;
    int L;
    const void *wbase;       // d_work: the tables [0, tables_bytes) are staged in shared memory
    long long tables_bytes, ardm_entries;
    int nsets;
};
constexpr int kPersistBlock = 256;
int small_static_smem(int M, bool lattice, bool sym);
cudaError_t launch_small(int M, bool lattice, bool sym, const PersistArgs &pa, size_t dyn, cudaStream_t s);

int fused2s_block();
int fused2s_occupancy(bool lattice);
// class weights beta of both sub-steps, passed by value (kernel parameter space: the moment loop takes
// them as constant-bank operands): [s][kap][d][old], copied from SmallLayout::beta(var[s], kap)
struct Beta2s {
    double2 b[2][2][kMaxM * (kMaxM - 1) < 6 ? kMaxM * (kMaxM - 1) : 6][9];
};
cudaError_t launch_fused2s(bool lattice, const FusedArgs &a, const Beta2s &b, bool ro, int grid, cudaStream_t s);
// k_fused2t (slide2t.cu): M = 3 lattice, S = 2, unsharded launch sets: TMA-staged 27-fibre units,
// warp-specialised (load / store / 2 x 9 consumer warps); a.f4_layout = view kind VK (0..3)
int fused2t_block();
int fused2t_unit_fibres();
int fused2t_e0_block();  // double2 entries of one unit's block: factors [S][2][D][27] + 27 int2 ('last')
int fused2t_occupancy();
cudaError_t launch_fused2t(const FusedArgs &a, const Beta2s &b, bool ro, int grid, cudaStream_t s);
// k_fused4 (slide4.cu): M = 2, S = 4, TMA load + store of 8-fibre rounds, warp-specialised
int fused4_block();
int fused4_round_fibres();
int fused4_e0_block();  // double2 entries of one round's E0 block
int fused4_occupancy(bool sym);
int fused4_layout_type(const int (&lpos)[11], const int (&spos)[11], int q1swap, int q2swap, int swz);
cudaError_t launch_fused4(bool sym, const FusedArgs &a, bool ro, int grid, cudaStream_t s);

// Path-filtered step (ofpf.cu): one growth or slide step on the compacted list.
struct OfpfArgs {
    const long long *key_in;
    const double2 *val_in;
    long long *key_out;
    double2 *val_out;
    const long long *n_in;   // device: entries of the input list
    long long *n_out;        // device: entries of the output list (written by the scan)
    unsigned short *flags;   // [cap]: keep flags of the N outputs of the group headed by entry i
    int *blkcnt;             // [nblk][N]
    long long *blkbase;      // [nblk][N]
    long long *kept;         // device: kept[k]
    int *overflow;           // device: set when the output exceeds cap
    long long cap;
    const double2 *small;    // SmallLayout (K', beta, growth psi rows)
    const double2 *tab;      // [2][kMaxL + 1][N]: psi(sigma'; eta_lag) / psi(sigma'; E_lag) (slide partners)
    double2 *partials;
    double2 *rho;            // readout of step k, or nullptr
    unsigned *counter;
    double th2;              // theta^2
    long long top;           // N^(L-1)
    long long grow_w;        // growth: N^k
    int k, L, slide, var;
    double delta[kMaxD];
};
cudaError_t launch_ofpf_step(int M, bool lattice, const OfpfArgs &a, int nblk, cudaStream_t s);

// Batched sweeps (batch.cu): B independent problems, one CTA each, every step in one launch.
// Table image (double2 entries) at `tab`: psi_eta[L+1][N], psi_E[L+1][N], psi_TI[L+1][N] (lag j = 1..L;
// psi(sigma', e) = -(e s+(sigma') - conj(e) s-(sigma'))), psi_self[2][N] (self interior G(1), self end
// G(1/2)), H0[M*M], H1[M*M].
struct BatchArgs {
    double2 *A;              // [B][N^L] in place
    const double2 *tab;
    const double2 *ptab;     // per-problem psi tables [B][(3(L+1)+2) N] (layout of tab's psi part), or nullptr
    const double *f;         // [B][n_steps] drive amplitudes (nullptr: none)
    const double2 *rho0;     // [B][N]
    const int *out_idx;      // [n_steps + 1]: output slot of step k, or -1
    double2 *rho;            // [B][n_out][N]
    long long NL;            // N^L
    long long n_steps;
    double dt;
    int L, n_out, D;
    int cls[kMaxN];          // Delta-s class of pair state n (0: Delta s = 0, else d + 1)
    double dsig[kMaxN];      // Delta s(n)
    double delta[kMaxD];     // Delta s of class d + 1
};
size_t batch_dyn_smem(int M, int L, int D);  // tables only (the ARDM may add N^L entries)
// Device eta setup (eta.cu): kind as qp_bath_kind (0..3), xi = coupling.
struct EtaBath {
    int kind;
    double xi, wc, kT;
};
constexpr int kEtaBatchMax = 512;  // baths per launch (passed by value as a __grid_constant__ parameter)
struct EtaBatch {
    EtaBath b[kEtaBatchMax];
};
cudaError_t launch_eta(const EtaBatch &baths, int B, int L, double dt, double2 *d_eta, double *d_err, cudaStream_t s);
cudaError_t launch_batch(int M, const BatchArgs &a, int B, cudaStream_t s);
// psi rows of B problems from their eta classes [B][3L+2] (qp_plan_eta order): ptab[b] in tab's layout
cudaError_t launch_psi_tables(int M, const double (&s)[kMaxM], const double2 *eta, double2 *ptab, int B, int L, cudaStream_t st);
constexpr int kBatchBlock = 256;

}  // namespace qp
