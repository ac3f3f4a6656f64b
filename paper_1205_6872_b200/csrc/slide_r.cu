// slide_r.cu -- k_fused_r: S (1 or 2) consecutive slide steps k..k+S-1 (k >= L) of the iterative
// tensor propagator (the Makri-Makarov scheme the paper accelerates; its "BSXFUN" lines
// P:384) in ONE pass over HBM, in place on the ring-buffer ARDM, with the rho(t_k) readout of every
// requested step ("line 169") fused into the same pass.  Used for M = 3, 4 and
// for the partial fusion groups (S < 3) of M = 2 plans (slide3.cu holds the M = 2, S = 3 kernel).
//
// ARDM layout: N^L complex FP64 entries, flat index x = sum_q d_q N^q; time point t
// lives in digit ("ring slot") q = t mod L, so nothing is ever transposed.  Step k contracts slot
// k mod L (holding sigma_{k-L}) and writes sigma_k into the same slot.  For one fibre (all slots
// except the contracted one fixed) with old values a[old]:
//   out[new] = K'(new, last) * exp(Ds(new) Psi(mid)) * sum_old exp(Ds(new) psi_L(old)) a[old]
// Ds = s+ - s- of the new pair state, K' = self factor x bare propagator pair (Eq. 8),
// Psi(mid) = sum_j psi_j(partner at lag j) the Eq. 9 exponent of the kept partners.  Rows with the
// same Ds share one moment S_d = sum_old beta_d(old) a[old] and one factor E_d = exp(delta_d Psi),
// a product of host-built tables (no transcendental in the kernel).
//
// Step fusion: step k only reads/writes slot p = k mod L, and its factors depend on the other slots
// only through their values, so for every fixed value of the other L-S ("outer") slots the N^S
// entries of the "super-fibre" evolve independently through all S steps.  One thread loads its
// super-fibre once, applies S steps in registers (reading rho of each step from the pre-step
// values) and stores it once: HBM traffic per step drops from 32 B to 32/S B per ARDM entry.
//
// Warps are independent: each warp owns a contiguous, static range of (tile, 32-fibre chunk) units
// (tile = T = N^v outer fibres), builds the tile's factor table KU in its own shared-memory slice
// (warp-synchronous, no CTA barrier in the main loop) and sweeps the tile in chunks of 32 outer
// fibres, lane = outer fibre.  Readout accumulators live in shared memory; the CTA reduction at the
// end is in fixed order (deterministic).
#include <cooperative_groups.h>

#include "common.cuh"

namespace qp {

// One fused launch's work (every CTA of the grid runs it): the body of k_fused_r and of the
// persistent k_persist_r (one call per fusion group).
// Readout modes of fused_r_body: the grid-wide finalize (last CTA sums the block partials), the block
// partials only (the persistent kernel sums them after its grid barrier), or straight into rho (grid
// of one CTA).
enum RoMode { kRoFinalize = 0, kRoDefer = 1, kRoDirect = 2 };
// loads / stores of the table and ARDM pointers: global-memory cache hints, or plain generic accesses
// when SMEM (k_small_r: every table and the ARDM live in shared memory)
template <bool SMEM, typename T> __device__ __forceinline__ T ld_tab(const T *p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}
template <bool SMEM> __device__ __forceinline__ double2 ld_ardm(const double2 *p) {
    if constexpr (SMEM) return *p;
    else return __ldcs(p);
}
template <bool SMEM> __device__ __forceinline__ void st_ardm(double2 *p, double2 v) {
    if constexpr (SMEM) *p = v;
    else __stcs(p, v);
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, bool RO, int RMODE = kRoFinalize, bool SMEM = false>
__device__ __forceinline__ void fused_r_body(const FusedArgs &a) {
    constexpr int N = M * M;
    constexpr int D = n_classes(M, LAT);
    constexpr int Q = cpow(N, S - 1);    // fibres per super-fibre and sub-step
    constexpr int NS = Q * N;
    constexpr int NK = RO ? 2 : 1;
    constexpr int W = BLOCK / 32;
    static_assert(!SYM || (M == 2 && D == 2), "symmetric moments are the M = 2 s = (+s,-s) case");
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    // dynamic shared memory: readout accumulators [S][N][BLOCK] (RO only)
    extern __shared__ double2 dyn_smem[];
    auto accS = reinterpret_cast<double2(*)[RO ? N : 1][RO ? BLOCK : 1]>(dyn_smem);
    for (int i = threadIdx.x; i < 2 * N * N; i += BLOCK) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < S * S * 2 * D * N; i += BLOCK) (&sIn[0][0][0][0][0])[i] = a.inner[i];
    __shared__ double2 sBeta[S][2][D][N];  // beta_d(old) of each sub-step (first slide: initial-edge classes)
    for (int i = threadIdx.x; i < S * 2 * D * N; i += BLOCK) {
        const int s_ = i / (2 * D * N), kap = (i / (D * N)) % 2, r_ = i % (D * N);
        (&sBeta[0][0][0][0])[i] = a.small[lay.beta(a.var[s_], kap) + r_];
    }
    if constexpr (RO)
        for (int s = 0; s < S; ++s)
            for (int n = 0; n < N; ++n) accS[s][n][threadIdx.x] = make_double2(0.0, 0.0);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // work unit = (tile, chunk of 32 outer fibres); contiguous, static unit range per warp
    // (deterministic readout order); the warp rebuilds its tile tables when the tile changes
    const int CH = (a.T + 31) >> 5;
    const long long n_units = (long long)a.n_tiles * CH;
    const int gw = (int)blockIdx.x * W + warp, nw_tot = (int)gridDim.x * W;
    const long long per = n_units / nw_tot, rem = n_units % nw_tot;
    const long long u_begin = gw * per + min((long long)gw, rem);
    const long long u_end = u_begin + per + (gw < rem ? 1 : 0);
    constexpr int NKU = S * NK * Q * N * N;
    // KI (tile independent, per CTA): K'_kap(new, last) * prod_{i != s} inner_i(class(new), digit_i(r))
    __shared__ double2 KI[S][NK][Q][N][N];
    // per warp: KU = KI * Ehi(tile) and the tile's base offset / 'last' digit
    __shared__ double2 KU[W][S][NK][Q][N][N];
    __shared__ double2 sEhi[W][S][NK][D];
    __shared__ long long sBase[W];
    __shared__ int sLast[W];
    __syncthreads();
    for (int j = threadIdx.x; j < NKU; j += BLOCK) {
        const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                  s = j / (N * N * Q * NK);
        const int c = class_of(M, LAT, nw / M, nw % M);
        double2 e = sK[kap][nw][last];
        if (c > 0)
            for (int i = 0; i < S; ++i)
                if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
        KI[s][kap][rr][nw][last] = e;
    }
    __syncthreads();
    const double2(&ki)[S][NK][Q][N][N] = KI;
    double2(&ku_w)[S][NK][Q][N][N] = KU[warp];
    int cur_tile = -1;
    long long tbase = 0;
    int last_t = 0;
    for (long long u = u_begin; u < u_end; ++u) {
        const int tau = (int)(u / CH), t = (int)(u % CH) * 32 + lane;
        if (tau != cur_tile) {  // warp-synchronous tile setup
            __syncwarp();       // previous tile's KU no longer in use
            cur_tile = tau;
            if (lane < S * NK * D) {
                const int s = lane / (NK * D), kap = (lane / D) % NK, d = lane % D;
                double2 e = make_double2(1.0, 0.0);
                for (int g = 1; g < a.G; ++g)
                    e = cmul(e, ld_tab<SMEM>(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
                sEhi[warp][s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
            }
            if (lane == 31) {
                long long b = 0;
                for (int g = 1; g < a.G; ++g) b += ld_tab<SMEM>(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
                sBase[warp] = b;
                sLast[warp] = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
            }
            __syncwarp();
            for (int j = lane; j < NKU; j += 32) {
                const int last = j % N, nw = (j / N) % N, rr = (j / (N * N)) % Q, kap = (j / (N * N * Q)) % NK,
                          s = j / (N * N * Q * NK);
                const int c = class_of(M, LAT, nw / M, nw % M);
                const double2 e = ki[s][kap][rr][nw][last];
                ku_w[s][kap][rr][nw][last] = c > 0 ? cmul(e, sEhi[warp][s][kap][c - 1]) : e;
            }
            __syncwarp();
            tbase = sBase[warp];
            last_t = sLast[warp];
        }
        if (t >= a.T) continue;
        const int2 lo = ld_tab<SMEM>(&a.lofs[t]);
        const long long base = tbase + lo.x;
        double2 x[NS];
#pragma unroll
        for (int e = 0; e < NS; ++e) {
            long long o = base;
#pragma unroll
            for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
            x[e] = ld_ardm<SMEM>(a.A + o);
        }
        const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool ro = RO && a.rho[s] != nullptr;
            double2 E0[NK][D];  // outer group-0 factor of this outer fibre
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    E0[kap][d] = (kap == 0 || ro) ? ld_tab<SMEM>(&a.Etab[(((size_t)s * 2 + kap) * a.G * D + d) * a.X + t])
                                                  : make_double2(0.0, 0.0);
            double2 acc[RO ? N : 1];
#pragma unroll
            for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < Q; ++r) {
                double2 xf[N];
#pragma unroll
                for (int v = 0; v < N; ++v) xf[v] = x[fib_elem<N, S>(s, r, v)];
                const int last = s == 0 ? last0 : fib_digit<N, S>(s, r, s - 1);
                const double2(&ku)[NK][Q][N][N] = ku_w[s];
                double2 S0, m[NK][D];
                if constexpr (SYM) {
                    const double2 u = cadd(xf[0], xf[3]), w = csub(xf[0], xf[3]);
                    const double2 p = cadd(xf[1], xf[2]), q = csub(xf[1], xf[2]);
                    S0 = cadd(u, p);
#pragma unroll
                    for (int kap = 0; kap < NK; ++kap) {
                        if (kap == 1 && !ro) break;
                        const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2],
                                     sh = a.sym[s][kap][3];
                        const double2 A = make_double2(fma(cr, u.x, ch * p.x), fma(cr, u.y, ch * p.y));
                        const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                        m[kap][0] = cadd(A, Bv);
                        m[kap][D - 1] = csub(A, Bv);
                    }
                } else {
                    S0 = xf[0];
#pragma unroll
                    for (int v = 1; v < N; ++v) S0 = cadd(S0, xf[v]);
#pragma unroll
                    for (int kap = 0; kap < NK; ++kap) {
                        if (kap == 1 && !ro) break;
#pragma unroll
                        for (int d = 0; d < D; ++d) {
                            double2 mm = cmul(sBeta[s][kap][d][0], xf[0]);
#pragma unroll
                            for (int v = 1; v < N; ++v) mm = cfma(sBeta[s][kap][d][v], xf[v], mm);
                            m[kap][d] = mm;
                        }
                    }
                }
                if (ro) {
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const double2 pt = cmul(E0[NK - 1][d], m[NK - 1][d]);
#pragma unroll
                        for (int aa = 0; aa < M; ++aa)
#pragma unroll
                            for (int bb = 0; bb < M; ++bb)
                                if (class_of(M, LAT, aa, bb) == d + 1)
                                    acc[RO ? aa * M + bb : 0] =
                                        cfma(ku[NK - 1][r][aa * M + bb][last], pt, acc[RO ? aa * M + bb : 0]);
                    }
                }
                double2 P[D];
#pragma unroll
                for (int d = 0; d < D; ++d) P[d] = cmul(E0[0][d], m[0][d]);
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = 0; bb < M; ++bb) {
                        const int nw = aa * M + bb;
                        const int c = class_of(M, LAT, aa, bb);
                        const double2 o = cmul(ku[0][r][nw][last], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
                        x[fib_elem<N, S>(s, r, nw)] = o;
                        if (ro && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
                    }
            }
            if (ro) {
#pragma unroll
                for (int n = 0; n < N; ++n)
                    accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0] =
                        cadd(accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0], acc[RO ? n : 0]);
            }
        }
#pragma unroll
        for (int e = 0; e < NS; ++e) {
            long long o = base;
#pragma unroll
            for (int i = 0; i < S; ++i) o += (long long)((e / cpow(N, i)) % N) * a.pw_in[i];
            st_ardm<SMEM>(a.A + o, x[e]);
        }
    }
    if constexpr (RO) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr) {
                double2 tt[N];
#pragma unroll
                for (int n = 0; n < N; ++n) tt[n] = accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0];
                if constexpr (RMODE == kRoDefer)
                    reduce_block_to<N, BLOCK>(tt, a.partials + ((size_t)s * kPartialsMax + blockIdx.x) * N);
                else if constexpr (RMODE == kRoDirect)
                    reduce_block_to<N, BLOCK>(tt, a.rho[s]);
                else
                    reduce_finalize<N, BLOCK>(tt, a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                              a.rho_accumulate != 0);
            }
    }
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused_r(const __grid_constant__ FusedArgs a) {
    fused_r_body<M, LAT, SYM, S, BLOCK, RO>(a);
}

// ---------------------------------------------------------------------------------- persistent
// k_persist_r: the slide steps k_begin..k_end-1 of a small (L2-resident) ARDM in ONE cooperative
// launch.  Per fusion group (aligned on k - L, depth S <= PA.Smax <= 2): the group's launch-set
// arguments are copied from the device table into shared memory, the per-step fields (rho
// destination, beta variant, symmetric-moment constants) are set from k, every CTA runs
// fused_r_body, and a grid-wide barrier orders the group's in-place update before the next group.
// The readout stops at the block partials (double buffered by group parity); after the barrier CTA 0
// sums them into rho while the others start the next group.  The launch count per qp_steps call
// drops from one per group to one.
template <int M, bool LAT, bool SYM, int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_persist_r(const __grid_constant__ PersistArgs pa) {
    __shared__ FusedArgs sa;
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    constexpr int N = M * M;
    int par = 0;
    for (long long k = pa.k_begin; k < pa.k_end; par ^= 1) {
        const long long grp_end = pa.L + ((k - pa.L) / pa.Smax + 1) * pa.Smax;
        const int S = (int)(grp_end < pa.k_end ? grp_end - k : pa.k_end - k);
        const int p0 = (int)(k % pa.L);
        {
            const int4 *src = reinterpret_cast<const int4 *>(pa.sets + (size_t)p0 * pa.Smax + (S - 1));
            int4 *dst = reinterpret_cast<int4 *>(&sa);
            for (int i = threadIdx.x; i < (int)(sizeof(FusedArgs) / 16); i += BLOCK) dst[i] = src[i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            sa.A = pa.A;
            sa.partials = pa.partials + (size_t)2 * par * kPartialsMax * N;
            for (int st = 0; st < S; ++st) {
                const int slot = pa.slot[k + st];
                const int var = (k + st == pa.L) ? 1 : 0;
                sa.rho[st] = slot >= 0 ? pa.rho_base + (size_t)slot * (M * M) : nullptr;
                sa.var[st] = var;
                for (int kap = 0; kap < 2; ++kap)
                    for (int j = 0; j < 4; ++j) sa.sym[st][kap][j] = pa.sym[var][kap][j];
            }
        }
        __syncthreads();
        if (M == 2 && S == 2) fused_r_body<M, LAT, SYM, (M == 2 ? 2 : 1), BLOCK, true, kRoDefer>(sa);
        else fused_r_body<M, LAT, SYM, 1, BLOCK, true, kRoDefer>(sa);
        grid.sync();
        if (blockIdx.x == 0)
            for (int st = 0; st < S; ++st)
                if (sa.rho[st] != nullptr)
                    reduce_partials_sum<N, BLOCK>(sa.partials + (size_t)st * kPartialsMax * N, (int)gridDim.x, sa.rho[st], false);
        k += S;
    }
}

// ---------------------------------------------------------------------------------- dispatch
// (M, S) -> block, tile digits v (T = N^v outer fibres per tile), min blocks per SM
#define QP_FUSED_R_CFGS(X) \
    X(2, 1, 256, 4, 2)     \
    X(2, 2, 256, 4, 2)     \
    X(3, 1, 256, 3, 2)     \
    X(4, 1, 64, 2, 4)

// k_small_r: the same group loop for an ARDM small enough to live in ONE CTA's shared memory together
// with every factor table of the plan: the tables ([0, tables_bytes) of the workspace) and the ARDM
// are copied in once, the launch-set arguments are re-pointed at the shared copies, the groups run
// with CTA barriers only (readout straight into rho), and the ARDM is copied back at the end.
// Dynamic shared memory: [body readout accumulators][tables][ARDM][launch-set arguments].
template <int M, bool LAT, bool SYM, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1) k_small_r(const __grid_constant__ PersistArgs pa) {
    constexpr int N = M * M;
    extern __shared__ __align__(16) double2 dyn_smem[];
    __shared__ FusedArgs sa;
    unsigned char *base = reinterpret_cast<unsigned char *>(dyn_smem);
    unsigned char *tab = base + pa.acc_bytes;
    double2 *sA = reinterpret_cast<double2 *>(tab + pa.tables_bytes);
    FusedArgs *sets = reinterpret_cast<FusedArgs *>(reinterpret_cast<unsigned char *>(sA) + pa.ardm_entries * 16);
    {
        const int4 *src = reinterpret_cast<const int4 *>(pa.wbase);
        int4 *dst = reinterpret_cast<int4 *>(tab);
        for (long long i = threadIdx.x; i < pa.tables_bytes / 16; i += BLOCK) dst[i] = src[i];
        const int4 *srcA = reinterpret_cast<const int4 *>(pa.A);
        int4 *dstA = reinterpret_cast<int4 *>(sA);
        for (long long i = threadIdx.x; i < pa.ardm_entries; i += BLOCK) dstA[i] = srcA[i];
        const int4 *srcS = reinterpret_cast<const int4 *>(pa.sets);
        int4 *dstS = reinterpret_cast<int4 *>(sets);
        for (long long i = threadIdx.x; i < (long long)pa.nsets * (long long)(sizeof(FusedArgs) / 16); i += BLOCK) dstS[i] = srcS[i];
    }
    __syncthreads();
    auto rebase = [&](const void *p) -> unsigned char * {
        return tab + (reinterpret_cast<const unsigned char *>(p) - reinterpret_cast<const unsigned char *>(pa.wbase));
    };
    for (int i = threadIdx.x; i < pa.nsets; i += BLOCK) {
        FusedArgs &f = sets[i];
        f.A = sA;
        f.small = reinterpret_cast<const double2 *>(rebase(f.small));
        f.inner = reinterpret_cast<const double2 *>(rebase(f.inner));
        f.Etab = reinterpret_cast<const double2 *>(rebase(f.Etab));
        f.goff = reinterpret_cast<const long long *>(rebase(f.goff));
        f.lofs = reinterpret_cast<const int2 *>(rebase(f.lofs));
    }
    __syncthreads();
    for (long long k = pa.k_begin; k < pa.k_end;) {
        const long long grp_end = pa.L + ((k - pa.L) / pa.Smax + 1) * pa.Smax;
        const int S = (int)(grp_end < pa.k_end ? grp_end - k : pa.k_end - k);
        const int p0 = (int)(k % pa.L);
        {
            const int4 *src = reinterpret_cast<const int4 *>(sets + (size_t)p0 * pa.Smax + (S - 1));
            int4 *dst = reinterpret_cast<int4 *>(&sa);
            for (int i = threadIdx.x; i < (int)(sizeof(FusedArgs) / 16); i += BLOCK) dst[i] = src[i];
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int st = 0; st < S; ++st) {
                const int slot = pa.slot[k + st];
                const int var = (k + st == pa.L) ? 1 : 0;
                sa.rho[st] = slot >= 0 ? pa.rho_base + (size_t)slot * N : nullptr;
                sa.var[st] = var;
                for (int kap = 0; kap < 2; ++kap)
                    for (int j = 0; j < 4; ++j) sa.sym[st][kap][j] = pa.sym[var][kap][j];
            }
        __syncthreads();
        if (M == 2 && S == 2) fused_r_body<M, LAT, SYM, (M == 2 ? 2 : 1), BLOCK, true, kRoDirect, true>(sa);
        else fused_r_body<M, LAT, SYM, 1, BLOCK, true, kRoDirect, true>(sa);
        __syncthreads();
        k += S;
    }
    {
        const int4 *srcA = reinterpret_cast<const int4 *>(sA);
        int4 *dstA = reinterpret_cast<int4 *>(pa.A);
        for (long long i = threadIdx.x; i < pa.ardm_entries; i += BLOCK) dstA[i] = srcA[i];
    }
}

namespace {
template <int M, bool LAT, bool SYM, int BLOCK>
cudaError_t small_t(const PersistArgs &pa, size_t dyn, cudaStream_t s) {
    auto f = k_small_r<M, LAT, SYM, BLOCK>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    f<<<1, BLOCK, dyn, s>>>(pa);
    return cudaGetLastError();
}
template <int M, bool LAT, bool SYM, int BLOCK>
int small_static_t() {
    cudaFuncAttributes at{};
    if (cudaFuncGetAttributes(&at, k_small_r<M, LAT, SYM, BLOCK>) != cudaSuccess) return 1 << 30;
    return (int)at.sharedSizeBytes;
}

template <int M, bool LAT, bool SYM, int BLOCK, int MINB>
cudaError_t persist_t(const PersistArgs &pa, int grid, cudaStream_t s) {
    const size_t dyn = (size_t)(M == 2 ? 2 : 1) * M * M * BLOCK * 16;  // readout accumulators of the deepest body
    auto f = k_persist_r<M, LAT, SYM, BLOCK, MINB>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    void *args[] = {(void *)&pa};
    return cudaLaunchCooperativeKernel((const void *)f, dim3(grid), dim3(BLOCK), args, dyn, s);
}
template <int M, bool LAT, bool SYM, int BLOCK, int MINB>
int persist_occ_t() {
    const size_t dyn = (size_t)(M == 2 ? 2 : 1) * M * M * BLOCK * 16;
    auto f = k_persist_r<M, LAT, SYM, BLOCK, MINB>;
    int o = 0;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, f, BLOCK, dyn);
    return o;
}

template <int M, int S, int BLOCK>
constexpr size_t fused_r_dyn_smem(bool ro) {
    return (ro ? (size_t)S * M * M * BLOCK : 0) * 16;
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB>
cudaError_t fused_r_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    const size_t dyn = fused_r_dyn_smem<M, S, BLOCK>(ro);
    if (ro) {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true><<<grid, BLOCK, dyn, s>>>(a);
    } else {
        cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false><<<grid, BLOCK, dyn, s>>>(a);
    }
    return cudaGetLastError();
}

template <int M, bool LAT, bool SYM, int S, int BLOCK, int MINB>
int fused_r_occ_t() {
    int o1 = 0, o2 = 0;
    const size_t d1 = fused_r_dyn_smem<M, S, BLOCK>(true), d2 = fused_r_dyn_smem<M, S, BLOCK>(false);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaFuncSetAttribute(k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d2);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused_r<M, LAT, SYM, S, BLOCK, MINB, false>, BLOCK, d2);
    return o1 < o2 ? o1 : o2;
}
}  // namespace

bool fused_r_has(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return true;
    QP_FUSED_R_CFGS(X)
#undef X
    return false;
}
int fused_r_tile_digits(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return V;
    QP_FUSED_R_CFGS(X)
#undef X
    return -1;
}
int fused_r_block(int M, int S) {
#define X(M_, S_, B, V, MB) if (M == M_ && S == S_) return B;
    QP_FUSED_R_CFGS(X)
#undef X
    return 0;
}

cudaError_t launch_fused_r(int M, bool lattice, bool sym, int S, const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
#define X(M_, S_, B, V, MB)                                                                       \
    if (M == M_ && S == S_) {                                                                     \
        if (M_ == 2 && sym) return fused_r_t<M_, false, (M_ == 2), S_, B, MB>(a, ro, grid, s);    \
        if (M_ > 2 && lattice) return fused_r_t<M_, (M_ > 2), false, S_, B, MB>(a, ro, grid, s);  \
        return fused_r_t<M_, false, false, S_, B, MB>(a, ro, grid, s);                            \
    }
    QP_FUSED_R_CFGS(X)
#undef X
    return cudaErrorInvalidValue;
}

// persistent kernel: per M the block / min-blocks of k_fused_r at S = 1 (M = 2: 128 threads so that the
// static shared memory of both bodies, S = 1 and 2, fits)
int persist_max_S(int M) { return M == 2 ? 2 : 1; }
cudaError_t launch_persist(int M, bool lattice, bool sym, const PersistArgs &pa, int grid, cudaStream_t s) {
    switch (M) {
    case 2: return sym ? persist_t<2, false, true, 128, 4>(pa, grid, s) : persist_t<2, false, false, 128, 4>(pa, grid, s);
    case 3: return lattice ? persist_t<3, true, false, 256, 2>(pa, grid, s) : persist_t<3, false, false, 256, 2>(pa, grid, s);
    case 4: return lattice ? persist_t<4, true, false, 64, 4>(pa, grid, s) : persist_t<4, false, false, 64, 4>(pa, grid, s);
    }
    return cudaErrorInvalidValue;
}
int persist_occupancy(int M, bool lattice, bool sym) {
    switch (M) {
    case 2: return sym ? persist_occ_t<2, false, true, 128, 4>() : persist_occ_t<2, false, false, 128, 4>();
    case 3: return lattice ? persist_occ_t<3, true, false, 256, 2>() : persist_occ_t<3, false, false, 256, 2>();
    case 4: return lattice ? persist_occ_t<4, true, false, 64, 4>() : persist_occ_t<4, false, false, 64, 4>();
    }
    return 0;
}
int persist_block(int M) { return M == 4 ? 64 : (M == 2 ? 128 : 256); }
size_t small_acc_bytes(int M) { return (size_t)persist_max_S(M) * M * M * persist_block(M) * 16; }
cudaError_t launch_small(int M, bool lattice, bool sym, const PersistArgs &pa, size_t dyn, cudaStream_t s) {
    switch (M) {
    case 2: return sym ? small_t<2, false, true, 128>(pa, dyn, s) : small_t<2, false, false, 128>(pa, dyn, s);
    case 3: return lattice ? small_t<3, true, false, 256>(pa, dyn, s) : small_t<3, false, false, 256>(pa, dyn, s);
    case 4: return lattice ? small_t<4, true, false, 64>(pa, dyn, s) : small_t<4, false, false, 64>(pa, dyn, s);
    }
    return cudaErrorInvalidValue;
}
int small_static_smem(int M, bool lattice, bool sym) {
    switch (M) {
    case 2: return sym ? small_static_t<2, false, true, 128>() : small_static_t<2, false, false, 128>();
    case 3: return lattice ? small_static_t<3, true, false, 256>() : small_static_t<3, false, false, 256>();
    case 4: return lattice ? small_static_t<4, true, false, 64>() : small_static_t<4, false, false, 64>();
    }
    return 1 << 30;
}

int fused_r_occupancy(int M, bool lattice, bool sym, int S) {
#define X(M_, S_, B, V, MB)                                                             \
    if (M == M_ && S == S_) {                                                           \
        if (M_ == 2 && sym) return fused_r_occ_t<M_, false, (M_ == 2), S_, B, MB>();    \
        if (M_ > 2 && lattice) return fused_r_occ_t<M_, (M_ > 2), false, S_, B, MB>();  \
        return fused_r_occ_t<M_, false, false, S_, B, MB>();                            \
    }
    QP_FUSED_R_CFGS(X)
#undef X
    return 0;
}

}  // namespace qp
