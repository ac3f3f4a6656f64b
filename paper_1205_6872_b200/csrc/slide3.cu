// slide3.cu -- k_fused3: three consecutive slide steps k, k+1, k+2 (k >= L) of the iterative tensor
// propagator for M = 2 (N = 4) in ONE pass over HBM, in place on the ring-buffer ARDM, with the
// rho(t_k) readout of every requested step fused (algebra and step
// fusion as in slide_r.cu).  HBM traffic per step: 32/3 B per ARDM entry.
//
// The 64-entry super-fibre of an outer fibre is held by 4 lanes of a warp (part j = lane >> 3 holds
// inner digit 2 = j: 16 entries), so sub-steps 0 and 1 (fibres along digits 0 and 1) are
// lane-local; before sub-step 2 the four lanes transpose digit 0 <-> digit 2 through a per-warp
// shared-memory buffer and then hold the fibres along digit 2.  Lane l works on outer fibre (l & 7)
// of the warp's 8; a CTA sweeps a tile of T outer fibres in rounds of 8 W.  Factor tables KU are
// CTA-wide per tile.
//
// How a round reaches registers (fixed per launch set at plan time, host.cpp build_launch_set):
//   VW = -1 : plain loads (lane map 0: 16 loads per thread, 32-byte pairs along ring slot 0 when an
//             inner digit is slot 0; lane map 1: 32 consecutive outer fibres per warp load).
//   VW >= 0 : per-warp TMA staging.  Each warp's 8 fibres of a round are one 5-D
//             cp.async.bulk.tensor box (8 KB) plus one bulk copy of their outer factors E0 and
//             tile-local offsets, completing on the warp's own mbarrier; after its lanes have read
//             the stage the warp (__syncwarp) refills it with its next unit -- no CTA barrier per
//             round.  The view (box dimension order + swizzle) depends on which inner digit is
//             ring slot 0 so that the stage reads are conflict-free:
//               VW 0 (A, 1 <= p0 <= L-3): stage [d2][d1][d0][f]
//               VW 1 (B, p0 = L-2, d2 = slot 0): 128-B rows (f & 1, d2) of rows (d1, d0, f / 2)
//               VW 2 (C, p0 = L-1, d1 = slot 0): 128-B rows (d2 & 1, d1) of rows (d0, d2 / 2, f)
//               VW 3 (D, p0 = 0,   d0 = slot 0): 128-B rows (d1 & 1, d0) of rows (d2, d1 / 2, f)
//             with the 128-B swizzle (16-B chunk ^= row & 7).
#include "common.cuh"

namespace qp {

// KU row swizzle: the 16 entries (new, last) of KU row r are stored at (4 new + last) ^ f(r).  The
// lanes of a warp read rows r = d + 4j (sub-steps 0, 1) or j + 4d (sub-step 2) for their digit-2
// value j; rows are 256 B apart (same banks), so without the swizzle the 4 rows conflict 4-way.
// f(r) = g(r / 4) ^ g(r % 4), g(x) = 4 (x & 1) + x / 2: distinct 16-B bank groups for the 4 rows,
// and at most 2-way for sub-step 0 whose 'last' also varies across lanes.
__device__ __forceinline__ int f3_swizzle(int r) {
    const int hi = r >> 2, lo = r & 3;
    return (((hi & 1) << 2) | (hi >> 1)) ^ (((lo & 1) << 2) | (lo >> 1));
}

template <bool SYM, int MAP, int BLOCK, int MINB, int VW, bool RO>
__global__ void __launch_bounds__(BLOCK, MINB) k_fused3(const __grid_constant__ FusedArgs a) {
    constexpr int M = 2, N = 4, S = 3, Q = 16, D = 2;
    constexpr bool TW = VW >= 0;         // per-warp TMA staging
    static_assert(!TW || MAP == 0, "TMA staging reads the stage with lane map 0");
    constexpr int FS = 8;                // fibres per warp and round (one TMA box)
    constexpr int NK = RO ? 2 : 1;
    constexpr int W = BLOCK / 32;
    constexpr bool LAT = false;
    const SmallLayout lay{N, D, 0};
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][S][2][D][N];
    __shared__ double2 KU[S][NK][Q][N][N];
    __shared__ double2 sEhi[S][NK][D];
    __shared__ long long sBase;
    __shared__ int sLast;
    // dynamic: (TW) per warp the TMA stage [FS x 64 entries] and two E0 blocks, then the exchange
    // buffer (W x 16 x 8 entries), then the readout accumulators [S][N][BLOCK] (RO only)
    constexpr int E0B = S * 2 * D * FS + FS / 2;  // one (round, warp) block: factors [S][2][D][FS] + FS int2 offsets
    extern __shared__ __align__(1024) double2 dyn_smem_raw[];
    double2 *const stage = dyn_smem_raw;
    double2 *const sE0 = dyn_smem_raw + (TW ? W * FS * 64 : 0);
    double2 *const dyn_smem = sE0 + (TW ? W * 2 * E0B : 0);
    __shared__ __align__(8) unsigned long long sFullW[TW ? W : 1];
    auto accS = reinterpret_cast<double2(*)[RO ? N : 1][RO ? BLOCK : 1]>(dyn_smem + W * 16 * 8);
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
    static_assert(MAP == 0 || W % 4 == 0, "lane map 1: groups of 4 warps (one per digit-2 value)");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lane map 0: lane = (j, t8), 8 outer fibres per warp, the 4 quarters of a super-fibre in one warp
    // lane map 1: lane = one of 32 consecutive outer fibres, warp -> j (512 contiguous bytes per load
    //             when the lowest ARDM digit is an outer digit); quarters exchanged across 4 warps
    const int j = MAP == 0 ? lane >> 3 : warp & 3;
    const int fib = MAP == 0 ? warp * 8 + (lane & 7) : (warp >> 2) * 32 + lane;  // fibre within a round
    // map 0: [W][16][8] per warp; map 1: [16][8 W] (same size)
    auto xch_at = [&](int e) -> double2 & {
        return MAP == 0 ? dyn_smem[(warp * 16 + e) * 8 + (lane & 7)] : dyn_smem[e * 8 * W + fib];
    };
    const int per = a.n_tiles / (int)gridDim.x, rem = a.n_tiles % (int)gridDim.x;
    const int t_begin = (int)blockIdx.x * per + min((int)blockIdx.x, rem);
    const int t_end = t_begin + per + ((int)blockIdx.x < rem ? 1 : 0);
    constexpr int NKU = S * NK * Q * N * N;
    const int rounds = (a.T + 8 * W - 1) / (8 * W);

    // one fibre: xf holds the N old values; on return the N new values.  r = inner combination,
    // last = value of the previous time point's slot.  acc: readout of this sub-step.
    auto fibre = [&](double2 (&xf)[N], int s, int r, int last, bool ro, const double2 (&E0)[D],
                     double2 (&acc)[RO ? N : 1]) {
        double2 S0, m[NK][D];
        if constexpr (SYM) {
            const double2 uu = cadd(xf[0], xf[3]), w = csub(xf[0], xf[3]);
            const double2 p = cadd(xf[1], xf[2]), q = csub(xf[1], xf[2]);
            S0 = cadd(uu, p);
#pragma unroll
            for (int kap = 0; kap < NK; ++kap) {
                if (kap == 1 && !ro) break;
                const double cr = a.sym[s][kap][0], ci = a.sym[s][kap][1], ch = a.sym[s][kap][2], sh = a.sym[s][kap][3];
                const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                m[kap][0] = cadd(A, Bv);
                m[kap][1] = csub(A, Bv);
            }
        } else {
            S0 = cadd(cadd(xf[0], xf[1]), cadd(xf[2], xf[3]));
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
        const int sw = MAP == 0 ? f3_swizzle(r) : 0;
        const double2 *ku0 = &KU[s][0][r][0][0], *ku1 = &KU[s][NK - 1][r][0][0];
        if (ro) {  // off-diagonal readout without the outer factor E0 (applied once per step below)
#pragma unroll
            for (int d = 0; d < D; ++d)
#pragma unroll
                for (int nw = 0; nw < N; ++nw)
                    if (class_of(M, LAT, nw / M, nw % M) == d + 1)
                        acc[RO ? nw : 0] = cfma(ku1[(nw * N + last) ^ sw], m[NK - 1][d], acc[RO ? nw : 0]);
        }
        double2 P[D];
#pragma unroll
        for (int d = 0; d < D; ++d) P[d] = cmul(E0[d], m[0][d]);
#pragma unroll
        for (int nw = 0; nw < N; ++nw) {
            const int c = class_of(M, LAT, nw / M, nw % M);
            const double2 o = cmul(ku0[(nw * N + last) ^ sw], c == 0 ? S0 : P[c > 0 ? c - 1 : 0]);
            xf[nw] = o;
            if (ro && c == 0) acc[RO ? nw : 0] = cadd(acc[RO ? nw : 0], o);
        }
    };

    // tile base offset (outer digit groups >= 1) and one unit's plain loads: unit = (tile tau, round
    // rd), lane -> outer fibre t = rd 8W + fib and digit-2 value j; X[d1][d0]
    auto tile_base = [&](int tau) {
        long long b = 0;
        for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
        return b;
    };
    auto load_unit = [&](int tau, int rd, double2 (&Y)[N][N], int2 &lo) {
        const int t = rd * 8 * W + fib;
        if (t < a.T) {
            lo = __ldg(&a.lofs[t]);
            const long long base = tile_base(tau) + lo.x + (long long)j * a.pw_in[2];
            if (a.pw_in[0] == 1) {  // d0 is ring slot 0: entry pairs (d0, d0 + 1) are adjacent, 32-B loads
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; d0 += 2) ld2_cs(a.A + base + d0 + (long long)d1 * a.pw_in[1], Y[d1][d0], Y[d1][d0 + 1]);
            } else if (a.pw_in[1] == 1) {  // d1 is slot 0: pairs (d1, d1 + 1)
#pragma unroll
                for (int d1 = 0; d1 < N; d1 += 2)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) ld2_cs(a.A + base + (long long)d0 * a.pw_in[0] + d1, Y[d1][d0], Y[d1 + 1][d0]);
            } else {
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0)
                        Y[d1][d0] = __ldcs(a.A + base + (long long)d0 * a.pw_in[0] + (long long)d1 * a.pw_in[1]);
            }
        } else {
            lo = make_int2(0, 0);
        }
    };
    // TW: warp w's stage and its two E0 blocks; the (round, warp) unit rw = rd W + w covers the tile's
    // outer fibres rw FS .. rw FS + 7, i.e. global outer fibre G = tau T + rw FS
    const int sfib = lane & 7;
    double2 *const sE0w = sE0 + (size_t)warp * 2 * E0B;
    double2 *const stg = stage + (size_t)warp * FS * 64;
    unsigned long long *const sFull = &sFullW[TW ? warp : 0];
    auto tma_issue = [&](int tau, int rd, int buf) {
        const int rw = rd * W + warp;
        const long long G = (long long)tau * a.T + (long long)rw * FS;
        fence_proxy_async();
        mbar_expect_tx(sFull, FS * 64 * 16 + E0B * 16);
        const int sh = a.tma_nA_log2;  // power-of-two run length (M = 2): shifts, no 64-bit division
        const long long q = sh >= 0 ? (G >> sh) : G / a.tma_nA, rm = sh >= 0 ? (G & (a.tma_nA - 1)) : G - q * a.tma_nA;
        tma_load_5d(stg, &a.tmap, sFull, (int)(a.tma_c0m * rm), (int)q);
        bulk_g2s(sE0w + buf * E0B, a.E0r + (size_t)rw * E0B, E0B * 16, sFull);
    };
    unsigned phase = 0, cur = 0;
    if constexpr (TW) {
        if (lane == 0) {
            mbar_init(sFull, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (lane == 0 && t_begin < t_end) tma_issue(t_begin, 0, 0);
    }

    for (int tau = t_begin; tau < t_end; ++tau) {
        __syncthreads();  // previous tile's KU no longer in use
        if ((int)threadIdx.x < S * NK * D) {
            const int s = threadIdx.x / (NK * D), kap = (threadIdx.x / D) % NK, d = threadIdx.x % D;
            double2 e = make_double2(1.0, 0.0);
            for (int g = 1; g < a.G; ++g)
                e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
            sEhi[s][kap][d] = cmul(e, a.fixfac[s][kap][d]);
        }
        if ((int)threadIdx.x == BLOCK - 1) {
            sBase = tile_base(tau);
            sLast = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
        }
        __syncthreads();
        for (int jj = threadIdx.x; jj < NKU; jj += BLOCK) {
            const int last = jj % N, nw = (jj / N) % N, rr = (jj / (N * N)) % Q, kap = (jj / (N * N * Q)) % NK,
                      s = jj / (N * N * Q * NK);
            const int c = class_of(M, LAT, nw / M, nw % M);
            double2 e = sK[kap][nw][last];
            if (c > 0) {
                e = cmul(e, sEhi[s][kap][c - 1]);
                for (int i = 0; i < S; ++i)
                    if (i != s) e = cmul(e, sIn[s][i][kap][c - 1][fib_digit<N, S>(s, rr, i)]);
            }
            (&KU[s][kap][rr][0][0])[(nw * N + last) ^ (MAP == 0 ? f3_swizzle(rr) : 0)] = e;
        }
        __syncthreads();
        const long long tbase = sBase;
        const int last_t = sLast;
        for (int rd = 0; rd < rounds; ++rd) {
            const int t = rd * 8 * W + fib;
            const bool valid = t < a.T;
            int2 lo;
            double2 X[N][N];  // X[d1][d0], d2 = j
            if constexpr (TW) {  // the stage holds this unit (issued one unit ago)
                mbar_wait(sFull, phase);
                cur = phase;
                phase ^= 1;
                lo = reinterpret_cast<const int2 *>(sE0w + cur * E0B + S * 2 * D * FS)[sfib];
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) {
                        if constexpr (VW == 0) {  // view A: [d2][d1][d0][f]
                            X[d1][d0] = stg[((j * N + d1) * N + d0) * FS + sfib];
                        } else if constexpr (VW == 1) {  // view B: row r of 8 entries (fibre parity, d2)
                            const int r = (d1 * N + d0) * (FS / 2) + (sfib >> 1);
                            X[d1][d0] = stg[r * 8 + ((((sfib & 1) << 2) | j) ^ (r & 7))];
                        } else if constexpr (VW == 2) {  // view C: row r = (d0, d2 / 2, f) of entries (d2 & 1, d1)
                            const int r = (d0 * 2 + (j >> 1)) * FS + sfib;
                            X[d1][d0] = stg[r * 8 + ((((j & 1) << 2) | d1) ^ (r & 7))];
                        } else {  // view D: row r = (d2, d1 / 2, f) of entries (d1 & 1, d0)
                            const int r = (j * 2 + (d1 >> 1)) * FS + sfib;
                            X[d1][d0] = stg[r * 8 + ((((d1 & 1) << 2) | d0) ^ (r & 7))];
                        }
                    }
                const int rn = rd + 1 < rounds ? rd + 1 : 0, taun = rd + 1 < rounds ? tau : tau + 1;
                __syncwarp();  // the warp's stage is free: refill it with the warp's next unit
                if (lane == 0 && taun < t_end) tma_issue(taun, rn, phase);
            } else {
                load_unit(tau, rd, X, lo);
            }
            const long long base = tbase + lo.x;
            const int last0 = lo.y >= 0 ? lo.y : last_t;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == 2) {  // transpose digit 0 <-> digit 2 among the 4 lanes of an outer fibre
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) {  // one digit-1 value at a time (16 entries)
                        if (valid) {
#pragma unroll
                            for (int d0 = 0; d0 < N; ++d0) xch_at(d0 + 4 * j) = X[d1][d0];
                        }
                        if constexpr (MAP == 0) __syncwarp(); else __syncthreads();
                        if (valid) {  // X[d1][d2] := (digit0 = j, digit1 = d1, digit2 = d2)
#pragma unroll
                            for (int d2 = 0; d2 < N; ++d2) X[d1][d2] = xch_at(j + 4 * d2);
                        }
                        if constexpr (MAP == 0) __syncwarp(); else __syncthreads();
                    }
                }
                if (!valid) continue;
                const bool ro = RO && a.rho[s] != nullptr;
                double2 E0[D];  // outer group-0 factor (propagate classes; readout's applied after the step)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    E0[d] = TW ? sE0w[cur * E0B + (s * 2 * D + d) * FS + sfib] : __ldg(&a.Etab[((size_t)s * 2 * a.G * D + d) * a.X + t]);
                double2 acc[RO ? N : 1];
#pragma unroll
                for (int n = 0; n < (RO ? N : 1); ++n) acc[n] = make_double2(0.0, 0.0);
                if (s == 0) {  // fibres along digit 0: X[d1][.], other digits (d1, d2 = j)
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) fibre(X[d1], 0, d1 + 4 * j, last0, ro, E0, acc);
                } else if (s == 1) {  // along digit 1: X[.][d0], other digits (d0, d2 = j); last = d0
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) {
                        double2 xf[N];
#pragma unroll
                        for (int v = 0; v < N; ++v) xf[v] = X[v][d0];
                        fibre(xf, 1, d0 + 4 * j, d0, ro, E0, acc);
#pragma unroll
                        for (int v = 0; v < N; ++v) X[v][d0] = xf[v];
                    }
                } else {  // along digit 2: X[d1][.], other digits (d0 = j, d1); last = d1
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1) fibre(X[d1], 2, j + 4 * d1, d1, ro, E0, acc);
                }
                if (ro) {
                    // the outer factor E0 (fixed for this thread's outer fibre) of the off-diagonal
                    // readout rows, factored out of the sum over its four fibres
#pragma unroll
                    for (int n = 0; n < N; ++n) {
                        const int c = class_of(M, LAT, n / M, n % M);
                        if (c > 0)
                            acc[RO ? n : 0] =
                                cmul(TW ? sE0w[cur * E0B + (s * 2 * D + D + (c > 0 ? c - 1 : 0)) * FS + sfib]
                                        : __ldg(&a.Etab[(((size_t)s * 2 + 1) * a.G * D + (c > 0 ? c - 1 : 0)) * a.X + t]),
                                     acc[RO ? n : 0]);
                    }
#pragma unroll
                    for (int n = 0; n < N; ++n)
                        accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0] =
                            cadd(accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0], acc[RO ? n : 0]);
                }
            }
            if (valid) {  // X[d1][d2] with digit 0 = j
                const long long b0 = base + (long long)j * a.pw_in[0];
                // store path: which inner digit is ring slot 0 follows from the view when it is fixed
                // (view B: d2 = slot 0; view C: d1 = slot 0; views A and D: neither)
                const bool st_d2 = TW ? VW == 1 : a.pw_in[2] == 1;
                const bool st_d1 = TW ? VW == 2 : a.pw_in[1] == 1;
                if (st_d2) {  // d2 is ring slot 0: 32-B stores of adjacent pairs
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                        for (int d2 = 0; d2 < N; d2 += 2) st2_cs(a.A + b0 + (long long)d1 * a.pw_in[1] + d2, X[d1][d2], X[d1][d2 + 1]);
                } else if (st_d1) {
#pragma unroll
                    for (int d1 = 0; d1 < N; d1 += 2)
#pragma unroll
                        for (int d2 = 0; d2 < N; ++d2) st2_cs(a.A + b0 + d1 + (long long)d2 * a.pw_in[2], X[d1][d2], X[d1 + 1][d2]);
                } else {
#pragma unroll
                    for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                        for (int d2 = 0; d2 < N; ++d2)
                            __stcs(a.A + b0 + (long long)d1 * a.pw_in[1] + (long long)d2 * a.pw_in[2], X[d1][d2]);
                }
            }
        }
    }
    if constexpr (RO) {
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr) {
                double2 tt[N];
#pragma unroll
                for (int n = 0; n < N; ++n) tt[n] = accS[RO ? s : 0][RO ? n : 0][RO ? threadIdx.x : 0];
                reduce_finalize<N, BLOCK>(tt, a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                          a.rho_accumulate != 0);
            }
    }
}

// ---------------------------------------------------------------------------------- dispatch
// Launch shapes: plain loads lane map 0 (192 threads, 2 CTAs/SM), lane map 1 (128, 3), per-warp TMA
// (128, 2; one instantiation per stage view).  M = 2: the lattice and general class maps coincide;
// the host uses LAT = false.
namespace {
constexpr int kPlainBlock0 = 192, kPlainMinB0 = 2;
constexpr int kPlainBlock1 = 128, kPlainMinB1 = 3;
constexpr int kTmaBlock = 128, kTmaMinB = 2;

constexpr size_t fused3_dyn(int block, bool ro, bool tw) {
    return ((tw ? (size_t)(block / 32) * (8 * 64 + 2 * (3 * 2 * 2 * 8 + 4)) : 0) + (size_t)(block / 32) * 16 * 8 +
            (ro ? (size_t)3 * 4 * block : 0)) * 16;
}

template <bool SYM, int MAP, int BLOCK, int MINB, int VW>
cudaError_t fused3_t(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    const size_t dyn = fused3_dyn(BLOCK, ro, VW >= 0);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        kern<<<grid, BLOCK, dyn, s>>>(a);
    };
    if (ro) go(k_fused3<SYM, MAP, BLOCK, MINB, VW, true>);
    else go(k_fused3<SYM, MAP, BLOCK, MINB, VW, false>);
    return cudaGetLastError();
}

template <bool SYM, int MAP, int BLOCK, int MINB, int VW>
int fused3_occ_t() {
    int o1 = 0, o2 = 0;
    const size_t d1 = fused3_dyn(BLOCK, true, VW >= 0), d2 = fused3_dyn(BLOCK, false, VW >= 0);
    cudaFuncSetAttribute(k_fused3<SYM, MAP, BLOCK, MINB, VW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d1);
    cudaFuncSetAttribute(k_fused3<SYM, MAP, BLOCK, MINB, VW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d2);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_fused3<SYM, MAP, BLOCK, MINB, VW, true>, BLOCK, d1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused3<SYM, MAP, BLOCK, MINB, VW, false>, BLOCK, d2);
    return o1 < o2 ? o1 : o2;
}

template <bool SYM>
cudaError_t fused3_dispatch(const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    if (a.use_tma) {
        switch (a.tma_view) {
        case 0: return fused3_t<SYM, 0, kTmaBlock, kTmaMinB, 0>(a, ro, grid, s);
        case 1: return fused3_t<SYM, 0, kTmaBlock, kTmaMinB, 1>(a, ro, grid, s);
        case 2: return fused3_t<SYM, 0, kTmaBlock, kTmaMinB, 2>(a, ro, grid, s);
        case 3: return fused3_t<SYM, 0, kTmaBlock, kTmaMinB, 3>(a, ro, grid, s);
        default: return cudaErrorInvalidValue;
        }
    }
    if (a.lane_map == 1) return fused3_t<SYM, 1, kPlainBlock1, kPlainMinB1, -1>(a, ro, grid, s);
    return fused3_t<SYM, 0, kPlainBlock0, kPlainMinB0, -1>(a, ro, grid, s);
}
}  // namespace

int fused3_block(int lane_map, bool tma) { return tma ? kTmaBlock : (lane_map == 1 ? kPlainBlock1 : kPlainBlock0); }
int fused3_round_fibres(int lane_map, bool tma) { return fused3_block(lane_map, tma) / 4; }

cudaError_t launch_fused3(bool sym, const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    return sym ? fused3_dispatch<true>(a, ro, grid, s) : fused3_dispatch<false>(a, ro, grid, s);
}

int fused3_occupancy(bool sym, int lane_map, bool tma) {
    // every TMA view has the same resources (one instantiation per view of the same code shape)
    if (tma) return sym ? fused3_occ_t<true, 0, kTmaBlock, kTmaMinB, 0>() : fused3_occ_t<false, 0, kTmaBlock, kTmaMinB, 0>();
    if (lane_map == 1)
        return sym ? fused3_occ_t<true, 1, kPlainBlock1, kPlainMinB1, -1>() : fused3_occ_t<false, 1, kPlainBlock1, kPlainMinB1, -1>();
    return sym ? fused3_occ_t<true, 0, kPlainBlock0, kPlainMinB0, -1>() : fused3_occ_t<false, 0, kPlainBlock0, kPlainMinB0, -1>();
}

}  // namespace qp
