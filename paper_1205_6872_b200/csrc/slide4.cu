// slide4.cu -- k_fused4: four consecutive slide steps k..k+3 (k >= L) of the iterative tensor
// propagator for M = 2 (N = 4) in ONE pass over HBM, in place on the ring-buffer ARDM, with the
// rho(t_k) readout of every requested step fused (the algebra and
// the step fusion are those of slide_r.cu).  HBM traffic per step: 32/4 = 8 B per ARDM entry.
//
// Super-fibre: the 256 entries of the four inner digits d0..d3 (ring slots p0..p0+3 mod L) of one
// outer fibre.  Sixteen lanes hold one super-fibre, 16 entries each:
//   phase 1 (sub-steps 0, 1: fibres along d0, d1): lane q1 holds fixed (d2, d3), X[d1][d0];
//   phase 2 (sub-steps 2, 3: fibres along d2, d3): lane q2 holds fixed (d0, d1), Y[d3][d2];
// between the phases the 16 lanes transpose through shared memory (__syncwarp only).
//
// Warp specialisation: one CTA per SM of 8 consumer warps in two groups of 4 and 1 producer warp.
// A round is 8 outer fibres (2 per consumer warp, one per half-warp); the groups take alternate
// rounds.  The producer streams rounds through a ring of kF4NS 32 KB shared-memory stages with TMA:
// a 5-D cp.async.bulk.tensor box of the round's 8 x 256 entries (load tensor map) plus one bulk copy
// of the round's outer factors, completing on full[b]; the group's consumers read the stage, run the
// four sub-steps in registers, write the results back into the stage in the store map's layout,
// fence the async proxy and arrive on done[b]; the producer writes each finished stage back with one
// cp.async.bulk.tensor store (store tensor map) as soon as it is done and, once the store has read
// the stage, refills it with the round kF4NS ahead.  The load and store maps order the box dimensions
// (host.cpp: f4_layout) so that the phase-1 reads and the phase-2 writes are free of bank conflicts
// under the 128-B swizzle; the transpose uses its own conflict-free placement inside the stage.
//
// Factors (no transcendental in the kernel): an output row nw of a fibre at sub-step s gets
//   K'(nw, last) x inner factor of the lane-varying inner digit   (KU, CTA-wide, built once)
//   x inner factors of the lane-fixed inner digits x outer digit groups >= 1   (LF, per tile)
//   x outer group-0 factor of the fibre                                   (E0, per round)
// Readout: Re rho_00, Re rho_11 and rho_01 per step (rho_10 = conj rho_01 and a real diagonal: rho(t)
// is Hermitian), per-thread shared-memory accumulators, fixed-order reduction at the end.
#include "tmem.cuh"

namespace qp {

namespace {

#ifndef QP_F4_GROUPS
#define QP_F4_GROUPS 2
#endif
#ifndef QP_F4_NS
#define QP_F4_NS 6
#endif
constexpr int kF4Groups = QP_F4_GROUPS;             // consumer groups of 4 warps (alternate rounds)
constexpr int kF4Consumers = 4 * kF4Groups;         // consumer warps
constexpr int kF4Block = 32 * (kF4Consumers + 2);  // + a store warp and a load warp
constexpr int kF4NS = QP_F4_NS;                     // stages in the ring
constexpr int kF4F = 8;                            // outer fibres per round
constexpr int kF4Stage = kF4F * 256;               // entries per stage (32 KB)
constexpr int kF4E0B = 4 * 2 * 2 * kF4F + kF4F / 2;  // E0 block: factors [s][kap][c][f] + 8 int2 (offset, 'last' digit)

__device__ __forceinline__ void tma_load_5dc(void *dst, const void *tmap, unsigned long long *bar, int c0, int c1, int c2,
                                             int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_addr(dst)), "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_5dc(const void *tmap, const void *src, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(src)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
// 128-B swizzle of a stage offset in 16-B units (stage 1024-B aligned): chunk bits 0-2 ^= bits 3-5
__device__ __forceinline__ int swz(int o, int on) { return on ? o ^ ((o >> 3) & 7) : o; }

// TMA box coordinates of the round whose first outer fibre is G (FusedArgs::f4_*).
struct Coords {
    int c[5];
};
__device__ __forceinline__ Coords f4_coords(const FusedArgs &a, long long G, int which) {
    Coords k{{0, 0, 0, 0, 0}};
    const int dA = a.f4_cdimA[which], dB = a.f4_cdimB[which];
    const long long nA = a.tma_nA;
    const int sh = a.tma_nA_log2;  // power-of-two run length (M = 2): shifts, no 64-bit division
    const long long q = sh >= 0 ? (G >> sh) : G / nA, rm = sh >= 0 ? (G & (nA - 1)) : G - q * nA;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (i == dA) k.c[i] = (int)(a.tma_c0m * rm);
        if (i == dB) k.c[i] = (int)q;
    }
    return k;
}

}  // namespace

template <bool SYM, bool RO, int LT>
__global__ void __maxnreg__(168) k_fused4(const __grid_constant__ FusedArgs a) {
    constexpr int M = 2, N = 4, S = 4, D = 2;
    constexpr bool LAT = false;
    constexpr int NK = RO ? 2 : 1;
    extern __shared__ __align__(1024) double2 smem4[];
    double2 *const stage = smem4;                                    // [kF4NS][kF4Stage]
    double2 *const sE0 = smem4 + kF4NS * kF4Stage;                   // [kF4NS][kF4E0B]
    double2 *const sLF = sE0 + kF4NS * kF4E0B;                       // [2][S][NK][D][16]
    double2 *const sKU = sLF + 2 * S * 2 * D * 16;                   // [S][NK][4 vd][N nw][N last]
    __shared__ double2 sBeta[S][2][D][N];
    __shared__ double2 sQ[S * 2 * D * 16];  // [S][NK][D][16] (tile-independent part of LF)
    __shared__ unsigned tmem_base;
    __shared__ __align__(8) unsigned long long bar_full[kF4NS], bar_done[kF4NS], bar_empty[kF4NS], bar_lf[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const SmallLayout lay{N, D, 0};

    const int per = a.n_tiles / (int)gridDim.x, rem = a.n_tiles % (int)gridDim.x;
    const int t_begin = (int)blockIdx.x * per + min((int)blockIdx.x, rem);
    const int t_end = t_begin + per + ((int)blockIdx.x < rem ? 1 : 0);
    const int rounds = a.T / kF4F;                 // >= 2 (host: T >= 16)
    const int R = (t_end - t_begin) * rounds;      // this CTA's rounds, in order
    // ring depth: the load warp refills the stage of round j with round j + NS once j has been stored and
    // builds a tile's LF table (buffer tile & 1) only then, so every round of the tile two back is done
    // when NS <= rounds + 1
    const int NS = min(kF4NS, rounds + 1);
    constexpr int kLoadWarp = kF4Consumers + 1;
    auto issue_load = [&](int b, int tau, int rd) {  // lane 0 of the load warp: round (tau, rd) into stage b
        fence_proxy_async();
        mbar_expect_tx(&bar_full[b], kF4Stage * 16 + kF4E0B * 16);
        const Coords k = f4_coords(a, (long long)tau * a.T + (long long)rd * kF4F, 0);
        tma_load_5dc(stage + b * kF4Stage, &a.tmap, &bar_full[b], k.c[0], k.c[1], k.c[2], k.c[3], k.c[4]);
        bulk_g2s(sE0 + b * kF4E0B, a.E0r + (size_t)rd * kF4E0B, kF4E0B * 16, &bar_full[b]);
    };

    // ---- CTA-wide setup.  The load warp initialises the barriers and puts the first NS rounds in
    // flight while the other warps build KU (tile independent) and beta; warp 0 allocates TMEM.
    if (warp == kLoadWarp) {
        if (lane == 0) {
            for (int b = 0; b < kF4NS; ++b) {
                mbar_init(&bar_full[b], 1);
                mbar_init(&bar_done[b], 4);
                mbar_init(&bar_empty[b], 1);
            }
            for (int b = 0; b < 2; ++b) mbar_init(&bar_lf[b], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            // programmatic dependent launch: everything above overlapped the previous launch's tail;
            // the ARDM it writes is read from here on
            asm volatile("griddepcontrol.wait;" ::: "memory");
            for (int r = 0; r < min(R, NS); ++r) issue_load(r, t_begin + r / rounds, r % rounds);
        }
    } else {
        constexpr int kSetup = kF4Block - 32;
        for (int i = tid; i < S * NK * 4 * N * N; i += kSetup) {
            const int last = i % N, nw = (i / N) % N, vd = (i / (N * N)) % 4, kap = (i / (N * N * 4)) % NK, s = i / (N * N * 4 * NK);
            // lane-varying inner digit of sub-step s: s = 0 -> d1, 1 -> d0, 2 -> d3, 3 -> d2
            const int iv = s == 0 ? 1 : (s == 1 ? 0 : (s == 2 ? 3 : 2));
            const int c = class_of(M, LAT, nw / M, nw % M);
            double2 e = a.small[lay.kp(kap) + nw * N + last];
            if (c > 0) e = cmul(e, a.inner[((((size_t)s * S + iv) * 2 + kap) * D + (c - 1)) * N + vd]);
            sKU[i] = e;
        }
        for (int i = tid; i < S * 2 * D * N; i += kSetup) {
            const int s_ = i / (2 * D * N), kap = (i / (D * N)) % 2, r_ = i % (D * N);
            (&sBeta[0][0][0][0])[i] = a.small[lay.beta(a.var[s_], kap) + r_];
        }
        // sQ[s][kap][c][q] = shard-digit factor x inner factors of the two lane-fixed digits of lane
        // mapping q (tile independent; a tile's LF multiplies in its outer groups >= 1)
        for (int i = tid; i < S * NK * D * 16; i += kSetup) {
            const int q = i % 16, c = (i / 16) % D, kap = (i / (16 * D)) % NK, s = i / (16 * D * NK);
            int da, db, ia, ib;  // the two lane-fixed digits (ia, ib) and their values for lane q
            if (s < 2) {
                ia = 2, ib = 3;
                if (a.f4_q1swap) db = q & 3, da = q >> 2; else da = q & 3, db = q >> 2;
            } else {
                ia = 0, ib = 1;
                if (a.f4_q2swap) db = q & 3, da = q >> 2; else da = q & 3, db = q >> 2;
            }
            double2 e = a.fixfac[s][kap][c];
            e = cmul(e, a.inner[((((size_t)s * S + ia) * 2 + kap) * D + c) * N + da]);
            e = cmul(e, a.inner[((((size_t)s * S + ib) * 2 + kap) * D + c) * N + db]);
            sQ[i] = e;
        }
    }
    // readout accumulators in TMEM: 32 columns per consumer thread (warps w, w + 4 share lanes: columns
    // 32 (w / 4) .. + 31), allocated by warp 0, zeroed by their threads
    if constexpr (RO)
        if (warp == 0) tmem_alloc(&tmem_base, 32 * kF4Groups);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous launch's ARDM / readout writes visible
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const unsigned tacc = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + 32u * (unsigned)(warp >> 2);
    if constexpr (RO)
        if (warp < kF4Consumers) {
            const double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int s = 0; s < S; ++s) tmem_st_d4(tacc + 8 * s, z);
            tmem_wait_st();
        }

    if (warp == kF4Consumers) {
        // =========================================================== store warp
        // round j: wait for its group (done), store the stage; once the store of round j - 1 has read
        // its stage (bulk wait_group.read 1: the store of j may still be reading), release that stage.
        // Stage index / phase / tile position advance incrementally (no divisions in the chain).
        if (lane == 0) {
            int b = 0, ph = 0, bp = 0, tau = t_begin, rd = 0;
            for (int j = 0; j < R; ++j) {
                mbar_wait(&bar_done[b], ph);
                const Coords k = f4_coords(a, (long long)tau * a.T + (long long)rd * kF4F, 1);
                tma_store_5dc(&a.tmapS, stage + b * kF4Stage, k.c[0], k.c[1], k.c[2], k.c[3], k.c[4]);
                bulk_commit();
                if (j >= 1) {
                    bulk_wait_read1();
                    mbar_arrive(&bar_empty[bp]);
                }
                bp = b;
                if (++b == NS) b = 0, ph ^= 1;
                if (++rd == rounds) rd = 0, ++tau;
            }
            bulk_wait0();
        }
    } else if (warp == kF4Consumers + 1) {
        // =========================================================== load warp
        // round r into stage r % NS once the stage's previous round (r - NS) has been stored and read.
        // A tile's LF = Ehi(tile)[s][kap][c] x sQ[s][kap][c][q]: lanes 0..15 form the 16 outer-group
        // products (independent loads), every lane then 8 entries from the CTA's sQ table.
        int b = 0, ph = 1, tau = t_begin, rd = 0;
        for (int r = 0; r < R; ++r) {
            if (r >= NS) {  // (rounds < NS went out during the setup)
                mbar_wait(&bar_empty[b], ph);
                if (lane == 0) issue_load(b, tau, rd);
            }
            if (rd == 0) {  // (after the round's TMA load is in flight: consumers wait for both)
                // this tile's LF (buffer tau & 1: every round of tile tau - 2 has been stored, as NS <= rounds + 1)
                const int lb = (tau - t_begin) & 1;
                double2 e = make_double2(1.0, 0.0);
                if (lane < S * NK * D) {
                    const int c = lane % D, kap = (lane / D) % NK, s = lane / (D * NK);
                    for (int g = 1; g < a.G; ++g)
                        e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + c) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
                }
#pragma unroll
                for (int i0 = 0; i0 < S * NK * D * 16; i0 += 32) {
                    const int i = i0 + lane, src = i / 16;
                    const double2 eh = make_double2(__shfl_sync(0xffffffffu, e.x, src), __shfl_sync(0xffffffffu, e.y, src));
                    sLF[(size_t)lb * S * 2 * D * 16 + i] = cmul(eh, sQ[i]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_lf[lb]);
            }
            __syncwarp();
            if (++b == NS) b = 0, ph ^= 1;
            if (++rd == rounds) rd = 0, ++tau;
        }
    } else {
        // =========================================================== consumer warps
        // stage layout: compile-time for the common layout types (LT > 0), else from the launch arguments
        constexpr int kLP[4][11] = {{0}, {6, 7, 8, 9, 3, 4, 5, 10, 0, 1, 2}, {0, 1, 2, 6, 3, 4, 5, 7, 8, 9, 10},
                                    {4, 5, 6, 7, 0, 1, 2, 3, 8, 9, 10}};
        constexpr int kSP[4][11] = {{0}, {3, 4, 5, 6, 7, 8, 9, 10, 0, 1, 2}, {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10},
                                    {3, 4, 5, 7, 0, 1, 2, 6, 8, 9, 10}};
        int lpos[11], spos[11];
#pragma unroll
        for (int i = 0; i < 11; ++i) lpos[i] = LT ? kLP[LT][i] : a.f4_lpos[i], spos[i] = LT ? kSP[LT][i] : a.f4_spos[i];
        const int q1swap = LT ? 0 : a.f4_q1swap, q2swap = LT ? 0 : a.f4_q2swap;
        const int colreg = LT ? (LT == 1) : a.f4_colregion, swon = LT ? 1 : a.f4_swz;
        const int h = lane >> 4, q = lane & 15;
        const int grp = warp >> 2;          // consumer group: rounds grp, grp + kF4Groups, ...
        const int f = 2 * (warp & 3) + h;   // fibre of this half-warp within the round
        // phase-1 lane digits (d2, d3) and phase-2 lane digits (d0, d1)
        const int l2 = q1swap ? (q >> 2) : (q & 3), l3 = q1swap ? (q & 3) : (q >> 2);
        const int l0 = q2swap ? (q >> 2) : (q & 3), l1 = q2swap ? (q & 3) : (q >> 2);
        // stage offsets (16-B units, before the swizzle): bit b of digit i contributes 1 << pos[2i + b]
        auto dig_off = [&](const int *pos, int i, int v) { return ((v & 1) << pos[2 * i]) + ((v >> 1) << pos[2 * i + 1]); };
        const int fofsL = ((f & 1) << lpos[8]) + (((f >> 1) & 1) << lpos[9]) + ((f >> 2) << lpos[10]);
        const int fofsS = ((f & 1) << spos[8]) + (((f >> 1) & 1) << spos[9]) + ((f >> 2) << spos[10]);
        const int baseL = fofsL + dig_off(lpos, 2, l2) + dig_off(lpos, 3, l3);
        const int baseS = fofsS + dig_off(spos, 0, l0) + dig_off(spos, 1, l1);
        // transpose placement of entry (d0..d3) of fibre f: p = (q1 & 7) ^ (q2 & 7), rho = q2 & 7 | (q1 >> 3) << 3 | (q2 >> 3) << 4
        auto q1v = [&](int d2, int d3) { return q1swap ? d3 + 4 * d2 : d2 + 4 * d3; };
        auto q2v = [&](int d0, int d1) { return q2swap ? d1 + 4 * d0 : d0 + 4 * d1; };
        auto xpos = [&](int qa, int qb) {  // qa = q1 value, qb = q2 value -> physical stage offset
            const int p = (qa & 7) ^ (qb & 7), rho = (qb & 7) + 8 * (qa >> 3) + 16 * (qb >> 3);
            // col-region: fibre f owns chunk f ^ (row & 7) (swizzled) or f (dense) of every row
            return colreg ? (p + 8 * rho) * 8 + (swon ? f ^ p : f) : (32 * f + rho) * 8 + p;
        };

        // one fibre at sub-step s: xf = old values along the contracted digit -> new values.
        // vd = value of the lane-varying inner digit, last = previous time point's value.
        auto fibre = [&](double2 (&xf)[N], int s, int vd, int last, bool ro, const double2 (&E0e)[D], double2 &t01,
                         double &a00, double &a11) {
            double2 S0, m0[D], m10;
            if constexpr (SYM) {
                const double2 uu = cadd(xf[0], xf[3]), w = csub(xf[0], xf[3]);
                const double2 p = cadd(xf[1], xf[2]), qq = csub(xf[1], xf[2]);
                S0 = cadd(uu, p);
                {
                    const double cr = a.sym[s][0][0], ci = a.sym[s][0][1], ch = a.sym[s][0][2], sh = a.sym[s][0][3];
                    const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                    const double2 Bv = make_double2(fma(-ci, w.y, sh * qq.x), fma(ci, w.x, sh * qq.y));
                    m0[0] = cadd(A, Bv);
                    m0[1] = csub(A, Bv);
                }
                if (ro) {
                    const double cr = a.sym[s][1][0], ci = a.sym[s][1][1], ch = a.sym[s][1][2], sh = a.sym[s][1][3];
                    const double2 A = make_double2(fma(cr, uu.x, ch * p.x), fma(cr, uu.y, ch * p.y));
                    const double2 Bv = make_double2(fma(-ci, w.y, sh * qq.x), fma(ci, w.x, sh * qq.y));
                    m10 = cadd(A, Bv);
                }
            } else {
                S0 = cadd(cadd(xf[0], xf[1]), cadd(xf[2], xf[3]));
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double2 mm = cmul(sBeta[s][0][d][0], xf[0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) mm = cfma(sBeta[s][0][d][v], xf[v], mm);
                    m0[d] = mm;
                }
                if (ro) {
                    double2 mm = cmul(sBeta[s][1][0][0], xf[0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) mm = cfma(sBeta[s][1][0][v], xf[v], mm);
                    m10 = mm;
                }
            }
            const double2 *ku0 = sKU + ((s * NK + 0) * 4 + vd) * N * N + last;  // [nw * N]
            const double2 P0 = cmul(E0e[0], m0[0]), P1 = cmul(E0e[1], m0[1]);
            xf[0] = cmul(ku0[0 * N], S0);
            xf[3] = cmul(ku0[3 * N], S0);
            xf[1] = cmul(ku0[1 * N], P0);  // class 1 = (0, 1)
            xf[2] = cmul(ku0[2 * N], P1);  // class 2 = (1, 0)
            if (ro) {
                const double2 *ku1 = sKU + ((s * NK + (NK - 1)) * 4 + vd) * N * N + last;
                a00 += xf[0].x;
                a11 += xf[3].x;
                t01 = cfma(ku1[1 * N], m10, t01);
            }
        };
        // per lane and sub-step: the fibre's outer factor E0eff[kap][c] = E0[s][kap][c][f] x LF[s][kap][c][q]
        auto e0eff = [&](const double2 *e0b, const double2 *lf, int s, int kap, int c) {
            return cmul(e0b[((s * 2 + kap) * D + c) * kF4F + f], lf[((s * NK + kap) * D + c) * 16 + q]);
        };
        // readout: per consumer thread Re rho_00, Re rho_11, rho_01 (re, im) per sub-step in shared memory
        // readout: Re rho_00, Re rho_11, rho_01 (re, im) of sub-step s in TMEM columns 8 s .. 8 s + 7
        auto flush = [&](int s, double a00, double a11, double2 t01, const double2 &E0t) {
            double p[4];
            tmem_wait_st();  // this thread's previous store to the columns (a sub-step ago) has landed
            tmem_ld_d4(tacc + 8 * s, p);
            p[0] += a00;
            p[1] += a11;
            p[2] = fma(E0t.x, t01.x, fma(-E0t.y, t01.y, p[2]));
            p[3] = fma(E0t.x, t01.y, fma(E0t.y, t01.x, p[3]));
            tmem_st_d4(tacc + 8 * s, p);
        };

        int cur = -1, last_t = 0;
        const double2 *lf = sLF;
        // round r = grp, grp + kF4Groups, ...: stage b, its phase ph and tile tau advance incrementally
        int b = grp % NS, ph = (grp / NS) & 1, tau = t_begin + grp / rounds, rd = grp % rounds;
        for (int r = grp; r < R; r += kF4Groups) {
            if (tau != cur) {  // a new tile: its LF table (buffer tau & 1) and sub-step 0's 'last' digit
                cur = tau;
                const int lb = (tau - t_begin) & 1;
                mbar_wait(&bar_lf[lb], ((tau - t_begin) >> 1) & 1);
                lf = sLF + (size_t)lb * S * 2 * D * 16;
                last_t = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
            }
            {
                mbar_wait(&bar_full[b], ph);
                double2 *const st = stage + b * kF4Stage;
                const double2 *const e0b = sE0 + b * kF4E0B;
                const int lastf = reinterpret_cast<const int2 *>(e0b + 4 * 2 * 2 * kF4F)[f].y;
                const int last0 = lastf >= 0 ? lastf : last_t;
                // ---------------- phase 1: X[d1][d0] of lane (d2, d3) = (l2, l3)
                double2 X[N][N];
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0)
                        X[d1][d0] = st[swz(baseL + dig_off(lpos, 0, d0) + dig_off(lpos, 1, d1), swon)];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    constexpr bool ro = RO;  // every sub-step reads out; steps without output are not reduced
                    double2 E0e[D], E0t = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < D; ++c) E0e[c] = e0eff(e0b, lf, s, 0, c);
                    if (ro) E0t = e0eff(e0b, lf, s, NK - 1, 0);
                    double2 t01 = make_double2(0.0, 0.0);
                    double a00 = 0.0, a11 = 0.0;
                    if (s == 0) {
#pragma unroll
                        for (int d1 = 0; d1 < N; ++d1) fibre(X[d1], 0, d1, last0, ro, E0e, t01, a00, a11);
                    } else {
#pragma unroll
                        for (int d0 = 0; d0 < N; ++d0) {
                            double2 xf[N];
#pragma unroll
                            for (int v = 0; v < N; ++v) xf[v] = X[v][d0];
                            fibre(xf, 1, d0, d0, ro, E0e, t01, a00, a11);
#pragma unroll
                            for (int v = 0; v < N; ++v) X[v][d0] = xf[v];
                        }
                    }
                    if (ro) flush(s, a00, a11, t01, E0t);
                }
                // ---------------- transpose (inside the warp's part of the stage)
                __syncwarp();
#pragma unroll
                for (int d1 = 0; d1 < N; ++d1)
#pragma unroll
                    for (int d0 = 0; d0 < N; ++d0) st[xpos(q1v(l2, l3), q2v(d0, d1))] = X[d1][d0];
                __syncwarp();
                double2 Y[N][N];  // Y[d3][d2] of lane (d0, d1) = (l0, l1)
#pragma unroll
                for (int d3 = 0; d3 < N; ++d3)
#pragma unroll
                    for (int d2 = 0; d2 < N; ++d2) Y[d3][d2] = st[xpos(q1v(d2, d3), q2v(l0, l1))];
                // ---------------- phase 2: sub-steps 2 (along d2, last = d1) and 3 (along d3, last = d2)
#pragma unroll
                for (int s = 2; s < 4; ++s) {
                    constexpr bool ro = RO;  // every sub-step reads out; steps without output are not reduced
                    double2 E0e[D], E0t = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < D; ++c) E0e[c] = e0eff(e0b, lf, s, 0, c);
                    if (ro) E0t = e0eff(e0b, lf, s, NK - 1, 0);
                    double2 t01 = make_double2(0.0, 0.0);
                    double a00 = 0.0, a11 = 0.0;
                    if (s == 2) {
#pragma unroll
                        for (int d3 = 0; d3 < N; ++d3) fibre(Y[d3], 2, d3, l1, ro, E0e, t01, a00, a11);
                    } else {
#pragma unroll
                        for (int d2 = 0; d2 < N; ++d2) {
                            double2 xf[N];
#pragma unroll
                            for (int v = 0; v < N; ++v) xf[v] = Y[v][d2];
                            fibre(xf, 3, d2, d2, ro, E0e, t01, a00, a11);
#pragma unroll
                            for (int v = 0; v < N; ++v) Y[v][d2] = xf[v];
                        }
                    }
                    if (ro) flush(s, a00, a11, t01, E0t);
                }
                // ---------------- results into the stage in the store map's layout, then release it
                __syncwarp();
#pragma unroll
                for (int d3 = 0; d3 < N; ++d3)
#pragma unroll
                    for (int d2 = 0; d2 < N; ++d2)
                        st[swz(baseS + dig_off(spos, 2, d2) + dig_off(spos, 3, d3), swon)] = Y[d3][d2];
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_done[b]);
            }
            if ((b += kF4Groups) >= NS) b -= NS, ph ^= 1;
            if ((rd += kF4Groups) >= rounds) rd -= rounds, ++tau;
        }
    }
    // the next launch (programmatic dependent launch) may start its setup on SMs this grid frees
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __syncthreads();  // every warp (incl. the store warp's last bulk wait) is done
    if constexpr (RO) {
        // one fixed-order grid reduction of the four steps' per-thread accumulators (the producer warps
        // contribute 0); the stages are free now and hold the scratch
        // per step two values: (Re rho_00, Re rho_11) and rho_01 (rho_10 = conj rho_01)
        double2 tt[2 * S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (warp < kF4Consumers) {
                double p[4];
                tmem_wait_st();
                tmem_ld_d4(tacc + 8 * s, p);
                tt[2 * s] = make_double2(p[0], p[1]), tt[2 * s + 1] = make_double2(p[2], p[3]);
            } else {
                tt[2 * s] = tt[2 * s + 1] = make_double2(0.0, 0.0);
            }
        }
        grid_sum_multi<2 * S, kF4Block>(tt, stage, a.partials, a.counter, [&](int v, double2 x) {
            double2 *r = a.rho[v / 2];
            if (r == nullptr) return;
            const bool acc = a.rho_accumulate != 0;
            if (v & 1) {
                r[1] = acc ? cadd(r[1], x) : x;
                const double2 xc = make_double2(x.x, -x.y);
                r[2] = acc ? cadd(r[2], xc) : xc;
            } else {
                r[0] = acc ? make_double2(r[0].x + x.x, r[0].y) : make_double2(x.x, 0.0);
                r[3] = acc ? make_double2(r[3].x + x.y, r[3].y) : make_double2(x.y, 0.0);
            }
        });
        tmem_fence_before();
        __syncthreads();
        if (warp == 0) {
            tmem_fence_after();
            tmem_dealloc(tmem_base, 32 * kF4Groups);
        }
    }
}

// ---------------------------------------------------------------------------------- dispatch
namespace {
constexpr size_t fused4_dyn() {
    return (size_t)(kF4NS * kF4Stage + kF4NS * kF4E0B + 2 * 4 * 2 * 2 * 16 + 4 * 2 * 4 * 16) * 16;
}
template <bool SYM, bool RO, int LT>
cudaError_t fused4_t(const FusedArgs &a, int grid, cudaStream_t s) {
    const size_t dyn = fused4_dyn();
    cudaFuncSetAttribute(k_fused4<SYM, RO, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    // programmatic dependent launch: the CTA setup (tables, barriers, TMEM) of this launch overlaps the
    // tail of the previous one; the kernel waits (griddepcontrol.wait) before it touches the ARDM
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kF4Block);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_fused4<SYM, RO, LT>, a);
}
template <bool SYM, bool RO>
cudaError_t fused4_lt(const FusedArgs &a, int grid, cudaStream_t s) {
    switch (a.f4_layout) {
    case 1: return fused4_t<SYM, RO, 1>(a, grid, s);
    case 2: return fused4_t<SYM, RO, 2>(a, grid, s);
    case 3: return fused4_t<SYM, RO, 3>(a, grid, s);
    default: return fused4_t<SYM, RO, 0>(a, grid, s);
    }
}
template <bool SYM, bool RO>
int fused4_occ_t() {
    int o = 0;
    const size_t dyn = fused4_dyn();
    cudaFuncSetAttribute(k_fused4<SYM, RO, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused4<SYM, RO, 0>, kF4Block, dyn);
    return o;
}
}  // namespace

int fused4_block() { return kF4Block; }
int fused4_round_fibres() { return kF4F; }
int fused4_e0_block() { return kF4E0B; }

// the compile-time stage layouts of k_fused4<.., LT> (load, store), LT = 1 (slot 0 outer), 2 (slot 0 = inner
// digit 0), 3 (slot 0 = inner digit 2); the host uses LT only when its layout search found exactly these
int fused4_layout_type(const int (&lpos)[11], const int (&spos)[11], int q1swap, int q2swap, int swz) {
    static const int LP[4][11] = {{0}, {6, 7, 8, 9, 3, 4, 5, 10, 0, 1, 2}, {0, 1, 2, 6, 3, 4, 5, 7, 8, 9, 10},
                                  {4, 5, 6, 7, 0, 1, 2, 3, 8, 9, 10}};
    static const int SP[4][11] = {{0}, {3, 4, 5, 6, 7, 8, 9, 10, 0, 1, 2}, {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10},
                                  {3, 4, 5, 7, 0, 1, 2, 6, 8, 9, 10}};
    if (q1swap || q2swap || !swz) return 0;
    for (int t = 1; t < 4; ++t) {
        bool eq = true;
        for (int i = 0; i < 11; ++i) eq = eq && LP[t][i] == lpos[i] && SP[t][i] == spos[i];
        if (eq) return t;
    }
    return 0;
}

cudaError_t launch_fused4(bool sym, const FusedArgs &a, bool ro, int grid, cudaStream_t s) {
    if (sym) return ro ? fused4_lt<true, true>(a, grid, s) : fused4_lt<true, false>(a, grid, s);
    return ro ? fused4_lt<false, true>(a, grid, s) : fused4_lt<false, false>(a, grid, s);
}

int fused4_occupancy(bool sym) {
    const int a = sym ? fused4_occ_t<true, true>() : fused4_occ_t<false, true>();
    const int b = sym ? fused4_occ_t<true, false>() : fused4_occ_t<false, false>();
    return a < b ? a : b;
}

}  // namespace qp
