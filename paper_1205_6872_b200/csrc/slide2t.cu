// slide2t.cu -- k_fused2t: two consecutive slide steps k, k+1 (k >= L) of the iterative tensor
// propagator for M = 3 (N = 9, s = (c, 0, -c)) in ONE pass over HBM, in place on the ring-buffer ARDM, with
// the rho(t_k) readout of both steps fused (the algebra and the step
// fusion are those of slide_r.cu / slide2.cu).  HBM traffic per step: 32/2 = 16 B per ARDM entry.
// The TMA-staged, warp-specialised form of k_fused2s (unsharded launch sets and shard blocks: the
// tensor map is over the block's local layout).
//
// A unit is 27 consecutive outer fibres x the 81 entries of the inner digits (d0, d1) = ring slots
// (p0, p0+1): one TMA box (35 KB) of a tensor map over the ARDM whose shape depends on where ring slot
// 0 sits (view VK, host.cpp: encode_f2t_tmap); the stage holds entry (f, d0, d1) at
//   VK 0 (p0 = 0)        : d0 + 9 d1 + 81 f          (the unit is one contiguous 35 KB block)
//   VK 1 (p0 = L-1)      : d1 + 9 f + 243 d0
//   VK 2 (2 <= p0 <= L-2): f + 27 d0 + 243 d1        (27 consecutive fibres of the run of slots < p0)
//   VK 3 (p0 = 1)        : f%9 + 9 d0 + 81 d1 + 729 (f/9)   (one contiguous block)
// (VK 0, 1, 3 merge the two lowest slots into one box dimension: 27 rows of 1296 B per unit.)
// -- conflict-free 16-B accesses for consecutive fibres in every case.  One CTA per SM, 18 warps:
//   load warp   : unit r into stage r % NS once the stage's previous unit has been stored (empty[b]):
//                 one cp.async.bulk.tensor box + one bulk copy of the unit's outer group-0 factors and
//                 'last' digits, completing on full[b]; also builds each tile's constants;
//   consumers   : two groups of 8 warps take alternate units; thread t < 243 of a group (fibre t % 27,
//                 digit w = t / 27): sub-step 0 the fibre along d0 with d1 = w, group barrier (named),
//                 sub-step 1 along d1 with d0 = w, both in place in the stage; fence the async proxy,
//                 arrive on done[b];
//   store warp  : unit j: wait done[b], one cp.async.bulk.tensor store; once it has read the stage,
//                 arrive on the stage's empty barrier.
// Used for s = (c, 0, -c) (the class moments use the structure of the weights: old-state pairs instead
// of 9 complex products).  13 of a group's 256 threads idle (a box of 27 fibres tiles every view
// exactly: no padding traffic).  Readout: each thread's per-fibre terms go into tensor memory after
// every sub-step (tcgen05.ld / st), the class-moment terms summed per tile without the tile's inner
// factor (applied once per tile); fixed-order CTA and grid reductions at the end (deterministic).
#include "tmem.cuh"

namespace qp {

namespace {
constexpr int kT2N = 9, kT2F = 27;                  // N, outer fibres per unit
constexpr int kT2GW = 8, kT2Groups = 2;             // warps per consumer group, groups (alternate units)
constexpr int kT2Consumers = kT2Groups * kT2GW;     // 16: a group's 256 threads take the 243 fibres of a sub-step
constexpr int kT2Block = 32 * (kT2Consumers + 2);   // + store warp + load warp
constexpr int kT2NS = 5;                            // ring depth
constexpr int kT2Data = 2192;                       // 27 x 81 = 2187 entries, padded to a 128-B multiple
constexpr int kT2D = 4;                             // classes (lattice s, M = 3)
constexpr int kT2E0B = 2 * 2 * kT2D * kT2F + 14;    // unit block: factors [s][kap][d][27] + 27 int2 ('last')

__device__ __forceinline__ void tma_load_5d_t(void *dst, const void *tmap, unsigned long long *bar, const int (&c)[5]) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
        ::"r"(smem_addr(dst)), "l"(tmap), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_5d_t(const void *tmap, const void *src, const int (&c)[5]) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(tmap), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(smem_addr(src)) : "memory");
}
__device__ __forceinline__ void arrive_t(unsigned long long *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void group_sync_t(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(32 * kT2GW) : "memory");
}
// TMA box coordinates of consecutive units: G (first outer fibre of the unit) = cB nA + cA, advanced by
// 27 fibres per unit without division (nA = 0: one coordinate cB = G)
struct Cursor {
    long long cA, cB, nA;
    int dA, dB, mA;  // box dimensions of the two coordinates; cA in units of mA doubles
    __device__ void init(const FusedArgs &a, long long G) {
        nA = a.tma_nA, dA = a.f4_cdimA[0], dB = a.f4_cdimB[0], mA = a.tma_c0m;
        if (nA > 0) cA = G % nA, cB = G / nA; else cA = 0, cB = G;
    }
    __device__ void next() {
        if (nA > 0) {
            cA += kT2F;
            while (cA >= nA) cA -= nA, ++cB;
        } else {
            cB += kT2F;
        }
    }
    __device__ void coords(int (&c)[5]) const {
#pragma unroll
        for (int i = 0; i < 5; ++i) c[i] = 0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if (i == dA) c[i] = (int)(cA * mA);
            if (i == dB) c[i] = (int)cB;
        }
    }
};
}  // namespace

template <int VK, bool RO>
__global__ void __maxnreg__(96) k_fused2t(const __grid_constant__ FusedArgs a, const __grid_constant__ Beta2s bt) {
    constexpr int M = 3, N = kT2N, S = 2, D = kT2D;
    constexpr bool LAT = true;
    constexpr int NU = M * (M + 1) / 2;  // readout accumulators: the upper triangle a <= b
    // stage offset of entry (f, d0, d1): cf(f) + S0 d0 + S1 d1 (16-B units)
    constexpr int S0 = VK == 0 ? 1 : (VK == 1 ? 243 : (VK == 2 ? 27 : 9));
    constexpr int S1 = VK == 0 ? 9 : (VK == 1 ? 1 : (VK == 2 ? 243 : 81));
    const SmallLayout lay{N, D, 0};
    extern __shared__ __align__(128) double2 smem2t[];
    double2 *const sData = smem2t;                       // [kT2NS][kT2Data]
    double2 *const sE0 = smem2t + kT2NS * kT2Data;       // [kT2NS][kT2E0B]
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][2][D][N];  // inner factor of the other inner digit: [s][kap][d][value]
    // class-weight constants [s][kap][d] (see the moments): Re P ch1, Re P sh1, Im P ch1, Im P sh1, ch2, sh2,
    // Re P^2, Im P^2 with ch_j = (R^j + R^-j) / 2, sh_j = (R^j - R^-j) / 2
    __shared__ __align__(16) double sC[S][2][D][8];
    // per tile (double buffered by tile parity, built by the load warp): Ehi (outer groups >= 1) x inner
    // factor of the digit value, and sub-step 0's 'last' when it is a tile digit
    __shared__ double2 sEI[2][S][2][D][N];
    __shared__ int sLast[2];
    __shared__ unsigned tmem_base;
    __shared__ __align__(8) unsigned long long bar_full[kT2NS], bar_done[kT2NS], bar_empty[kT2NS], bar_ei[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto upper_class = [](int d) {
        for (int aa = 0; aa < M; ++aa)
            for (int bb = aa + 1; bb < M; ++bb)
                if (class_of(M, LAT, aa, bb) == d + 1) return true;
        return false;
    };
    const int CH = a.T / kT2F;  // units per tile (host: T % 27 == 0, CH >= 3)
    const long long n_units = (long long)a.n_tiles * CH;
    const long long per = n_units / gridDim.x, rem = n_units % gridDim.x;
    const long long u_begin = (long long)blockIdx.x * per + min((long long)blockIdx.x, rem);
    const long long R = per + ((long long)blockIdx.x < rem ? 1 : 0);
    const int tau0 = (int)(u_begin / CH);
    // ring depth <= units per tile: a tile's table buffer (parity) is rebuilt only after every unit of the
    // tile two back has been stored (the load warp refills a stage only after its previous unit is stored)
    const int NS = min(kT2NS, CH);

    for (int i = tid; i < 2 * N * N; i += kT2Block) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = tid; i < S * 2 * D * N; i += kT2Block) {
        const int s = i / (2 * D * N), kap = (i / (D * N)) % 2, d = (i / N) % D, v = i % N;
        const int other = s == 0 ? 1 : 0;  // sub-step 0: digit 1 (old value); sub-step 1: digit 0 (new value)
        sIn[s][kap][d][v] = a.inner[((((size_t)s * S + other) * 2 + kap) * D + d) * N + v];
    }
    if (tid < S * 2 * D) {  // from the weights of the old states (0,1), (1,0), (0,2), (2,0), (0,0)
        const int s = tid / (2 * D), kap = (tid / D) % 2, d = tid % D;
        const double2 *b = bt.b[s][kap][d];
        const double r1 = hypot(b[1].x, b[1].y), r1i = hypot(b[3].x, b[3].y);
        const double ch1 = 0.5 * (r1 + r1i), sh1 = 0.5 * (r1 - r1i), pr = b[1].x / r1, pi = b[1].y / r1;
        double *c = sC[s][kap][d];
        c[0] = pr * ch1, c[1] = pr * sh1, c[2] = pi * ch1, c[3] = pi * sh1;
        c[4] = 0.5 * (b[2].x + b[6].x), c[5] = 0.5 * (b[2].x - b[6].x);
        c[6] = b[0].x, c[7] = b[0].y;
    }
    if (tid == 0) {
        for (int b = 0; b < kT2NS; ++b) mbar_init(&bar_full[b], 1), mbar_init(&bar_done[b], kT2GW), mbar_init(&bar_empty[b], 1);
        for (int b = 0; b < 2; ++b) mbar_init(&bar_ei[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // readout sums in tensor memory (frees ~26 registers of the 96): consumer warp w owns 64 columns of
    // its lane quarter (warps w, w + 4, w + 8, w + 12 share the lanes 32 (w % 4) .. + 31); blocks of 8
    // columns (4 doubles) at tacc + 8 i: 0 = Re rho_00, Re rho_11, Re rho_22 (sub-step 0); 1 = the plain sum
    // (sub-step 1); the class-moment terms are summed per tile WITHOUT the tile's inner factor EI (a
    // common factor of the tile for the thread's digit w) in 2 = rho_01, rho_02, 3 = rho_12 (sub-step 0),
    // class-(b - a = 1) moment (sub-step 1), 4 = class-(b - a = 2) moment (sub-step 1), and folded (x EI)
    // into 5, 6, 7 (same order) when the tile changes
    if constexpr (RO)
        if (warp == 0) tmem_alloc(&tmem_base, 256);
    // programmatic dependent launch: the setup above overlapped the previous launch's tail
    asm volatile("griddepcontrol.wait;" ::: "memory");
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const unsigned tacc = tmem_base + ((unsigned)(32 * (warp & 3)) << 16) + 64u * (unsigned)((warp >> 2) & 3);
    if constexpr (RO)
        if (warp < kT2Consumers) {
            const double z[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int i = 0; i < 8; ++i) tmem_st_d4(tacc + 8 * i, z);
            tmem_wait_st();
        }

    if (warp < kT2Consumers) {
        // =========================================================== consumer groups
        // thread t of group g: fibre f = t % 27 of the unit, inner digit w = t / 27 (t < 243)
        const int g = warp / kT2GW, t = tid - g * 32 * kT2GW;
        const int f = t % kT2F, w = t / kT2F;
        const bool valid = t < kT2F * kT2N;
        const int cf = VK == 0 ? 81 * f : (VK == 1 ? 9 * f : (VK == 2 ? f : (f % 9) + 729 * (f / 9)));
        long long uu = u_begin + g;
        int tau = (int)(uu / CH), ch = (int)(uu % CH), b = g % NS, ph = (g / NS) & 1;
        int cur_tile = -1, last_t = 0, tp = 0;
        // the tile sums of blocks 2..4 x the tile's EI into blocks 5..7, blocks 2..4 zeroed (warp-collective)
        auto fold = [&](int tpo) {
            if constexpr (RO) {
                const int wc = w < N ? w : N - 1;  // (idle threads: zero sums)
                const double2 e02 = sEI[tpo][0][1][2][wc], e03 = sEI[tpo][0][1][3][wc];
                const double2 e12 = sEI[tpo][1][1][2][wc], e13 = sEI[tpo][1][1][3][wc];
                tmem_wait_st();
                unsigned r[6][8];
#pragma unroll
                for (int i = 0; i < 3; ++i) tmem_ld8_nowait(tacc + 16 + 8 * i, r[i]), tmem_ld8_nowait(tacc + 40 + 8 * i, r[3 + i]);
                tmem_wait_ld();
                double2 x[6][2];
#pragma unroll
                for (int i = 0; i < 6; ++i) tmem_unpack_c2(r[i], x[i][0], x[i][1]);
                tmem_st_c2(tacc + 40, cfma(e02, x[0][0], x[3][0]), cfma(e03, x[0][1], x[3][1]));
                tmem_st_c2(tacc + 48, cfma(e02, x[1][0], x[4][0]), cfma(e12, x[1][1], x[4][1]));
                tmem_st_c2(tacc + 56, cfma(e13, x[2][0], x[5][0]), x[5][1]);
                const double2 z = make_double2(0.0, 0.0);
#pragma unroll
                for (int i = 0; i < 3; ++i) tmem_st_c2(tacc + 16 + 8 * i, z, z);
            }
        };
        for (long long j = g; j < R; j += kT2Groups) {
            if (tau != cur_tile) {
                if (cur_tile >= 0) fold(tp);
                cur_tile = tau;
                tp = (tau - tau0) & 1;
                mbar_wait(&bar_ei[tp], ((tau - tau0) >> 1) & 1);
                last_t = sLast[tp];
            }
            mbar_wait(&bar_full[b], ph);
            double2 *const st = sData + b * kT2Data + cf;
            const double2 *const e0b = sE0 + b * kT2E0B;  // [s][kap][d][27], then 27 int2
            const int lastf = valid ? reinterpret_cast<const int2 *>(e0b + S * 2 * D * kT2F)[f].y : 0;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                // this fibre's readout terms (flushed into tensor memory after the sub-step)
                double2 acc0[RO ? NU : 1], accS1 = make_double2(0.0, 0.0), accM1[RO ? D : 1];
#pragma unroll
                for (int n = 0; n < (RO ? NU : 1); ++n) acc0[n] = make_double2(0.0, 0.0);
#pragma unroll
                for (int n = 0; n < (RO ? D : 1); ++n) accM1[n] = make_double2(0.0, 0.0);
                if (valid) {
                    auto slot = [&](int v) -> double2 & { return s == 0 ? st[S0 * v + S1 * w] : st[S0 * w + S1 * v]; };
                    const int last = s == 0 ? (lastf >= 0 ? lastf : last_t) : w;
                    // s = (c, 0, -c): with eta of the class weights = er + i ei, beta(a, b) = R^(s_a - s_b)
                    // P^(s_a + s_b) (R = e^(-delta er) real, |P| = 1), so the old-state pairs (0,2)/(2,0) have
                    // real weights R^(+-2), (0,0)/(2,2) conjugate weights P^(+-2), (0,1)/(1,0) and (1,2)/(2,1)
                    // weights P^(+-1) R^(+-1), and (1,1) weight 1 (sC per class, below): 16 instead of 36 FP64
                    // operations per class moment; one pair group live at a time
                    const double2 xc = slot(4);
                    double2 S0v = xc, mp[D], mr[RO ? D : 1];
#pragma unroll
                    for (int d = 0; d < D; ++d) mp[d] = xc;
#pragma unroll
                    for (int d = 0; d < (RO ? D : 1); ++d) mr[d] = xc;
                    // fn(class constants, moment, g) for every used (kap, d).  Classes d and d + 2 have opposite
                    // Delta s (R -> 1/R, P -> conj P): class d + 2's moment uses class d's constants with
                    // the signs of sh_j and Im P flipped (g = -1 on c[1], c[2], c[5], c[7])
                    auto each = [&](auto &&fn) {
#pragma unroll
                        for (int d = 0; d < D / 2; ++d) {
                            const double *c = &sC[s][0][d][0];
                            fn(c, mp[d], 1.0);
                            fn(c, mp[d + D / 2], -1.0);
                        }
                        if constexpr (RO)
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                if (upper_class(d)) fn(&sC[s][1][d][0], mr[d], 1.0);
                    };
                    {  // (0,2) / (2,0): real weights ch2 (x + y) + sh2 (x - y)
                        const double2 x = slot(2), y = slot(6), pp = cadd(x, y), qq = csub(x, y);
                        S0v = cadd(S0v, pp);
                        each([&](const double *c, double2 &m, double g) {
                            m.x = fma(c[4], pp.x, fma(g * c[5], qq.x, m.x));
                            m.y = fma(c[4], pp.y, fma(g * c[5], qq.y, m.y));
                        });
                    }
                    {  // (0,0) / (2,2): P^2 x + conj(P^2) y = Re P^2 (x + y) + i Im P^2 (x - y)
                        const double2 x = slot(0), y = slot(8), pp = cadd(x, y), qq = csub(x, y);
                        S0v = cadd(S0v, pp);
                        each([&](const double *c, double2 &m, double g) {
                            m.x = fma(c[6], pp.x, fma(-g * c[7], qq.y, m.x));
                            m.y = fma(c[6], pp.y, fma(g * c[7], qq.x, m.y));
                        });
                    }
                    {  // (0,1)/(1,0) -> A, (1,2)/(2,1) -> B, A = ch1 (x + y) + sh1 (x - y); P A + conj(P) B
                       // = Re P (A + B) + i Im P (A - B): with the per-fibre sums and differences of the two
                       // pairs and c[0..3] = Re P ch1, Re P sh1, Im P ch1, Im P sh1 it is 8 FMA per class
                        const double2 x1 = slot(1), y1 = slot(3), x5 = slot(5), y5 = slot(7);
                        const double2 p1 = cadd(x1, y1), q1 = csub(x1, y1), p5 = cadd(x5, y5), q5 = csub(x5, y5);
                        const double2 P15 = cadd(p1, p5), Q15 = cadd(q1, q5), Pd = csub(p1, p5), Qd = csub(q1, q5);
                        S0v = cadd(S0v, P15);
                        each([&](const double *c, double2 &m, double g) {
                            m.x = fma(c[0], P15.x, fma(g * c[1], Q15.x, fma(-g * c[2], Pd.y, fma(-c[3], Qd.y, m.x))));
                            m.y = fma(c[0], P15.y, fma(g * c[1], Q15.y, fma(g * c[2], Pd.x, fma(c[3], Qd.x, m.y))));
                        });
                    }
                    // class moment x its class factor E0 (outer group 0, this fibre) x EI (tile x inner digit w);
                    // the readout terms leave EI out (applied per tile by fold)
                    auto moment = [&](int kap, int d) {
                        const double2 mm = kap == 0 ? mp[d] : mr[RO ? d : 0];
                        if (kap == 1) return cmul(e0b[((s * 2 + kap) * D + d) * kT2F + f], mm);
                        return cmul(cmul(e0b[((s * 2 + kap) * D + d) * kT2F + f], sEI[tp][s][kap][d][w]), mm);
                    };
                    if constexpr (RO) {  // readout first (upper triangle only: rho_ba = conj rho_ab)
                        if (s == 0) {
                            int u = 0;
#pragma unroll
                            for (int aa = 0; aa < M; ++aa)
#pragma unroll
                                for (int bb = aa; bb < M; ++bb, ++u)
                                    if (aa == bb) {  // the diagonal of rho is real (Hermiticity, C.4): Re only
                                        const double2 k = sK[0][aa * M + bb][last];
                                        acc0[u].x = fma(k.x, S0v.x, fma(-k.y, S0v.y, acc0[u].x));
                                    }
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                if (upper_class(d)) {
                                    const double2 m1 = moment(1, d);
                                    u = 0;
#pragma unroll
                                    for (int aa = 0; aa < M; ++aa)
#pragma unroll
                                        for (int bb = aa; bb < M; ++bb, ++u)
                                            if (aa != bb && class_of(M, LAT, aa, bb) == d + 1)
                                                acc0[u] = cfma(sK[1][aa * M + bb][last], m1, acc0[u]);
                                }
                        } else {
                            accS1 = cadd(accS1, S0v);
#pragma unroll
                            for (int d = 0; d < D; ++d)
                                if (upper_class(d)) accM1[d] = cadd(accM1[d], moment(1, d));
                        }
                    }
                    // propagate, in place: every old value of this fibre has been read above
#pragma unroll
                    for (int nw = 0; nw < N; ++nw)
                        if (class_of(M, LAT, nw / M, nw % M) == 0) slot(nw) = cmul(sK[0][nw][last], S0v);
#pragma unroll
                    for (int d = 0; d < D; ++d) {
                        const double2 m = moment(0, d);
#pragma unroll
                        for (int nw = 0; nw < N; ++nw)
                            if (class_of(M, LAT, nw / M, nw % M) == d + 1) slot(nw) = cmul(sK[0][nw][last], m);
                    }
                }
                if constexpr (RO) {  // every lane (tcgen05 is warp-collective; idle threads add zeros)
                    tmem_wait_st();  // this thread's previous store to the columns has landed
                    if (s == 0) {
                        unsigned ra[8], rb[8], rc[8];
                        tmem_ld8_nowait(tacc, ra), tmem_ld8_nowait(tacc + 16, rb), tmem_ld8_nowait(tacc + 24, rc);
                        tmem_wait_ld();
                        double2 x0, x1, y0, y1, z0, z1;
                        tmem_unpack_c2(ra, x0, x1), tmem_unpack_c2(rb, y0, y1), tmem_unpack_c2(rc, z0, z1);
                        tmem_st_c2(tacc, make_double2(x0.x + acc0[0].x, x0.y + acc0[3].x), make_double2(x1.x + acc0[5].x, 0.0));
                        tmem_st_c2(tacc + 16, cadd(y0, acc0[1]), cadd(y1, acc0[2]));
                        tmem_st_c2(tacc + 24, cadd(z0, acc0[4]), z1);
                    } else {
                        unsigned ra[8], rc[8], re[8];
                        tmem_ld8_nowait(tacc + 8, ra), tmem_ld8_nowait(tacc + 24, rc), tmem_ld8_nowait(tacc + 32, re);
                        tmem_wait_ld();
                        double2 x0, x1, y0, y1, z0, z1;
                        tmem_unpack_c2(ra, x0, x1), tmem_unpack_c2(rc, y0, y1), tmem_unpack_c2(re, z0, z1);
                        tmem_st_c2(tacc + 8, cadd(x0, accS1), x1);
                        tmem_st_c2(tacc + 24, y0, cadd(y1, accM1[2]));
                        tmem_st_c2(tacc + 32, cadd(z0, accM1[3]), z1);
                    }
                }
                if (s == 0) group_sync_t(1 + g);  // sub-step 0 of the whole unit is in the stage
            }
            fence_proxy_async();  // this thread's stage writes -> visible to the TMA store
            __syncwarp();
            if (lane == 0) arrive_t(&bar_done[b]);
            for (int i = 0; i < kT2Groups; ++i) {
                if (++b == NS) b = 0, ph ^= 1;
                if (++ch == CH) ch = 0, ++tau;
            }
        }
        if (cur_tile >= 0) fold(tp);
    } else if (warp == kT2Consumers) {
        // =========================================================== store warp
        if (lane == 0) {
            Cursor cur;
            cur.init(a, u_begin * kT2F);
            // a unit takes a consumer group several microseconds, so the store warp waits for each store to
            // have read its stage and releases the stage at once (the load warp refills it a unit earlier
            // than if the release waited for the next unit's store)
            int b = 0, ph = 0;
            for (long long j = 0; j < R; ++j) {
                mbar_wait(&bar_done[b], ph);
                int c[5];
                cur.coords(c);
                tma_store_5d_t(&a.tmap, sData + b * kT2Data, c);
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                arrive_t(&bar_empty[b]);
                if (++b == NS) b = 0, ph ^= 1;
                cur.next();
            }
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    } else {
        // =========================================================== load warp
        Cursor cur;
        cur.init(a, u_begin * kT2F);
        int b = 0, ph = 1, tau = tau0, ch = (int)(u_begin % CH), built = -1;
        for (long long r = 0; r < R; ++r) {
            if (r >= NS) mbar_wait(&bar_empty[b], ph);
            if (lane == 0) {
                int c[5];
                cur.coords(c);
                mbar_expect_tx(&bar_full[b], (kT2F * N * N + kT2E0B) * 16);
                tma_load_5d_t(sData + b * kT2Data, &a.tmap, &bar_full[b], c);
                bulk_g2s(sE0 + b * kT2E0B, a.E0r + (size_t)ch * kT2E0B, kT2E0B * 16, &bar_full[b]);
            }
            if (tau != built) {  // this tile's constants into buffer (tau - tau0) & 1
                built = tau;
                const int lb = (tau - tau0) & 1;
                for (int i = lane; i < S * 2 * D * N; i += 32) {
                    const int s = i / (2 * D * N), kap = (i / (D * N)) % 2, d = (i / N) % D, v = i % N;
                    double2 e = make_double2(1.0, 0.0);
                    for (int gg = 1; gg < a.G; ++gg)
                        e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + gg) * D + d) * a.X + (tau / a.gdiv[gg]) % a.gmod[gg]]));
                    sEI[lb][s][kap][d][v] = cmul(cmul(e, a.fixfac[s][kap][d]), sIn[s][kap][d][v]);
                }
                if (lane == 0) sLast[lb] = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
                __syncwarp();
                if (lane == 0) arrive_t(&bar_ei[lb]);
            }
            __syncwarp();
            if (++b == NS) b = 0, ph ^= 1;
            if (++ch == CH) ch = 0, ++tau;
            cur.next();
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if constexpr (RO) {
        const int t = tid - (warp / kT2GW) * 32 * kT2GW, w = t / kT2F;
        const bool cons = warp < kT2Consumers && t < kT2F * kT2N;
        double2 acc0[NU], accS1, accM1[D];
        {
            double2 q[16];
            if (warp < kT2Consumers) {
                tmem_wait_st();
#pragma unroll
                for (int i = 0; i < 8; ++i) tmem_ld_c2(tacc + 8 * i, q[2 * i], q[2 * i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) q[i] = make_double2(0.0, 0.0);
            }
            acc0[0] = make_double2(q[0].x, 0.0), acc0[3] = make_double2(q[0].y, 0.0), acc0[5] = make_double2(q[1].x, 0.0);
            accS1 = q[2];
            acc0[1] = q[10], acc0[2] = q[11], acc0[4] = q[12], accM1[2] = q[13], accM1[3] = q[14];
            accM1[0] = accM1[1] = make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (a.rho[s] != nullptr) {
                double2 full[N];  // lower triangle = conj upper (Hermiticity)
                int u = 0;
#pragma unroll
                for (int aa = 0; aa < M; ++aa)
#pragma unroll
                    for (int bb = aa; bb < M; ++bb, ++u) {
                        const int nw = aa * M + bb, c = class_of(M, LAT, aa, bb);
                        double2 v = s == 0 ? acc0[u] : (c == 0 ? cmul(sK[0][nw][w], accS1) : cmul(sK[1][nw][w], accM1[c - 1]));
                        if (aa == bb) v.y = 0.0;  // real diagonal
                        if (!cons) v = make_double2(0.0, 0.0);
                        full[nw] = v;
                        full[bb * M + aa] = make_double2(v.x, -v.y);
                    }
                reduce_finalize<N, kT2Block>(full, a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                             a.rho_accumulate != 0);
            }
        tmem_fence_before();
        __syncthreads();
        if (warp == 0) {
            tmem_fence_after();
            tmem_dealloc(tmem_base, 256);
        }
    }
}

namespace {
constexpr size_t fused2t_dyn() { return (size_t)kT2NS * (kT2Data + kT2E0B) * 16; }
template <int VK, bool RO>
cudaError_t fused2t_t(const FusedArgs &a, const Beta2s &b, int grid, cudaStream_t s) {
    cudaFuncSetAttribute(k_fused2t<VK, RO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused2t_dyn());
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kT2Block);
    cfg.dynamicSmemBytes = fused2t_dyn();
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_fused2t<VK, RO>, a, b);
}
template <int VK>
cudaError_t fused2t_vk(const FusedArgs &a, const Beta2s &b, bool ro, int grid, cudaStream_t s) {
    return ro ? fused2t_t<VK, true>(a, b, grid, s) : fused2t_t<VK, false>(a, b, grid, s);
}
}  // namespace

int fused2t_block() { return kT2Block; }
int fused2t_unit_fibres() { return kT2F; }
int fused2t_e0_block() { return kT2E0B; }
int fused2t_occupancy() {
    int o = 0, o2 = 0;
    cudaFuncSetAttribute(k_fused2t<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused2t_dyn());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused2t<2, true>, kT2Block, fused2t_dyn());
    cudaFuncSetAttribute(k_fused2t<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused2t_dyn());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_fused2t<0, false>, kT2Block, fused2t_dyn());
    return o < o2 ? o : o2;
}
// a.f4_layout = VK (view kind, host.cpp: f2t_view)
cudaError_t launch_fused2t(const FusedArgs &a, const Beta2s &b, bool ro, int grid, cudaStream_t s) {
    switch (a.f4_layout) {
    case 0: return fused2t_vk<0>(a, b, ro, grid, s);
    case 1: return fused2t_vk<1>(a, b, ro, grid, s);
    case 2: return fused2t_vk<2>(a, b, ro, grid, s);
    default: return fused2t_vk<3>(a, b, ro, grid, s);
    }
}

}  // namespace qp
