// slide2.cu -- k_fused2s: two consecutive slide steps k, k+1 (k >= L) of the iterative tensor
// propagator for M = 3 (N = 9) in ONE pass over HBM, in place on the ring-buffer ARDM, with the
// rho(t_k) readout of both steps fused (the algebra and the step
// fusion are those of slide_r.cu).  HBM traffic per step: 32/2 = 16 B per ARDM entry.
//
// The 81-entry super-fibre of an outer fibre is too large for one thread's registers, so a CTA of 9
// warps stages units of 32 consecutive outer fibres x 81 entries (41.5 KB) in shared memory, double
// buffered with cp.async (unit u+1 lands while unit u is computed):
//   load / store : warp w moves rows e = w, w + 9, ... (e = d0 + 9 d1), lane = outer fibre
//                  (coalesced along the lowest outer slot);
//   sub-step 0   : thread (w, lane) takes the fibre along d0 with d1 = w -- the inner
//                  combination is warp-uniform; last = the outer slot p0-1;
//   sub-step 1   : thread (w, lane) takes the fibre along d1 with d0 = w; last = d0 = w.
// Class factors per fibre: E0 (outer group 0, per fibre; copied into shared memory with the unit) x Ehi (outer groups >= 1, per tile) x the
// inner factor of the other inner digit; K' from a CTA-wide table.  Readout accumulators in
// registers, fixed-order CTA reduction at the end (deterministic).
#include "common.cuh"

namespace qp {

namespace {
constexpr int kF2N = 9, kF2Block = 288, kF2F = 32;  // N, threads (9 warps), outer fibres per unit
}

template <bool LAT, bool RO>
__global__ void __maxnreg__(96) k_fused2s(const __grid_constant__ FusedArgs a, const __grid_constant__ Beta2s bt) {
    constexpr int M = 3, N = kF2N, S = 2, D = n_classes(M, LAT), NS = N * N, W = kF2Block / 32;
    constexpr int NU = M * (M + 1) / 2;  // readout accumulators: the upper triangle a <= b
    static_assert(W == N, "one warp per value of the inner digit");
    const SmallLayout lay{N, D, 0};
    extern __shared__ __align__(16) double2 smem2[];
    double2(*stage)[NS][kF2F] = reinterpret_cast<double2(*)[NS][kF2F]>(smem2);  // [2][81][32]
    // the unit's outer group-0 factors E0[s][kap][d][fibre], copied with the unit: [2][S][2][D][32]
    double2(*sE0u)[S][2][D][kF2F] = reinterpret_cast<double2(*)[S][2][D][kF2F]>(smem2 + 2 * NS * kF2F);
    __shared__ double2 sK[2][N][N];
    __shared__ double2 sIn[S][2][D][N];     // inner factor of the other inner digit: [s][kap][d][value]
    // per tile (double buffered by tile parity: written while other warps may still read the previous
    // tile's): Ehi (outer groups >= 1) x inner factor of the digit value, base offset, sub-step-0 'last'
    __shared__ double2 sEI[2][S][2][D][N];
    __shared__ long long sBase[2];
    __shared__ int sLast[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // classes of the pair states (a, b) with a < b (the readout's upper triangle)
    auto upper_class = [](int d) {
        for (int aa = 0; aa < M; ++aa)
            for (int bb = aa + 1; bb < M; ++bb)
                if (class_of(M, LAT, aa, bb) == d + 1) return true;
        return false;
    };
    for (int i = tid; i < 2 * N * N; i += kF2Block) (&sK[0][0][0])[i] = a.small[lay.kp(0) + i];
    for (int i = tid; i < S * 2 * D * N; i += kF2Block) {
        const int s = i / (2 * D * N), kap = (i / (D * N)) % 2, d = (i / N) % D, v = i % N;
        const int other = s == 0 ? 1 : 0;  // sub-step 0: digit 1 (old value); sub-step 1: digit 0 (new value)
        sIn[s][kap][d][v] = a.inner[((((size_t)s * S + other) * 2 + kap) * D + d) * N + v];
    }
    const int CH = (a.T + kF2F - 1) / kF2F;
    const long long n_units = (long long)a.n_tiles * CH;
    const long long per = n_units / gridDim.x, rem = n_units % gridDim.x;
    const long long u_begin = (long long)blockIdx.x * per + min((long long)blockIdx.x, rem);
    const long long u_end = u_begin + per + ((long long)blockIdx.x < rem ? 1 : 0);
    // readout accumulators.  Sub-step 0: per upper-triangle entry (last varies per fibre).  Sub-step 1:
    // last = w is fixed per thread, so K'(nw, w) is applied once at the end and only the plain sum
    // (class 0) and the upper-triangle class moments are accumulated.
    double2 acc0[RO ? NU : 1], accS1 = make_double2(0.0, 0.0), accM1[RO ? D : 1];
#pragma unroll
    for (int n = 0; n < (RO ? NU : 1); ++n) acc0[n] = make_double2(0.0, 0.0);
#pragma unroll
    for (int n = 0; n < (RO ? D : 1); ++n) accM1[n] = make_double2(0.0, 0.0);
    auto tile_base = [&](int tau) {
        long long b = 0;
        for (int g = 1; g < a.G; ++g) b += __ldg(&a.goff[(size_t)g * a.X + (tau / a.gdiv[g]) % a.gmod[g]]);
        return b;
    };
    // cp.async the entries of unit (tau, chunk ch) into stage[buf]: thread (w, lane) copies rows
    // e = w + 9 i of fibre `lane`; tbase = the tile's base offset, lofs_t = lofs[t] of the thread's fibre
    auto issue = [&](int tau, int ch, int buf, long long tbase_u, int lofs_x) {
        const int t0 = ch * kF2F, t = t0 + lane;
        // E0[s][kap][d][fibre t] = Etab[s][kap][group 0][d][t]: rows of kF2F consecutive entries
        for (int i = tid; i < S * 2 * D * kF2F; i += kF2Block) {
            const int f = i % kF2F, row = i / kF2F;  // row = (s * 2 + kap) * D + d
            if (t0 + f < a.T)
                cp_async16(&(&sE0u[buf][0][0][0][0])[i], a.Etab + ((size_t)(row / D) * a.G * D + row % D) * a.X + t0 + f);
        }
        if (t < a.T) {
            const long long base = tbase_u + lofs_x;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int e = warp + N * i, d0 = e % N, d1 = e / N;
                cp_async16(&stage[buf][e][lane], a.A + base + (long long)d0 * a.pw_in[0] + (long long)d1 * a.pw_in[1]);
            }
        }
        cp_async_commit();
    };
    // unit u = tau * CH + ch: (tau, ch) of this unit and of the next advance incrementally; the issuing
    // threads cache the base of the tile they last issued for and the next unit's lofs entry
    int tau = (int)(u_begin / CH), ch = (int)(u_begin % CH);
    int itau = tau;
    long long ibase = tile_base(tau);
    __syncthreads();
    if (u_begin < u_end) issue(tau, ch, 0, ibase, ch * kF2F + lane < a.T ? __ldg(&a.lofs[ch * kF2F + lane]).x : 0);
    int cur_tile = -1, last_t = 0;
    long long tbase = 0;
    // Per unit: barrier A (its copies landed; every warp is done with the previous unit) -> copies of
    // the next unit into the other buffer -> sub-step 0 (stage -> stage) -> barrier B -> sub-step 1
    // (stage -> HBM: each thread stores the fibre it computed).
    for (long long u = u_begin; u < u_end; ++u) {
        const int buf = (int)((u - u_begin) & 1);
        const int t = ch * kF2F + lane, tp = tau & 1;
        const bool valid = t < a.T;
        const int ntau = ch + 1 == CH ? tau + 1 : tau, nch = ch + 1 == CH ? 0 : ch + 1, nt = nch * kF2F + lane;
        const int nlofs = (u + 1 < u_end && nt < a.T) ? __ldg(&a.lofs[nt]).x : 0;  // in flight across the barrier
        if (tau != cur_tile) {  // tile constants into the parity-tau buffer (readers of tau-1 use the other)
            if (tid < S * 2 * D * N) {
                const int s = tid / (2 * D * N), kap = (tid / (D * N)) % 2, d = (tid / N) % D, v = tid % N;
                double2 e = make_double2(1.0, 0.0);
                for (int g = 1; g < a.G; ++g)
                    e = cmul(e, __ldg(&a.Etab[((((size_t)s * 2 + kap) * a.G + g) * D + d) * a.X + (tau / a.gdiv[g]) % a.gmod[g]]));
                sEI[tp][s][kap][d][v] = cmul(cmul(e, a.fixfac[s][kap][d]), sIn[s][kap][d][v]);
            }
            if (tid == kF2Block - 1) {
                sBase[tp] = tile_base(tau);
                sLast[tp] = a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (tau / a.last_div) % N : 0);
            }
        }
        const int2 lo = valid ? __ldg(&a.lofs[t]) : make_int2(0, 0);  // in flight across the barrier
        cp_async_wait<0>();  // this unit's copies (every thread's) have landed ...
        __syncthreads();     // A: ... and are visible, tile constants too; buf ^ 1 is free
        if (u + 1 < u_end) {
            if (ntau != itau) itau = ntau, ibase = tile_base(ntau);  // once per tile
            issue(ntau, nch, buf ^ 1, ibase, nlofs);
        }
        if (tau != cur_tile) cur_tile = tau, tbase = sBase[tp], last_t = sLast[tp];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (valid) {
                const int w = warp;  // s = 0: d1 = w, fibre along d0;  s = 1: d0 = w, fibre along d1
                auto slot = [&](int v) -> double2 & { return stage[buf][s == 0 ? v + N * w : w + N * v][lane]; };
                const int last = s == 0 ? (lo.y >= 0 ? lo.y : last_t) : w;
                // the plain sum and every class moment in one pass over the fibre's old values (one entry
                // live at a time: the register budget of 2 CTAs per SM holds no 9-entry fibre next to the
                // readout accumulators); D + NUC independent chains
                double2 S0 = make_double2(0.0, 0.0), mp[D], mr[RO ? D : 1];
#pragma unroll
                for (int d = 0; d < D; ++d) mp[d] = make_double2(0.0, 0.0);
#pragma unroll
                for (int d = 0; d < (RO ? D : 1); ++d) mr[d] = make_double2(0.0, 0.0);
#pragma unroll
                for (int v = 0; v < N; ++v) {
                    const double2 x = slot(v);
                    S0 = cadd(S0, x);
#pragma unroll
                    for (int d = 0; d < D; ++d) mp[d] = cfma(bt.b[s][0][d][v], x, mp[d]);
                    if constexpr (RO)
#pragma unroll
                        for (int d = 0; d < D; ++d)
                            if (upper_class(d)) mr[d] = cfma(bt.b[s][1][d][v], x, mr[d]);
                }
                // class moment of class d, weights kap (0: propagation, 1: readout), times its class
                // factor E0 (outer group 0, this fibre) x EI (tile groups x inner digit w)
                auto moment = [&](int kap, int d) {
                    const double2 mm = kap == 0 ? mp[d] : mr[RO ? d : 0];
                    return cmul(cmul(sE0u[buf][s][kap][d][lane], sEI[tp][s][kap][d][w]), mm);
                };
                // readout first (upper triangle only: rho_ba = conj rho_ab), one class moment live at a time
                if constexpr (RO) {
                    if (s == 0) {
                        int u = 0;
#pragma unroll
                        for (int aa = 0; aa < M; ++aa)
#pragma unroll
                            for (int bb = aa; bb < M; ++bb, ++u)
                                if (aa == bb) acc0[RO ? u : 0] = cfma(sK[0][aa * M + bb][last], S0, acc0[RO ? u : 0]);
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
                                            acc0[RO ? u : 0] = cfma(sK[1][aa * M + bb][last], m1, acc0[RO ? u : 0]);
                            }
                    } else {
                        accS1 = cadd(accS1, S0);
#pragma unroll
                        for (int d = 0; d < D; ++d)
                            if (upper_class(d)) accM1[RO ? d : 0] = cadd(accM1[RO ? d : 0], moment(1, d));
                    }
                }
                // propagate: the outputs of each class go straight out: sub-step 0 back into the fibre's
                // stage slots (all read above), sub-step 1 to HBM (entry d0 = w, d1 = nw of this fibre)
                double2 *out = a.A + tbase + lo.x + (long long)w * a.pw_in[0];
                auto put = [&](int nw, double2 v) {
                    if (s == 0) slot(nw) = v;
                    else __stcs(out + (long long)nw * a.pw_in[1], v);
                };
#pragma unroll
                for (int nw = 0; nw < N; ++nw)
                    if (class_of(M, LAT, nw / M, nw % M) == 0) put(nw, cmul(sK[0][nw][last], S0));
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    const double2 m = moment(0, d);
#pragma unroll
                    for (int nw = 0; nw < N; ++nw)
                        if (class_of(M, LAT, nw / M, nw % M) == d + 1) put(nw, cmul(sK[0][nw][last], m));
                }
            }
            if (s == 0) __syncthreads();  // B
        }
        tau = ntau, ch = nch;
    }
    cp_async_wait<0>();
    if constexpr (RO) {
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
                        const double2 v = s == 0 ? acc0[u]
                                                 : (c == 0 ? cmul(sK[0][nw][warp], accS1) : cmul(sK[1][nw][warp], accM1[c - 1]));
                        full[nw] = v;
                        full[bb * M + aa] = make_double2(v.x, -v.y);
                    }
                reduce_finalize<N, kF2Block>(full, a.partials + (size_t)s * kPartialsMax * N, a.rho[s], a.counter + s,
                                             a.rho_accumulate != 0);
            }
    }
}

namespace {
template <bool LAT>
constexpr size_t fused2s_dyn() { return (size_t)2 * (kF2N * kF2N + 2 * 2 * n_classes(3, LAT)) * kF2F * 16; }
template <bool LAT, bool RO>
cudaError_t fused2s_t(const FusedArgs &a, const Beta2s &b, int grid, cudaStream_t s) {
    cudaFuncSetAttribute(k_fused2s<LAT, RO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused2s_dyn<LAT>());
    k_fused2s<LAT, RO><<<grid, kF2Block, fused2s_dyn<LAT>(), s>>>(a, b);
    return cudaGetLastError();
}
template <bool LAT, bool RO>
int fused2s_occ_t() {
    int o = 0;
    cudaFuncSetAttribute(k_fused2s<LAT, RO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fused2s_dyn<LAT>());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_fused2s<LAT, RO>, kF2Block, fused2s_dyn<LAT>());
    return o;
}
}  // namespace

int fused2s_block() { return kF2Block; }
cudaError_t launch_fused2s(bool lattice, const FusedArgs &a, const Beta2s &b, bool ro, int grid, cudaStream_t s) {
    if (lattice) return ro ? fused2s_t<true, true>(a, b, grid, s) : fused2s_t<true, false>(a, b, grid, s);
    return ro ? fused2s_t<false, true>(a, b, grid, s) : fused2s_t<false, false>(a, b, grid, s);
}
int fused2s_occupancy(bool lattice) {
    const int a = lattice ? fused2s_occ_t<true, true>() : fused2s_occ_t<false, true>();
    const int b = lattice ? fused2s_occ_t<true, false>() : fused2s_occ_t<false, false>();
    return a < b ? a : b;
}

}  // namespace qp
