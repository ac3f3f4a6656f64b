// persist.cu -- k_small: the slide steps of a SMALL ARDM (<= QP_PERSIST_MAX_BYTES) in ONE launch per
// qp_steps call, the ARDM and every factor table resident in one CTA's shared memory.  The per-step arithmetic is that of k_fused_r at S = 1 (slide_r.cu: P:87-94 the
// Makri-Makarov propagation, P:384-390 the BSXFUN lines, P:415-418 the fused rho readout):
//   out[new] = K'(new, last) * F_d(fibre) * sum_old beta_d(old) a[old]      (Ds(new) = delta_d != 0)
//   out[new] = K'(new, last) * sum_old a[old]                                (Ds(new) = 0)
// with F_d the product of the outer digit-group factor tables (Etab) of the fibre's tile and
// tile-local index, and the readout rho(t_k)[n] = sum over fibres of the same with the readout
// weights (kappa = 1; the Ds = 0 rows read the propagated value).
//
// For such an ARDM a per-step launch (plus the per-tile table building of the fused kernels) costs
// far more than the step itself.  k_small copies the workspace tables and the ARDM into shared
// memory once, re-points the launch-set arguments at the copies and runs the steps one at a time:
// thread i takes fibres i, i + 256, ... of the step (one round of table lookups, N loads, the
// moments and N stores), CTA barriers between steps, the readout reduced straight into rho; the
// ARDM goes back to HBM at the end.  (A cooperative multi-CTA variant for L2-resident ARDMs of
// 1-64 MB measured slower than the per-group launches of the fused kernels -- DESIGN.md §5.)
#include "common.cuh"

namespace qp {

namespace {

template <bool SMEM, typename T> __device__ __forceinline__ T ld_(const T *p) {
    if constexpr (SMEM) return *p;
    else return __ldg(p);
}
template <bool SMEM> __device__ __forceinline__ double2 ld_a(const double2 *p) {
    if constexpr (SMEM) return *p;
    else return __ldcg(p);
}
template <bool SMEM> __device__ __forceinline__ void st_a(double2 *p, double2 v) {
    if constexpr (SMEM) *p = v;
    else __stcg(p, v);
}

// Per-step constants in shared memory: K'_kappa(new, last) and beta_d(old) of the step's variant.
template <int M, bool LAT>
struct StepTables {
    static constexpr int N = M * M, D = n_classes(M, LAT);
    double2 K[2][N][N];
    double2 beta[2][D][N];
};

// One slide step (S = 1) over the fibres f = gtid, gtid + nthr, ... of launch set `a`; returns the
// thread's readout contributions in acc (zero when ro is false).
template <int M, bool LAT, bool SYM, bool SMEM>
__device__ __forceinline__ void lean_step(const FusedArgs &a, const StepTables<M, LAT> &tb, const double (&sym)[2][4],
                                          bool ro, long long gtid, long long nthr, double2 (&acc)[M * M]) {
    constexpr int N = M * M, D = n_classes(M, LAT), NK = 2;
    const unsigned nf = (unsigned)a.n_tiles * (unsigned)a.T, T = (unsigned)a.T;  // < 2^31 (small ARDM)
    const long long pw = a.pw_in[0];
    for (unsigned f = (unsigned)gtid; f < nf; f += (unsigned)nthr) {
        const int tau = (int)(f / T), t = (int)(f - (unsigned)tau * T);
        const int2 lo = ld_<SMEM>(&a.lofs[t]);
        long long base = lo.x;
        double2 F[NK][D];
#pragma unroll
        for (int kap = 0; kap < NK; ++kap)
#pragma unroll
            for (int d = 0; d < D; ++d)
                F[kap][d] = (kap == 0 || ro) ? cmul(ld_<SMEM>(&a.Etab[((size_t)kap * a.G * D + d) * a.X + t]), a.fixfac[0][kap][d])
                                             : make_double2(0.0, 0.0);
        for (int g = 1; g < a.G; ++g) {
            const int idx = (int)(((unsigned)tau / (unsigned)a.gdiv[g]) % (unsigned)a.gmod[g]);
            base += ld_<SMEM>(&a.goff[(size_t)g * a.X + idx]);
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d)
                    if (kap == 0 || ro) F[kap][d] = cmul(F[kap][d], ld_<SMEM>(&a.Etab[(((size_t)kap * a.G + g) * D + d) * a.X + idx]));
        }
        const int last = lo.y >= 0 ? lo.y
                                   : (a.fixed_last >= 0 ? a.fixed_last : (a.last_div > 0 ? (int)(((unsigned)tau / (unsigned)a.last_div) % N) : 0));
        double2 x[N];
#pragma unroll
        for (int v = 0; v < N; ++v) x[v] = ld_a<SMEM>(a.A + base + v * pw);
        double2 S0, m[NK][D];
        if constexpr (SYM) {  // M = 2, s = (+s, -s): the four-sum moments (slide_r.cu)
            const double2 u = cadd(x[0], x[3]), w = csub(x[0], x[3]);
            const double2 p = cadd(x[1], x[2]), q = csub(x[1], x[2]);
            S0 = cadd(u, p);
#pragma unroll
            for (int kap = 0; kap < NK; ++kap) {
                const double cr = sym[kap][0], ci = sym[kap][1], ch = sym[kap][2], sh = sym[kap][3];
                const double2 A = make_double2(fma(cr, u.x, ch * p.x), fma(cr, u.y, ch * p.y));
                const double2 Bv = make_double2(fma(-ci, w.y, sh * q.x), fma(ci, w.x, sh * q.y));
                m[kap][0] = cadd(A, Bv);
                m[kap][D - 1] = csub(A, Bv);
            }
        } else {
            S0 = x[0];
#pragma unroll
            for (int v = 1; v < N; ++v) S0 = cadd(S0, x[v]);
#pragma unroll
            for (int kap = 0; kap < NK; ++kap)
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double2 mm = cmul(tb.beta[kap][d][0], x[0]);
#pragma unroll
                    for (int v = 1; v < N; ++v) mm = cfma(tb.beta[kap][d][v], x[v], mm);
                    m[kap][d] = mm;
                }
        }
#pragma unroll
        for (int nw = 0; nw < N; ++nw) {
            const int c = class_of(M, LAT, nw / M, nw % M);
            const double2 o = cmul(tb.K[0][nw][last], c == 0 ? S0 : cmul(F[0][c > 0 ? c - 1 : 0], m[0][c > 0 ? c - 1 : 0]));
            if (ro)
                acc[nw] = cadd(acc[nw], c == 0 ? o : cmul(tb.K[1][nw][last], cmul(F[1][c > 0 ? c - 1 : 0], m[1][c > 0 ? c - 1 : 0])));
            st_a<SMEM>(a.A + base + nw * pw, o);
        }
    }
}

template <int M, bool LAT>
__device__ __forceinline__ void load_tables(StepTables<M, LAT> &tb, const double2 *small, int var, bool with_k) {
    constexpr int N = M * M, D = n_classes(M, LAT);
    const SmallLayout lay{N, D, 0};
    if (with_k)
        for (int i = threadIdx.x; i < 2 * N * N; i += kPersistBlock) (&tb.K[0][0][0])[i] = small[lay.kp(0) + i];
    for (int i = threadIdx.x; i < 2 * D * N; i += kPersistBlock) {
        const int kap = i / (D * N), r = i % (D * N);
        (&tb.beta[0][0][0])[i] = small[lay.beta(var, kap) + r];
    }
}

}  // namespace

template <int M, bool LAT, bool SYM>
__global__ void __launch_bounds__(kPersistBlock, 1) k_small(const __grid_constant__ PersistArgs pa) {
    constexpr int N = M * M;
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ StepTables<M, LAT> tb;
    unsigned char *tab = dsm;
    double2 *sA = reinterpret_cast<double2 *>(tab + pa.tables_bytes);
    FusedArgs *sets = reinterpret_cast<FusedArgs *>(reinterpret_cast<unsigned char *>(sA) + pa.ardm_entries * 16);
    {
        const int4 *src = reinterpret_cast<const int4 *>(pa.wbase);
        int4 *dst = reinterpret_cast<int4 *>(tab);
        for (long long i = threadIdx.x; i < pa.tables_bytes / 16; i += kPersistBlock) dst[i] = src[i];
        const int4 *srcA = reinterpret_cast<const int4 *>(pa.A);
        int4 *dstA = reinterpret_cast<int4 *>(sA);
        for (long long i = threadIdx.x; i < pa.ardm_entries; i += kPersistBlock) dstA[i] = srcA[i];
        const int4 *srcS = reinterpret_cast<const int4 *>(pa.sets);
        int4 *dstS = reinterpret_cast<int4 *>(sets);
        for (long long i = threadIdx.x; i < (long long)pa.nsets * (long long)(sizeof(FusedArgs) / 16); i += kPersistBlock)
            dstS[i] = srcS[i];
    }
    __syncthreads();
    auto rebase = [&](const void *p) -> unsigned char * {
        return tab + (reinterpret_cast<const unsigned char *>(p) - reinterpret_cast<const unsigned char *>(pa.wbase));
    };
    for (int i = threadIdx.x; i < pa.nsets; i += kPersistBlock) {
        FusedArgs &f = sets[i];
        f.A = sA;
        f.Etab = reinterpret_cast<const double2 *>(rebase(f.Etab));
        f.goff = reinterpret_cast<const long long *>(rebase(f.goff));
        f.lofs = reinterpret_cast<const int2 *>(rebase(f.lofs));
    }
    const double2 *small = reinterpret_cast<const double2 *>(rebase(pa.small));
    int var_loaded = -1;
    for (long long k = pa.k_begin; k < pa.k_end; ++k) {
        const int var = (k == pa.L) ? 1 : 0;
        if (var != var_loaded) {
            __syncthreads();
            load_tables<M, LAT>(tb, small, var, var_loaded < 0);
            var_loaded = var;
        }
        __syncthreads();  // the previous step's stores (and the tables) are visible
        const FusedArgs &a = sets[(size_t)(k % pa.L) * pa.set_stride];
        const int slot = pa.slot[k];
        double2 acc[N];
#pragma unroll
        for (int n = 0; n < N; ++n) acc[n] = make_double2(0.0, 0.0);
        lean_step<M, LAT, SYM, true>(a, tb, pa.sym[var], slot >= 0, threadIdx.x, kPersistBlock, acc);
        if (slot >= 0) reduce_block_to<N, kPersistBlock>(acc, pa.rho_base + (size_t)slot * N);
    }
    __syncthreads();
    {
        const int4 *srcA = reinterpret_cast<const int4 *>(sA);
        int4 *dstA = reinterpret_cast<int4 *>(pa.A);
        for (long long i = threadIdx.x; i < pa.ardm_entries; i += kPersistBlock) dstA[i] = srcA[i];
    }
}

namespace {
template <int M, bool LAT, bool SYM>
cudaError_t small_t(const PersistArgs &pa, size_t dyn, cudaStream_t s) {
    cudaFuncSetAttribute(k_small<M, LAT, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    k_small<M, LAT, SYM><<<1, kPersistBlock, dyn, s>>>(pa);
    return cudaGetLastError();
}
template <int M, bool LAT, bool SYM>
int small_static_t() {
    cudaFuncAttributes at{};
    if (cudaFuncGetAttributes(&at, k_small<M, LAT, SYM>) != cudaSuccess) return 1 << 30;
    return (int)at.sharedSizeBytes;
}
}  // namespace

#define QP_PERSIST_DISPATCH(FN, ...)                                                        \
    switch (M) {                                                                            \
    case 2: return sym ? FN<2, false, true>(__VA_ARGS__) : FN<2, false, false>(__VA_ARGS__); \
    case 3: return lattice ? FN<3, true, false>(__VA_ARGS__) : FN<3, false, false>(__VA_ARGS__); \
    case 4: return lattice ? FN<4, true, false>(__VA_ARGS__) : FN<4, false, false>(__VA_ARGS__); \
    }

cudaError_t launch_small(int M, bool lattice, bool sym, const PersistArgs &pa, size_t dyn, cudaStream_t s) {
    QP_PERSIST_DISPATCH(small_t, pa, dyn, s)
    return cudaErrorInvalidValue;
}
int small_static_smem(int M, bool lattice, bool sym) {
    QP_PERSIST_DISPATCH(small_static_t)
    return 1 << 30;
}

}  // namespace qp
