// trsv.cu -- forward / backward substitution with the ILU factors (M^{-1} = U^{-1} L^{-1}).
//
// Applying the incomplete-LU preconditioner of sec. II inside the
// left-preconditioned GMRES of Eq. (8) is one forward substitution
// with the unit lower factor and one backward substitution with the upper factor per
// Arnoldi step.
//
// Why not plain level scheduling: the ILUT factors of an RCM-ordered Liouvillian fill
// the RCM band, and their dependency DAG is nearly a chain -- the row-level schedule of
// BASELINE configs[1] has 11,853 (L) and 17,714 (U) levels for n = 32,400 rows (DESIGN.md
// sec. 5).  Any row-level substitution pays one synchronisation per level.
//
// v2 (this file): block-level scheduling.  Rows are cut into blocks of B consecutive
// rows (the RCM band makes consecutive rows the dependency chain).  In the kernel's
// index space (the U factor is reversed at setup, i' = n-1-i, so both factors are
// lower triangular here):
//     x_k = D_k^{-1} ( b_k - sum_{j<k} T_kj x_j ),
// D_k the B x B diagonal block (its explicit inverse precomputed at setup, packed
// lower, column-major), T_kj the strictly-earlier part of the rows of block k.  The
// dependency chain shrinks from ~n/3 row levels to n/B block steps.  Per block:
//   * "far" entries (source blocks <= k-3) are streamed in fixed 32-entry chunks by
//     the warp that owns the row, each chunk issued as soon as every source block it
//     reads is finished (frontier of completion flags) -- this is the bulk of the
//     bytes and runs ahead of the chain on every SM, finishing a step early;
//   * "near" entries (source blocks k-2, k-1) form one flat list per block whose
//     column/value loads are issued before the wait; once block k-1 is published all
//     NT threads gather x for them at once and one thread per row sums its products
//     in order -- the only sparse work on the chain;
//   * the inverse block, staged in shared memory by a TMA bulk copy
//     (cp.async.bulk + mbarrier) issued when the CTA takes the block, is applied as a
//     dense triangular mat-vec by all NT threads;
//   * x_k is stored, then a gpu-scope release store of the block's completion flag
//     (value = launch epoch, so flags never need resetting) publishes it.
// One persistent CTA per SM (cooperative launch guarantees co-residency, so the spin
// waits cannot deadlock); CTA c takes blocks c, c+G, c+2G, ...  Each CTA keeps one
// completion frontier in shared memory; at most one of its warps polls the L2 flags
// at a time (a shared-memory lock), so ~148 pollers, not ~2,400 warps, share the hot
// flag lines.  Every reduction has a fixed order: the result is deterministic for a
// given B.
#include "problem.h"

namespace ssb {

namespace {

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double2 ld_cg2(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ double2 ld_relaxed2(const double2* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed2(double2* p, double2 v) {
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
// Sentinel the output is filled with before a substitution: a signalling-NaN payload
// that arithmetic never produces (it only yields quiet NaNs).
constexpr unsigned long long kSentinelBits = 0x7FF4DEADBEEF0BADull;
__device__ __forceinline__ bool is_sentinel(double2 v) {
    return __double_as_longlong(v.x) == (long long)kSentinelBits ||
           __double_as_longlong(v.y) == (long long)kSentinelBits;
}
__global__ void k_fill_sentinel(double2* x, int64_t n) {
    const double s = __longlong_as_double((long long)kSentinelBits);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = make_double2(s, s);
}
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }

// ---- mbarrier + TMA bulk copy (global -> shared), PTX ISA 8.0+, sm_90+
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ int ld_acq_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// Warp-collective: return once every block < target is published.  The CTA's frontier
// sF (all blocks < *sF are published) lives in shared memory; the warp holding sLock
// examines 32 L2 flags per round trip and advances it.
__device__ __forceinline__ void wait_frontier(int target, int* sF, int* sLock, const uint32_t* flags, int nblk,
                                              uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    int f = ld_acq_cta(sF);
    while (f < target) {
        int got = 0;
        if (lane == 0) got = atomicCAS(sLock, 0, 1) == 0;
        got = __shfl_sync(0xffffffffu, got, 0);
        if (got) {
            f = ld_acq_cta(sF);
            if (f < target) {
                const int s = f + lane;
                const bool ok = (s >= nblk) || ld_acquire(flags + s) == epoch;
                const unsigned m = __ballot_sync(0xffffffffu, ok);
                const int adv = (m == 0xffffffffu) ? 32 : (__ffs(~m) - 1);
                __syncwarp();
                if (lane == 0 && adv) st_rel_cta(sF, f + adv);
            }
            __syncwarp();
            if (lane == 0) st_rel_cta(sLock, 0);
        } else {
            __nanosleep(40);
        }
        f = ld_acq_cta(sF);
    }
    __syncwarp();   // every lane's acquire precedes every lane's later loads
}

constexpr int kGrp = 4;
constexpr int kTrace = 8;   // timestamps per block when tracing

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}   // far-phase rows in flight per warp

template <int B, int NT>
struct Cfg {
    static constexpr int kWarps = NT / 32;
    static constexpr int kRPW = B / kWarps;           // rows per warp in the far phase
    static constexpr int kParts = 2 * NT / B;         // threads per row pair in the mat-vec
    static constexpr int kPacked = B * (B + 1) / 2;   // packed lower-triangular inverse
    static constexpr int kPre = 8;                    // near entries prefetched per thread
    static constexpr int kNearCap = kPre * NT;        // near products staged per pass
    static constexpr size_t kSmem = (size_t)kPacked * 16 + (size_t)(2 + kParts) * B * 16 + (size_t)kNearCap * 16 + (size_t)2 * B * 16 +
                                   (size_t)B * 12 + 32;
    static_assert(NT % B == 0 && B % kWarps == 0 && B % 32 == 0, "layout");
};

template <int B, int NT>
__global__ void __launch_bounds__(NT, 1)
k_block_trsv(const TriArgs a, const double2* __restrict__ bvec, double2* x, uint32_t epoch,
             unsigned long long* __restrict__ trace) {
    using C = Cfg<B, NT>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* sInv = reinterpret_cast<double2*>(smem_raw);
    double2* sFar = sInv + C::kPacked;
    double2* sR = sFar + B;
    double2* sPart = sR + B;
    double2* sProd = sPart + C::kParts * B;
    double2* sX = sProd + C::kNearCap;   // x of source blocks k-2, k-1
    int64_t* sRowP = reinterpret_cast<int64_t*>(sX + 2 * B);
    int32_t* sRowL = reinterpret_cast<int32_t*>(sRowP + B);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sRowL + B);
    int* sF = reinterpret_cast<int*>(bar + 1);
    int* sLock = sF + 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int nblk = (int)a.nblk;
    const bool rev = a.rev != 0;
    auto phys = [&](int64_t i) -> int64_t { return rev ? n - 1 - i : i; };

    if (tid == 0) {
        mbar_init(bar, 1);
        *sF = 0;
        *sLock = 0;
    }
    __syncthreads();
    uint32_t phase = 0;

    for (int k = blockIdx.x; k < nblk; k += gridDim.x) {
        const int64_t row0 = (int64_t)k * B;
        const int64_t rowe = min(row0 + B, n);
        // 0. stage D_k^{-1} in shared memory (TMA bulk copy, completes on `bar`)
        if (tid == 0) {
            if (trace) trace[(int64_t)k * kTrace + 0] = gtime();
            mbar_expect_tx(bar, (uint32_t)(C::kPacked * 16));
            bulk_g2s(sInv, a.dinv + (int64_t)k * C::kPacked, (uint32_t)(C::kPacked * 16), bar);
        }

        // 1. far phase (sources <= k-3): warp w owns rows row0 + w*RPW .. +RPW; chunk c of
        //    every owned row before chunk c+1 of any (oldest sources first)
        {
            double2 acc[C::kRPW];
            int64_t* wp = sRowP + warp * C::kRPW;
            int32_t* wl = sRowL + warp * C::kRPW;
            if (lane < C::kRPW) {
                const int64_t i = row0 + warp * C::kRPW + lane;
                int64_t p0 = 0, l0 = 0;
                if (i < n) {
                    p0 = a.farptr[i];
                    l0 = a.farptr[i + 1] - p0;
                }
                wp[lane] = p0;
                wl[lane] = (int32_t)l0;
            }
            __syncwarp();
            int nch = 0;
#pragma unroll
            for (int r = 0; r < C::kRPW; r++) {
                acc[r] = make_double2(0.0, 0.0);
                nch = max(nch, (wl[r] + 31) >> 5);
            }
#pragma unroll 1
            for (int c = 0; c < nch; c++) {
                // issue the column/value loads of chunk c of every owned row, then wait
                // once, then gather x kGrp rows at a time
                const int32_t t = c * 32 + lane;
                int32_t cc[C::kRPW];
                double2 vv[C::kRPW];
                int32_t need = -1;
#pragma unroll
                for (int r = 0; r < C::kRPW; r++) {
                    cc[r] = -1;
                    if (t < wl[r]) {
                        cc[r] = ld_stream(a.fcol + wp[r] + t);
                        vv[r] = ld_stream2(a.fval + wp[r] + t);
                        need = max(need, cc[r]);
                    }
                }
                need = __reduce_max_sync(0xffffffffu, need);
                if (need >= 0) wait_frontier(need / B + 1, sF, sLock, a.flags, nblk, epoch);
#pragma unroll
                for (int g = 0; g < C::kRPW; g += kGrp) {
                    double2 xv[kGrp];
#pragma unroll
                    for (int r = 0; r < kGrp; r++)
                        if (cc[g + r] >= 0) xv[r] = ld_cg2(x + phys(cc[g + r]));
#pragma unroll
                    for (int r = 0; r < kGrp; r++)
                        if (cc[g + r] >= 0) acc[g + r] = cfma(acc[g + r], vv[g + r], xv[r]);
                }
            }
#pragma unroll
            for (int r = 0; r < C::kRPW; r++) {
                const double2 s = warp_sum2(acc[r]);
                const int64_t i = row0 + warp * C::kRPW + r;
                if (lane == 0) sFar[warp * C::kRPW + r] = (i < n) ? csub(__ldg(bvec + phys(i)), s) : make_double2(0.0, 0.0);
            }
        }


        // 2. near phase (sources k-2, k-1): the 2B x values are staged in shared memory by
        //    one coalesced load per value -- polled until it no longer holds the sentinel
        //    (each 8-byte half is single-copy atomic; both are checked), which is how the
        //    chain hands x_{k-1} over without a flag round trip -- then every near entry
        //    (flat list of the block) is multiplied out of shared memory, and one thread
        //    per row sums its products in order.
        double2 rr = make_double2(0.0, 0.0);
        {
            const int64_t nb = a.nrp[row0], ne = a.nrp[rowe];
            const int64_t xlo = row0 - 2 * B;   // first column of source block k-2
            int64_t q0 = 0, q1 = 0;
            if (tid < B && row0 + tid < n) {
                q0 = a.nrp[row0 + tid];
                q1 = a.nrp[row0 + tid + 1];
            }
            bool first = true;
            for (int64_t pb = nb; pb < ne || first; pb += C::kNearCap) {
                const int64_t pe = min(ne, pb + C::kNearCap);
                int32_t cc[C::kPre];
                double2 vv[C::kPre];
#pragma unroll
                for (int t = 0; t < C::kPre; t++) {
                    const int64_t e = pb + tid + (int64_t)t * NT;
                    cc[t] = -1;
                    if (e < pe) {
                        cc[t] = ld_stream(a.ncol + e);
                        vv[t] = ld_stream2(a.nval + e);
                    }
                }
                if (first) {
                    __syncthreads();   // sFar complete
                    if (trace && tid == 0) trace[(int64_t)k * kTrace + 2] = gtime();
                    if (tid < B) rr = sFar[tid];
                    for (int t = tid; t < 2 * B; t += NT) {
                        const int64_t j = xlo + t;
                        double2 v = make_double2(0.0, 0.0);
                        if (j >= 0) {
                            v = ld_relaxed2(x + phys(j));
                            while (is_sentinel(v)) v = ld_relaxed2(x + phys(j));
                        }
                        sX[t] = v;
                    }
                    if (trace && tid == 2 * B - 1) trace[(int64_t)k * kTrace + 1] = gtime();
                    __syncthreads();
                    first = false;
                }
#pragma unroll
                for (int t = 0; t < C::kPre; t++)
                    if (cc[t] >= 0) sProd[tid + t * NT] = cmul(vv[t], sX[cc[t] - xlo]);
                __syncthreads();
                if (tid < B)
                    for (int64_t e = max(q0, pb); e < min(q1, pe); e++) rr = csub(rr, sProd[e - pb]);
                __syncthreads();
                if (pe >= ne) break;
            }
            if (tid < B) sR[tid] = rr;
            if (trace && tid == 0) trace[(int64_t)k * kTrace + 3] = gtime();
        }
        __syncthreads();

        // 3. x_k = D_k^{-1} r with the packed column-major lower inverse.  Rows are paired
        //    (p, B-1-p: B+1 entries per pair, so every thread does the same work); the TP
        //    threads of a pair split the columns j = s, s+TP, ...; a warp's lanes share s
        //    and take consecutive p, so their shared-memory reads are contiguous.
        mbar_wait(bar, phase);
        phase ^= 1u;
        if (trace && tid == 0) trace[(int64_t)k * kTrace + 6] = gtime();
        {
            constexpr int kPairs = B / 2, TP = NT / kPairs;
            const int pr = tid % kPairs, sub = tid / kPairs;
            const int i1 = pr, i2 = B - 1 - pr;
            double2 s1 = make_double2(0.0, 0.0), s2 = make_double2(0.0, 0.0);
            double2 t1 = make_double2(0.0, 0.0), t2 = make_double2(0.0, 0.0);
            int j = sub;
            for (; j + TP <= i1; j += 2 * TP) {   // both rows, two columns per trip
                const int ja = j, jb = j + TP;
                const int ca = ja * B - (ja * (ja - 1)) / 2, cb = jb * B - (jb * (jb - 1)) / 2;
                const double2 ra = sR[ja], rb = sR[jb];
                const double2 a2 = sInv[ca + (i2 - ja)], b2 = sInv[cb + (i2 - jb)];
                const double2 a1 = sInv[ca + (i1 - ja)], b1 = sInv[cb + (i1 - jb)];
                s2 = cfma(s2, a2, ra);
                t2 = cfma(t2, b2, rb);
                s1 = cfma(s1, a1, ra);
                t1 = cfma(t1, b1, rb);
            }
            for (; j <= i2; j += TP) {
                const int cs = j * B - (j * (j - 1)) / 2;
                const double2 rj = sR[j];
                s2 = cfma(s2, sInv[cs + (i2 - j)], rj);
                if (j <= i1) s1 = cfma(s1, sInv[cs + (i1 - j)], rj);
            }
            sPart[sub * B + i1] = cadd(s1, t1);
            sPart[sub * B + i2] = cadd(s2, t2);
        }
        __syncthreads();
        if (trace && tid == 0) trace[(int64_t)k * kTrace + 7] = gtime();
        if (tid < B) {
            constexpr int TP = NT / (B / 2);
            const int64_t i = row0 + tid;
            double2 s = sPart[tid];
#pragma unroll
            for (int q = 1; q < TP; q++) s = cadd(s, sPart[q * B + tid]);
            if (i < n) st_relaxed2(x + phys(i), s);
        }
        __syncthreads();
        if (trace && tid == 0) trace[(int64_t)k * kTrace + 4] = gtime();
        if (tid == 0) st_release(a.flags + k, epoch);
        if (trace && tid == 0) trace[(int64_t)k * kTrace + 5] = gtime();
    }
}

template <int B, int NT>
void prepare(DevBlockTri& T) {
    using C = Cfg<B, NT>;
    auto fn = k_block_trsv<B, NT>;
    SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem));
    int dev = 0, sms = 0, per = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, NT, C::kSmem));
    SSB_CHECK(per >= 1, SS_ERR_CUDA, "block trsv kernel does not fit on an SM");
    T.grid = (int)std::max<int64_t>(1, std::min<int64_t>(T.nblk, (int64_t)sms * per));
}

template <int B, int NT>
void launch(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    using C = Cfg<B, NT>;
    auto fn = k_block_trsv<B, NT>;
    if (T.grid == 0) prepare<B, NT>(T);
    k_fill_sentinel<<<grid_for(T.n, 256, kNumSMs * 8), 256, 0, s>>>(x, T.n);
    SSB_LAUNCHED();
    T.epoch++;
    TriArgs a = T.args();
    uint32_t ep = T.epoch;
    void* args[] = {(void*)&a, (void*)&b, (void*)&x, (void*)&ep, (void*)&trace};
    SSB_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(T.grid), dim3(NT), args, C::kSmem, s));
    SSB_LAUNCHED();
}

}  // namespace

size_t block_trsv_packed(int B) { return (size_t)B * (B + 1) / 2; }

void block_trsv_prepare(DevBlockTri& T) {
    switch (T.B * 10000 + T.nt) {
        case 640256: prepare<64, 256>(T); break;
        case 1280256: prepare<128, 256>(T); break;
        case 1280512: prepare<128, 512>(T); break;
        default: SSB_CHECK(false, SS_ERR_ARG, "block substitution supports (B, NT) = (64, 256), (128, 256), (128, 512)");
    }
}

void block_trsv(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    if (T.n == 0) return;
    switch (T.B * 10000 + T.nt) {
        case 640256: launch<64, 256>(T, b, x, s, trace); break;
        case 1280256: launch<128, 256>(T, b, x, s, trace); break;
        case 1280512: launch<128, 512>(T, b, x, s, trace); break;
        default: SSB_CHECK(false, SS_ERR_ARG, "block substitution supports (B, NT) = (64, 256), (128, 256), (128, 512)");
    }
}

}  // namespace ssb
