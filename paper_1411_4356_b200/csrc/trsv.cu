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
// sec. 5).  Any row-level substitution pays one synchronisation per level; v1 (one CTA,
// one barrier per level) ran at 2.6 us per level.
//
// v4 (this file): block substitution with one chain SM and the other SMs as helpers.
// Rows are cut into blocks of B consecutive rows; in the kernel's index space (U
// reversed at setup, i' = n-1-i, so both factors are lower triangular)
//     x_k = D_k^{-1} ( b_k - sum_{j<k} T_kj x_j ),
// with the explicit inverse of every B x B diagonal block D_k precomputed at setup.
// The row entries left of block k are split at setup into
//   * "far"  (source blocks <= k-Q): the bulk of the factor bytes.  Helper CTAs stream
//     them in fixed 32-entry chunks as soon as the chain's completion frontier covers
//     the chunk's sources, and publish r_k = b_k - (far part) with a release flag;
//   * "near" (source blocks k-Q+1 .. k-1): a short list per block.
// The chain CTA walks the blocks in order.  Its producer warp waits for r_k's flag and
// stages D_k^{-1}, the near list and r_k in shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier, two stages), its 8 compute warps subtract the near part
// using the x of the last Q-1 blocks, which never leave the SM (shared-memory ring),
// apply D_k^{-1} (dense triangular mat-vec, trimv.cuh) and append x_k to the ring and
// to global memory, and its publisher warp advances a global frontier word
// (epoch << 32 | blocks done) with a gpu-scope release for the helpers.  For the U
// factor of ILUTP (A Pi = L U) the chain also scatters x through the column
// permutation into the output (x = Pi y).  The
// dependency chain therefore never crosses SMs: the only per-step work on it is the
// near products and the mat-vec, all out of shared memory, while the helpers run Q
// blocks ahead.  One persistent CTA per SM (cooperative launch: all CTAs co-resident,
// so the spin waits cannot deadlock).  Every reduction has a fixed order: the result
// is deterministic for given (B, Q).
#include "problem.h"
#include "trimv.cuh"

namespace ssb {

namespace {

// ------------------------------------------------------------------ memory-model helpers
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int ld_acq_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ double2 ld_cg2(const double2* p) { return __ldcg(p); }
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ void bar_compute(int nthreads) {   // named barrier 1 over the compute warps
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ mbarrier + TMA bulk copy
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

constexpr int kTrace = 8;   // stamps per block when tracing (include/ss_b200.h)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ configuration
template <int B>
struct Cfg {
    static constexpr int kCompute = 256;              // compute threads of the chain CTA
    static constexpr int kNT = kCompute + 64;         // + producer warp + publisher warp
    static constexpr int kFarWarps = kCompute / 32;   // helper warps streaming the far part
    static constexpr int kRPW = B / kFarWarps;        // far rows per helper warp
    static constexpr int kGrp = kRPW < 4 ? kRPW : 4;  // far rows gathered together
    static constexpr int kStages = 2;
    static constexpr int kRing = 8;                   // x of the last 8 blocks (Q <= 8)
    static constexpr int kPK = B * (B + 1) / 2;
    static constexpr int kNCap = near_cap(B);
    static constexpr int kCW = 16;
    static constexpr int kSegs = B / kCW;
    static constexpr int kNloc = B + 4;               // padded per-block row pointers (int32)
    static constexpr int kTPR = kCompute / B;         // near-phase threads per row
    // one stage: D_k^{-1} | near columns | near values | near row pointers | r_k
    static constexpr size_t kOffInv = 0;
    static constexpr size_t kOffNcol = kOffInv + (size_t)kPK * 16;
    static constexpr size_t kOffNval = kOffNcol + (size_t)kNCap * 4;
    static constexpr size_t kOffNloc = kOffNval + (size_t)kNCap * 16;
    static constexpr size_t kOffRfar = kOffNloc + (size_t)kNloc * 4;
    static constexpr size_t kStage = kOffRfar + (size_t)B * 16;
    static constexpr size_t kOffRing = kStage * kStages;
    static constexpr size_t kOffR = kOffRing + (size_t)kRing * B * 16;
    static constexpr size_t kOffPart = kOffR + (size_t)B * 16;
    static constexpr size_t kOffRowP = kOffPart + (size_t)kSegs * B * 16;
    static constexpr size_t kOffRowL = kOffRowP + (size_t)B * 8;
    static constexpr size_t kOffBar = kOffRowL + (size_t)B * 4;
    static constexpr size_t kSmem = kOffBar + 16 * kStages + 64;
    static_assert(kCompute % B == 0 && B % kFarWarps == 0 && kRPW % kGrp == 0 && B % 32 == 0, "layout");
    static_assert(kStage % 16 == 0 && kOffNval % 16 == 0 && kOffNloc % 16 == 0 && kOffRfar % 16 == 0, "TMA");
};

// Helper-side wait: return once the chain frontier (blocks < F published) reaches target.
// The CTA's view of F lives in shared memory; the warp holding sLock reads the global
// frontier word (one L2 round trip) and advances it.
__device__ __forceinline__ void helper_wait(int target, int* sF, int* sLock, const unsigned long long* xfront,
                                            uint32_t epoch) {
    const int lane = threadIdx.x & 31;
    int f = ld_acq_cta(sF);
    while (f < target) {
        int got = 0;
        if (lane == 0) got = atomicCAS(sLock, 0, 1) == 0;
        got = __shfl_sync(0xffffffffu, got, 0);
        if (got) {
            if (lane == 0) {
                const unsigned long long v = ld_acquire64(xfront);
                const int cnt = (uint32_t)(v >> 32) == epoch ? (int)(uint32_t)v : 0;
                if (cnt > ld_acq_cta(sF)) st_rel_cta(sF, cnt);
                st_rel_cta(sLock, 0);
            }
            __syncwarp();
        } else {
            __nanosleep(64);
        }
        f = ld_acq_cta(sF);
    }
    __syncwarp();   // every lane's later loads follow the acquire chain
}

template <int B>
__global__ void __launch_bounds__(Cfg<B>::kNT, 1)
k_chain_trsv(const TriArgs a, const double2* __restrict__ bvec, double2* out, double2* x, uint32_t epoch,
             unsigned long long* __restrict__ trace) {
    using C = Cfg<B>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* empty = full + C::kStages;
    int* sDone = reinterpret_cast<int*>(empty + C::kStages);
    int* sF = sDone + 1;
    int* sLock = sDone + 2;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int nblk = (int)a.nblk;
    const bool rev = a.rev != 0;
    auto phys = [&](int64_t i) -> int64_t { return rev ? n - 1 - i : i; };

    if (tid == 0) {
        for (int s = 0; s < C::kStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        *sDone = 0;
        *sF = 0;
        *sLock = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (blockIdx.x == 0) {
        // ============================================================ chain CTA
        if (warp == C::kCompute / 32) {   // producer: stage block k's operands (TMA)
            if (lane == 0) {
                for (int k = 0; k < nblk; k++) {
                    const int s = k % C::kStages;
                    if (k >= C::kStages) mbar_wait(empty + s, (uint32_t)((k / C::kStages - 1) & 1));
                    while (ld_acquire(a.fflag + k) != epoch) __nanosleep(20);
                    if (trace) trace[(int64_t)k * kTrace + 5] = gtime();
                    fence_proxy_async();   // r_k (generic-proxy stores of a helper) -> TMA reads
                    const int64_t nb0 = a.nbp[k];
                    const uint32_t cnt = (uint32_t)(a.nbp[k + 1] - nb0);
                    const uint32_t cpad = (cnt + 3u) & ~3u;
                    unsigned char* st = smem + C::kStage * s;
                    const uint32_t bytes = (uint32_t)(C::kPK * 16 + cpad * 4 + cnt * 16 + C::kNloc * 4 + B * 16);
                    mbar_expect_tx(full + s, bytes);
                    bulk_g2s(st + C::kOffInv, a.dinv + (int64_t)k * C::kPK, C::kPK * 16, full + s);
                    if (cnt) {
                        bulk_g2s(st + C::kOffNcol, a.ncol + nb0, cpad * 4, full + s);
                        bulk_g2s(st + C::kOffNval, a.nval + nb0, cnt * 16, full + s);
                    }
                    bulk_g2s(st + C::kOffNloc, a.nloc + (int64_t)k * C::kNloc, C::kNloc * 4, full + s);
                    bulk_g2s(st + C::kOffRfar, a.rfar + (int64_t)k * B, B * 16, full + s);
                }
            }
            return;
        }
        if (warp == C::kCompute / 32 + 1) {   // publisher: advance the global frontier word
            if (lane == 0) {
                int published = 0;
                while (published < nblk) {
                    const int d = ld_acq_cta(sDone);
                    if (d > published) {
                        st_release64(a.xfront, ((unsigned long long)epoch << 32) | (unsigned)d);

                        published = d;
                    } else {
                        __nanosleep(20);
                    }
                }
            }
            return;
        }
        // compute warps
        double2* ring = reinterpret_cast<double2*>(smem + C::kOffRing);
        double2* sR = reinterpret_cast<double2*>(smem + C::kOffR);
        double2* sPart = reinterpret_cast<double2*>(smem + C::kOffPart);
        constexpr int kRingMask = C::kRing * B - 1;
        for (int k = 0; k < nblk; k++) {
            const int s = k % C::kStages;
            unsigned char* st = smem + C::kStage * s;
            const double2* sInv = reinterpret_cast<const double2*>(st + C::kOffInv);
            const int32_t* sNcol = reinterpret_cast<const int32_t*>(st + C::kOffNcol);
            const double2* sNval = reinterpret_cast<const double2*>(st + C::kOffNval);
            const int32_t* sNloc = reinterpret_cast<const int32_t*>(st + C::kOffNloc);
            const double2* sRfar = reinterpret_cast<const double2*>(st + C::kOffRfar);
            mbar_wait(full + s, (uint32_t)((k / C::kStages) & 1));
            if (trace && tid == 0) trace[(int64_t)k * kTrace + 0] = gtime();
            // near part: kTPR threads per row, contiguous parts of the row's list
            {
                const int r = tid / C::kTPR, q = tid % C::kTPR;
                const int lo = sNloc[r], hi = sNloc[r + 1], len = hi - lo;
                const int e0 = lo + (q * len) / C::kTPR, e1 = lo + ((q + 1) * len) / C::kTPR;
                // 4 entries per trip: the column, value and x loads of a batch are issued
                // together (two dependent shared-memory round trips per batch, not per entry)
                double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
                int e = e0;
                for (; e + 4 <= e1; e += 4) {
                    const int c0 = sNcol[e], c1 = sNcol[e + 1], c2 = sNcol[e + 2], c3 = sNcol[e + 3];
                    const double2 v0 = sNval[e], v1 = sNval[e + 1], v2 = sNval[e + 2], v3 = sNval[e + 3];
                    const double2 x0 = ring[c0 & kRingMask], x1 = ring[c1 & kRingMask];
                    const double2 x2 = ring[c2 & kRingMask], x3 = ring[c3 & kRingMask];
                    acc = cfma(acc, v0, x0);
                    acc2 = cfma(acc2, v1, x1);
                    acc = cfma(acc, v2, x2);
                    acc2 = cfma(acc2, v3, x3);
                }
                for (; e < e1; e++) acc = cfma(acc, sNval[e], ring[sNcol[e] & kRingMask]);
                acc = cadd(acc, acc2);
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 6] = gtime();
#pragma unroll
                for (int o = 1; o < C::kTPR; o <<= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (q == 0) sR[r] = csub(sRfar[r], acc);
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 7] = gtime();
            }
            bar_compute(C::kCompute);
            if (trace && tid == 0) trace[(int64_t)k * kTrace + 1] = gtime();
            trimv::matvec_tiles<B, C::kCW, C::kCompute / 32>(sInv, sR, sPart, warp, lane);
            bar_compute(C::kCompute);
            if (trace && tid == 0) trace[(int64_t)k * kTrace + 2] = gtime();
            if (tid == 0) mbar_arrive(empty + s);   // stage s may be refilled
            if (tid < B) {
                const double2 v = trimv::sum_row<B, C::kCW>(sPart, tid);
                const int64_t i = (int64_t)k * B + tid;
                ring[i & kRingMask] = v;
                if (i < n) {
                    const int64_t pi = phys(i);
                    x[pi] = v;                              // kernel-space x (helpers read it)
                    if (a.operm) out[a.operm[pi]] = v;      // ILUTP: undo the column exchanges
                }
            }
            bar_compute(C::kCompute);
            if (tid == 0) {
                st_rel_cta(sDone, k + 1);
                if (trace) trace[(int64_t)k * kTrace + 3] = gtime();
            }
        }
        return;
    }

    // ================================================================ helper CTAs
    if (warp >= C::kFarWarps) return;
    const int H = gridDim.x - 1;
    int64_t* sRowP = reinterpret_cast<int64_t*>(smem + C::kOffRowP);
    int32_t* sRowL = reinterpret_cast<int32_t*>(smem + C::kOffRowL);
    for (int k = blockIdx.x - 1; k < nblk; k += H) {
        const int64_t row0 = (int64_t)k * B;

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
        // chunk c of every owned row before chunk c+1 of any (oldest sources first): issue
        // the column/value loads of all rows, wait once for the chunk's newest source
        // block, then gather x kGrp rows at a time
#pragma unroll 1
        for (int c = 0; c < nch; c++) {
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
            if (need >= 0) helper_wait(need / B + 1, sF, sLock, a.xfront, epoch);
#pragma unroll
            for (int g = 0; g < C::kRPW; g += C::kGrp) {
                double2 xv[C::kGrp];
#pragma unroll
                for (int r = 0; r < C::kGrp; r++)
                    if (cc[g + r] >= 0) xv[r] = ld_cg2(x + phys(cc[g + r]));
#pragma unroll
                for (int r = 0; r < C::kGrp; r++)
                    if (cc[g + r] >= 0) acc[g + r] = cfma(acc[g + r], vv[g + r], xv[r]);
            }
        }
#pragma unroll
        for (int r = 0; r < C::kRPW; r++) {
            const double2 sm = warp_sum2(acc[r]);
            const int64_t i = row0 + warp * C::kRPW + r;
            if (lane == 0) a.rfar[i] = (i < n) ? csub(__ldg(bvec + phys(i)), sm) : make_double2(0.0, 0.0);
        }
        bar_compute(C::kCompute);
        if (tid == 0) {
            st_release(a.fflag + k, epoch);
            if (trace) trace[(int64_t)k * kTrace + 4] = gtime();
        }
    }
}

template <int B>
void prepare(DevBlockTri& T) {
    using C = Cfg<B>;
    auto fn = k_chain_trsv<B>;
    SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem));
    int dev = 0, sms = 0, per = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, C::kNT, C::kSmem));
    SSB_CHECK(per >= 1, SS_ERR_CUDA, "block trsv kernel does not fit on an SM");
    // chain CTA + helpers; one CTA per SM (more helpers than blocks are useless)
    T.grid = (int)std::max<int64_t>(2, std::min<int64_t>(T.nblk + 1, (int64_t)sms));
    T.nt = C::kNT;
}

template <int B>
void launch(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    using C = Cfg<B>;
    auto fn = k_chain_trsv<B>;
    if (T.grid == 0) prepare<B>(T);
    T.epoch++;
    TriArgs a = T.args();
    uint32_t ep = T.epoch;
    double2* xw = T.operm ? T.xwork : x;
    void* args[] = {(void*)&a, (void*)&b, (void*)&x, (void*)&xw, (void*)&ep, (void*)&trace};
    SSB_CUDA(cudaLaunchCooperativeKernel((const void*)fn, dim3(T.grid), dim3(C::kNT), args, C::kSmem, s));
    SSB_LAUNCHED();
}

}  // namespace

size_t block_trsv_packed(int B) { return (size_t)B * (B + 1) / 2; }

void block_trsv_prepare(DevBlockTri& T) {
    switch (T.B) {
        case 32: prepare<32>(T); break;
        case 64: prepare<64>(T); break;
        default: SSB_CHECK(false, SS_ERR_ARG, "block substitution supports B = 32 or 64");
    }
}

void block_trsv(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    if (T.n == 0) return;
    switch (T.B) {
        case 32: launch<32>(T, b, x, s, trace); break;
        case 64: launch<64>(T, b, x, s, trace); break;
        default: SSB_CHECK(false, SS_ERR_ARG, "block substitution supports B = 32 or 64");
    }
}

}  // namespace ssb
