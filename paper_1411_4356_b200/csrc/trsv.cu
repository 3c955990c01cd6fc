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
// v5 (this file): block substitution on a chain SM, a lieutenant SM of the same thread-
// block cluster, and the other SMs as helpers.
// Rows are cut into blocks of B consecutive rows; in the kernel's index space (U
// reversed at setup, i' = n-1-i, so both factors are lower triangular)
//     x_k = D_k^{-1} ( b_k - sum_{j<k} T_kj x_j ),
// with the explicit inverse of every B x B diagonal block D_k precomputed at setup.
// The row entries left of block k are split at setup into
//   * "far"  (source blocks <= k-Q): the bulk of the factor bytes.  Helper CTAs stream
//     them in fixed 32-entry chunks as soon as the chain's completion frontier covers
//     the chunk's sources, and publish r_k = b_k - (far part) with a release flag;
//   * "near" (source blocks k-Q+1 .. k-1): per block two short lists -- list A (sources
//     k-Dc+1 .. k-1) applied on the chain SM, list B (k-Q+1 .. k-Dc) applied by the
//     lieutenant, which receives every x block through DSMEM (st.shared::cluster) and
//     returns its partial sums of block k the same way, Dc-1 steps ahead of the chain.
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
constexpr int kProducerSleep = 32, kPublisherSleep = 32;   // back-off of the polling warps (ns)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ configuration
// ------------------------------------------------------------------ cluster (DSMEM) helpers
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {   // peer CTA's address
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
// 16-byte store into a peer CTA's shared memory that completes 16 bytes of the peer's
// mbarrier transaction: no fence on the producer side, the consumer waits on the mbarrier
__device__ __forceinline__ void st_async2(uint32_t addr, double2 v, uint32_t mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(v.x), "d"(v.y), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release;\nbarrier.cluster.wait.acquire;" ::: "memory");
}

// ------------------------------------------------------------------ configuration
template <int B>
struct Cfg {
    static constexpr int kCompute = 256;              // compute threads per role
    static constexpr int kNT = kCompute + 64;         // + producer warp + publisher warp
    static constexpr int kFarWarps = kCompute / 32;   // helper warps streaming the far part
    static constexpr int kRPW = B / kFarWarps;        // far rows per helper warp
    static constexpr int kGrp = kRPW < 4 ? kRPW : 4;  // far rows gathered together
    static constexpr int kStages = 2;
    static constexpr int kRing = 8;                   // x of the last 8 blocks (Q <= 8)
    static constexpr int kPbuf = 4;                   // lieutenant partial-sum slots (Dc <= 4)
    static constexpr int kPK = B * (B + 1) / 2;
    static constexpr int kCapA = near_cap_a(B), kCapB = near_cap_b(B);
    static constexpr int kCW = B <= 32 ? 8 : 16;    // mat-vec tile width (4 tiles for B = 32)
    static constexpr int kSegs = B / kCW;
    static constexpr int kNloc = B + 4;               // padded per-block row pointers (int32)
    static constexpr int kTPR = kCompute / B;         // near-phase threads per row
    // chain stage: D_k^{-1} | list A columns | list A values | list A row pointers | r_k
    static constexpr size_t kOffInv = 0;
    static constexpr size_t kOffAcol = kOffInv + (size_t)kPK * 16;
    static constexpr size_t kOffAval = kOffAcol + (size_t)kCapA * 4;
    static constexpr size_t kOffAloc = kOffAval + (size_t)kCapA * 16;
    static constexpr size_t kOffRfar = kOffAloc + (size_t)kNloc * 4;
    static constexpr size_t kChainStage = kOffRfar + (size_t)B * 16;
    // lieutenant stage: list B columns | list B values | list B row pointers
    static constexpr size_t kOffBcol = 0;
    static constexpr size_t kOffBval = kOffBcol + (size_t)kCapB * 4;
    static constexpr size_t kOffBloc = kOffBval + (size_t)kCapB * 16;
    static constexpr size_t kLtStage = kOffBloc + (size_t)kNloc * 4;
    static constexpr size_t kStage = kChainStage > kLtStage ? kChainStage : kLtStage;
    static constexpr size_t kOffRing = kStage * kStages;
    static constexpr size_t kOffR = kOffRing + (size_t)kRing * B * 16;
    static constexpr size_t kOffPart = kOffR + (size_t)B * 16;
    static constexpr size_t kOffPbuf = kOffPart + (size_t)kSegs * B * 16;
    static constexpr size_t kOffRowP = kOffPbuf + (size_t)kPbuf * B * 16;
    static constexpr size_t kOffRowL = kOffRowP + (size_t)B * 8;
    static constexpr size_t kOffBar = kOffRowL + (size_t)B * 4;
    static constexpr size_t kOffXbar = kOffBar + 16 * kStages + 64;   // lieutenant: x block j landed
    static constexpr size_t kOffPbar = kOffXbar + 8 * kRing;          // chain: partial of block k landed
    static constexpr size_t kSmem = kOffPbar + 8 * kPbuf;
    static_assert(kCompute % B == 0 && B % kFarWarps == 0 && kRPW % kGrp == 0 && B % 32 == 0, "layout");
    static_assert(kChainStage % 16 == 0 && kLtStage % 16 == 0 && kOffAval % 16 == 0 && kOffAloc % 16 == 0 &&
                      kOffRfar % 16 == 0 && kOffBval % 16 == 0 && kOffBloc % 16 == 0,
                  "TMA alignment");
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

// Near products of one block's list (row pointers loc, kTPR threads per row, contiguous
// parts): returns the row sum on lane q == 0 of each row group, x read from the ring.
template <int B>
__device__ __forceinline__ double2 near_rows(const int32_t* loc, const int32_t* col, const double2* val,
                                             const double2* ring, int tid) {
    using C = Cfg<B>;
    constexpr int kRingMask = C::kRing * B - 1;
    const int r = tid / C::kTPR, q = tid % C::kTPR;
    const int lo = loc[r], hi = loc[r + 1], len = hi - lo;
    const int e0 = lo + (q * len) / C::kTPR, e1 = lo + ((q + 1) * len) / C::kTPR;
    double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
    int e = e0;
    for (; e + 4 <= e1; e += 4) {
        const int c0 = col[e], c1 = col[e + 1], c2 = col[e + 2], c3 = col[e + 3];
        const double2 v0 = val[e], v1 = val[e + 1], v2 = val[e + 2], v3 = val[e + 3];
        const double2 x0 = ring[c0 & kRingMask], x1 = ring[c1 & kRingMask];
        const double2 x2 = ring[c2 & kRingMask], x3 = ring[c3 & kRingMask];
        acc = cfma(acc, v0, x0);
        acc2 = cfma(acc2, v1, x1);
        acc = cfma(acc, v2, x2);
        acc2 = cfma(acc2, v3, x3);
    }
    for (; e < e1; e++) acc = cfma(acc, val[e], ring[col[e] & kRingMask]);
    acc = cadd(acc, acc2);
#pragma unroll
    for (int o = 1; o < C::kTPR; o <<= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    return acc;
}

// Stage one near list block (TMA): columns (padded to 4), values, row pointers.
__device__ __forceinline__ uint32_t stage_near(unsigned char* col_dst, unsigned char* val_dst,
                                               unsigned char* loc_dst, const int64_t* bp, const int32_t* col,
                                               const double2* val, const int32_t* loc, int k, int nloc,
                                               uint64_t* bar, bool issue) {
    const int64_t b0 = bp[k];
    const uint32_t cnt = (uint32_t)(bp[k + 1] - b0);   // already a multiple of 4
    const uint32_t bytes = cnt * 20 + (uint32_t)nloc * 4;
    if (issue) {
        if (cnt) {
            bulk_g2s(col_dst, col + b0, cnt * 4, bar);
            bulk_g2s(val_dst, val + b0, cnt * 16, bar);
        }
        bulk_g2s(loc_dst, loc + (int64_t)k * nloc, (uint32_t)nloc * 4, bar);
    }
    return bytes;
}

template <int B>
__global__ void __launch_bounds__(Cfg<B>::kNT, 1)
k_chain_trsv(const TriArgs a, const double2* __restrict__ bvec, double2* out, double2* x, uint32_t epoch,
             unsigned long long* __restrict__ trace) {
    using C = Cfg<B>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
    uint64_t* empty = full + C::kStages;
    int* sDone = reinterpret_cast<int*>(empty + C::kStages);   // chain: blocks of x done
    int* sF = sDone + 1;                                          // helpers: frontier view
    int* sLock = sDone + 2;
    int* sPub = sDone + 3;                                        // chain: blocks published to global
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + C::kOffXbar);
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + C::kOffPbar);
    double2* ring = reinterpret_cast<double2*>(smem + C::kOffRing);
    double2* pbuf = reinterpret_cast<double2*>(smem + C::kOffPbuf);
    constexpr int kRingMask = C::kRing * B - 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int nblk = (int)a.nblk;
    const int Dc = a.Dc;
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
        *sPub = 0;
        for (int j = 0; j < C::kRing; j++) mbar_init(xbar + j, 1);
        for (int j = 0; j < C::kPbuf; j++) mbar_init(pbar + j, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();   // counters of both CTAs of a cluster initialised before any DSMEM access

    if (blockIdx.x <= 1) {
        const bool chain = blockIdx.x == 0;
        const uint32_t peer = chain ? 1u : 0u;
        if (warp == C::kCompute / 32) {
            // ------------------------------------------------ producer: TMA staging
            if (lane == 0) {
                for (int k = 0; k < nblk; k++) {
                    const int s = k % C::kStages;
                    if (k >= C::kStages) mbar_wait(empty + s, (uint32_t)((k / C::kStages - 1) & 1));
                    unsigned char* st = smem + C::kStage * s;
                    if (chain) {
                        while (ld_acquire(a.fflag + k) != epoch) __nanosleep(kProducerSleep);
                        if (trace) trace[(int64_t)k * kTrace + 5] = gtime();
                        fence_proxy_async();   // r_k (generic-proxy stores of a helper) -> TMA reads
                        const uint32_t nb = stage_near(nullptr, nullptr, nullptr, a.nbpA, a.ncolA, a.nvalA,
                                                       a.nlocA, k, C::kNloc, full + s, false);
                        mbar_expect_tx(full + s, (uint32_t)(C::kPK * 16 + B * 16) + nb);
                        bulk_g2s(st + C::kOffInv, a.dinv + (int64_t)k * C::kPK, C::kPK * 16, full + s);
                        stage_near(st + C::kOffAcol, st + C::kOffAval, st + C::kOffAloc, a.nbpA, a.ncolA, a.nvalA,
                                   a.nlocA, k, C::kNloc, full + s, true);
                        bulk_g2s(st + C::kOffRfar, a.rfar + (int64_t)k * B, B * 16, full + s);
                    } else {
                        const uint32_t nb = stage_near(nullptr, nullptr, nullptr, a.nbpB, a.ncolB, a.nvalB,
                                                       a.nlocB, k, C::kNloc, full + s, false);
                        mbar_expect_tx(full + s, nb);
                        stage_near(st + C::kOffBcol, st + C::kOffBval, st + C::kOffBloc, a.nbpB, a.ncolB, a.nvalB,
                                   a.nlocB, k, C::kNloc, full + s, true);
                    }
                }
            }
        } else if (warp == C::kCompute / 32 + 1) {
            // ------------------------------------------------ publisher (chain only): copies
            // finished x blocks from the ring to global memory (and through the iLUTP column
            // permutation to the output), then advances the gpu-scope frontier word
            if (chain) {
                int published = 0;
                while (published < nblk) {
                    const int d = ld_acq_cta(sDone);
                    if (d > published) {
                        for (int j = published; j < d; j++)
                            for (int r = lane; r < B; r += 32) {
                                const int64_t i = (int64_t)j * B + r;
                                if (i < n) {
                                    const double2 v = ring[i & kRingMask];
                                    const int64_t pi = phys(i);
                                    x[pi] = v;
                                    if (a.operm) out[a.operm[pi]] = v;
                                }
                            }
                        __syncwarp();
                        if (lane == 0) {
                            st_release64(a.xfront, ((unsigned long long)epoch << 32) | (unsigned)d);
                            st_rel_cta(sPub, d);
                        }
                        published = d;
                    } else {
                        __nanosleep(kPublisherSleep);
                    }
                }
            }
        } else if (chain) {
            // ------------------------------------------------ chain compute warps
            double2* sR = reinterpret_cast<double2*>(smem + C::kOffR);
            double2* sPart = reinterpret_cast<double2*>(smem + C::kOffPart);
            const uint32_t peer_ring = mapa(smem_u32(ring), peer);
            const uint32_t peer_xbar = mapa(smem_u32(xbar), peer);
            for (int k = 0; k < nblk; k++) {
                const int s = k % C::kStages;
                unsigned char* st = smem + C::kStage * s;
                const double2* sInv = reinterpret_cast<const double2*>(st + C::kOffInv);
                const double2* sRfar = reinterpret_cast<const double2*>(st + C::kOffRfar);
                mbar_wait(full + s, (uint32_t)((k / C::kStages) & 1));
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 0] = gtime();
                const double2 accA = near_rows<B>(reinterpret_cast<const int32_t*>(st + C::kOffAloc),
                                                  reinterpret_cast<const int32_t*>(st + C::kOffAcol),
                                                  reinterpret_cast<const double2*>(st + C::kOffAval), ring, tid);
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 6] = gtime();
                if (tid % C::kTPR == 0) {
                    const int r = tid / C::kTPR, pk = k % C::kPbuf;
                    // the lieutenant's partial of block k (B values, st.async) lands on pbar[pk]
                    if (r == 0) mbar_expect_tx(pbar + pk, (uint32_t)(B * 16));
                    mbar_wait(pbar + pk, (uint32_t)((k / C::kPbuf) & 1));
                    sR[r] = csub(csub(sRfar[r], accA), pbuf[pk * B + r]);
                }
                bar_compute(C::kCompute);
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 1] = gtime();
                trimv::matvec_tiles<B, C::kCW, C::kCompute / 32>(sInv, sR, sPart, warp, lane);
                bar_compute(C::kCompute);
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 2] = gtime();
                if (tid == 0) mbar_arrive(empty + s);   // stage s may be refilled
                if (tid < B) {
                    // ring slot of block k held block k-8: the publisher must have copied it
                    if (k >= C::kRing)
                        while (ld_acq_cta(sPub) < k - C::kRing + 1) {
                        }
                    const double2 v = trimv::sum_row<B, C::kCW>(sPart, tid);
                    const int64_t i = (int64_t)k * B + tid;
                    ring[i & kRingMask] = v;
                    st_async2(peer_ring + (uint32_t)((i & kRingMask) * 16), v,
                              peer_xbar + (uint32_t)((k % C::kRing) * 8));   // lieutenant's ring
                }
                bar_compute(C::kCompute);
                if (tid == 0) {
                    st_rel_cta(sDone, k + 1);   // the publisher copies x_k to global memory
                    if (trace) trace[(int64_t)k * kTrace + 3] = gtime();
                }
            }
        } else {
            // ------------------------------------------------ lieutenant compute warps
            const uint32_t peer_pbuf = mapa(smem_u32(pbuf), peer);
            const uint32_t peer_pbar = mapa(smem_u32(pbar), peer);
            int xseen = 0;   // x blocks < xseen have landed in the ring
            for (int k = 0; k < nblk; k++) {
                const int s = k % C::kStages;
                unsigned char* st = smem + C::kStage * s;
                mbar_wait(full + s, (uint32_t)((k / C::kStages) & 1));
                // list B of block k reads x of blocks <= k - Dc: consume their arrivals in
                // order (each xbar phase exactly once); pbuf slot k % 4 was last read by
                // the chain for block k - 4 < k - Dc + 1
                for (; xseen <= k - Dc; xseen++) {
                    const int j = xseen % C::kRing;
                    if (tid == 0) mbar_expect_tx(xbar + j, (uint32_t)(B * 16));
                    mbar_wait(xbar + j, (uint32_t)((xseen / C::kRing) & 1));
                }
                if (trace && tid == 0) trace[(int64_t)k * kTrace + 7] = gtime();
                const double2 accB = near_rows<B>(reinterpret_cast<const int32_t*>(st + C::kOffBloc),
                                                  reinterpret_cast<const int32_t*>(st + C::kOffBcol),
                                                  reinterpret_cast<const double2*>(st + C::kOffBval), ring, tid);
                if (tid % C::kTPR == 0) {
                    const int pk = k % C::kPbuf;
                    st_async2(peer_pbuf + (uint32_t)((pk * B + tid / C::kTPR) * 16), accB, peer_pbar + (uint32_t)(pk * 8));
                }
                bar_compute(C::kCompute);
                if (tid == 0) mbar_arrive(empty + s);
            }
            for (; xseen < nblk; xseen++) {   // drain the remaining arrivals before leaving
                const int j = xseen % C::kRing;
                if (tid == 0) mbar_expect_tx(xbar + j, (uint32_t)(B * 16));
                mbar_wait(xbar + j, (uint32_t)((xseen / C::kRing) & 1));
            }
        }
        // all threads of both CTAs: no CTA of the cluster leaves while its peer may still
        // access its shared memory
        __syncwarp();
        cluster_sync();
        return;
    }

    // ================================================================ helper CTAs
    if (warp >= C::kFarWarps) return;
    const int H = gridDim.x - 2;
    int64_t* sRowP = reinterpret_cast<int64_t*>(smem + C::kOffRowP);
    int32_t* sRowL = reinterpret_cast<int32_t*>(smem + C::kOffRowL);
    for (int k = blockIdx.x - 2; k < nblk; k += H) {
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
    SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    int dev = 0, sms = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // clusters of 2 (chain + lieutenant, then pairs of helpers), one CTA per SM; every
    // cluster must be resident at once (the CTAs spin on one another)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(C::kNT);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    cfg.gridDim = dim3((unsigned)(sms & ~1));
    SSB_CUDA(cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg));
    SSB_CHECK(clusters >= 2, SS_ERR_CUDA, "block trsv: fewer than two co-resident CTA pairs");
    const int64_t want = std::max<int64_t>(4, 2 * ((T.nblk + 3) / 2));   // chain, lieutenant, >= 2 helpers
    T.grid = (int)std::min<int64_t>(want, 2 * (int64_t)clusters);
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
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(T.grid);
    cfg.blockDim = dim3(C::kNT);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SSB_CUDA(cudaLaunchKernelEx(&cfg, fn, a, b, x, xw, ep, trace));
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
