// trsv.cu -- forward / backward substitution with the ILU factors (M^{-1} = Pi U^{-1} L^{-1}).
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
// v6 (this file): block substitution whose dependency chain runs in ONE WARP.
// Rows are cut into blocks of B = 32 consecutive rows; in the kernel's index space (U
// reversed at setup, i' = n-1-i, so both factors are lower triangular)
//     x_k = D_k^{-1} ( b_k - sum_{j<k} T_kj x_j ) = y_k - G_k x_{k-1},
//     y_k = D_k^{-1} ( b_k - sum_{j<k-1} T_kj x_j ),   G_k = D_k^{-1} T_{k,k-1},
// with D_k^{-1} and G_k (dense 32 x 32) precomputed at setup.  Only x_k = y_k - G_k x_{k-1}
// is on the chain: one warp, lane i = row i, x_{k-1} in registers (shuffles), G_k out of
// shared memory -- no barrier on the critical path.  Everything else runs ahead of it:
//   * y warps (7 warps of the chain CTA): y_k from the entries with source distance 2
//     (list A, x_{k-2} from the shared-memory ring), the lieutenants' partial sums, the
//     helpers' r_k and the triangular mat-vec with D_k^{-1} (trimv.cuh), one block ahead;
//   * lieutenants (3 CTAs of the chain's thread-block cluster): the entries with source
//     distance 3 .. Q_k-1 (list B), each for a third of the rows; every x block reaches
//     their rings by st.async (DSMEM) and their partial sums come back the same way,
//     both completing mbarrier transactions (no fences on the chain);
//   * helpers (the other SMs): the "far" entries (source distance >= Q_k, the bulk of
//     the factor bytes) streamed in fixed 32-entry chunks as the published frontier
//     covers them; r_k = b_k - far part is published with a gpu-scope release flag;
//   * producer warp: TMA bulk copies (cp.async.bulk + mbarrier) of D_k^{-1}, G_k, list A
//     and r_k (chain CTA) or list B (lieutenants), stages ahead;
//   * publisher warp: copies finished x blocks from the ring to global memory (and
//     through the iLUTP column permutation to the output, x = Pi y) and advances the
//     frontier word (epoch << 32 | blocks done) with a gpu-scope release.
// One CTA per SM, clusters of 4; the grid never exceeds the co-resident cluster count, so
// the spin waits cannot deadlock.  Every reduction has a fixed order: the result is
// deterministic for given (B, Q).
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
constexpr int kProducerSleep = 32, kPublisherSleep = 16;   // back-off of the polling warps (ns)
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

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
    static constexpr int kCluster = 4;                // chain + 3 lieutenants
    static constexpr int kLt = kCluster - 1;
    static constexpr int kCompute = 256;              // compute threads (8 warps)
    static constexpr int kNT = kCompute + 64;         // + producer warp + publisher warp
    // chain CTA warp roles, placed for the SMSP arbiter (highest warp id first): the chain
    // team = warps 6, 7, 8, 9 (the highest id on each SMSP), y = warps 2 .. 5, producer 0,
    // publisher 1.
    static constexpr int kTeam = 4, kTeamW0 = 6;
    static constexpr int kYWarps = 4, kYW0 = 2;
    static constexpr int kWProducerChain = 0, kWPublisher = 1;
    static constexpr int kSlice = B / kTeam;          // columns of G per team warp
    static constexpr int kCapA = near_cap_a(B);
    static constexpr int kFarWarps = kCompute / 32;   // helper warps streaming the far part
    static constexpr int kRPW = B / kFarWarps;        // far rows per helper warp
    static constexpr int kGrp = kRPW < 4 ? kRPW : 4;
    static constexpr int kStages = 3;
    static constexpr int kRing = 8;                   // x of the last 8 blocks (Q <= 8)
    static constexpr int kPbuf = 4;                   // lieutenant partial-sum slots
    static constexpr int kYbuf = 2;                   // y slots
    static constexpr int kPK = B * (B + 1) / 2;
    static constexpr int kCapB = near_cap_b(B);
    static constexpr int kCW = 8;                     // mat-vec tile width
    static constexpr int kSegs = B / kCW;
    static constexpr int kNloc = B + 4;               // padded per-block row pointers (int32)

    static constexpr int kTPRl = 8;                   // lieutenants: threads per row
    // chain stage: D_k^{-1} | G1_k | G2_k | list A (d = 3) columns | values | row pointers | r_k
    static constexpr size_t kOffInv = 0;
    static constexpr size_t kOffG = kOffInv + (size_t)kPK * 16;
    static constexpr size_t kOffAcol = kOffG + (size_t)2 * B * B * 16;
    static constexpr size_t kOffAval = kOffAcol + (size_t)kCapA * 4;
    static constexpr size_t kOffAloc = kOffAval + (size_t)kCapA * 16;
    static constexpr size_t kOffRfar = kOffAloc + (size_t)kNloc * 4;
    static constexpr size_t kChainStage = kOffRfar + (size_t)B * 16;
    // lieutenant stage: list B columns | list B values | list B row pointers
    static constexpr size_t kOffBcol = 0;
    static constexpr size_t kOffBval = kOffBcol + (size_t)kCapB * 4;
    static constexpr size_t kOffBloc = kOffBval + (size_t)kCapB * 16;
    static constexpr size_t kLtStage = kOffBloc + (size_t)kNloc * 4;
    static constexpr int kLtStages = 2;
    static constexpr size_t kStageRegion =
        kChainStage * kStages > kLtStage * kLtStages ? kChainStage * kStages : kLtStage * kLtStages;
    static constexpr size_t kOffRing = kStageRegion;
    static constexpr size_t kOffR = kOffRing + (size_t)kRing * B * 16;
    static constexpr size_t kOffPart = kOffR + (size_t)2 * B * 16;
    static constexpr int kTPRy = kYWarps * 32 / B;     // y warps: threads per row of list A
    static constexpr int kPartRows = kSegs > kTPRy ? kSegs : kTPRy;
    static constexpr size_t kOffPbuf = kOffPart + (size_t)kPartRows * B * 16;
    static constexpr size_t kOffYbuf = kOffPbuf + (size_t)kPbuf * B * 16;
    static constexpr size_t kOffTpart = kOffYbuf + (size_t)kYbuf * B * 16;   // [2][kTeam][B] partials
    static constexpr size_t kOffRowP = kOffTpart + (size_t)2 * kTeam * B * 16;
    static constexpr size_t kOffRowL = kOffRowP + (size_t)B * 8;
    static constexpr size_t kOffBar = kOffRowL + (size_t)B * 4;
    // mbarriers: full/empty per stage, xbar (lieutenant: x block landed), pbar (chain:
    // partial landed), yfull/yempty (y slots), then int counters
    static constexpr size_t kOffFull = kOffBar;
    static constexpr size_t kOffEmpty = kOffFull + 8 * kStages;
    static constexpr size_t kOffXbar = kOffEmpty + 8 * kStages;
    static constexpr size_t kOffPbar = kOffXbar + 8 * kRing;
    static constexpr size_t kOffYfull = kOffPbar + 8 * kPbuf;
    static constexpr size_t kOffYempty = kOffYfull + 8 * kYbuf;
    static constexpr size_t kOffPready = kOffYempty + 8 * kYbuf;
    static constexpr size_t kOffInts = kOffPready + 8 * 2;
    static constexpr size_t kSmem = kOffInts + 64;
    static_assert(B == 32, "the chain warp holds one row per lane");
    static_assert(kCompute % B == 0 && B % kFarWarps == 0 && kRPW % kGrp == 0, "layout");
    static_assert(kChainStage % 16 == 0 && kLtStage % 16 == 0 && kOffG % 16 == 0 && kOffRfar % 16 == 0 &&
                      kOffAval % 16 == 0 && kOffAloc % 16 == 0 && kOffBval % 16 == 0 && kOffBloc % 16 == 0,
                  "TMA alignment");
    static_assert(kSmem <= 232448, "shared memory");
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

// Near products of row r of one block's list (TPR threads per row, contiguous parts,
// thread q of the row): returns the row sum on every thread of the row group, x read
// from the ring.  TPR need not be a power of two; the groups must not straddle warps
// unevenly, so the reduction goes through shared memory when TPR is not a power of two.
template <int B, int TPR>
__device__ __forceinline__ double2 near_part(const int32_t* loc, const int32_t* col, const double2* val,
                                             const double2* ring, int r, int q) {
    constexpr int kRingMask = Cfg<B>::kRing * B - 1;
    const int lo = loc[r], hi = loc[r + 1], len = hi - lo;
    const int e0 = lo + (q * len) / TPR, e1 = lo + ((q + 1) * len) / TPR;
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
    return cadd(acc, acc2);
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

__device__ __forceinline__ void bar_named(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int B>
__global__ void __launch_bounds__(Cfg<B>::kNT, 1)
k_chain_trsv(const TriArgs a, const double2* __restrict__ bvec, double2* out, double2* x, uint32_t epoch,
             unsigned long long* __restrict__ trace) {
    using C = Cfg<B>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kOffFull);
    uint64_t* empty = reinterpret_cast<uint64_t*>(smem + C::kOffEmpty);
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + C::kOffXbar);
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + C::kOffPbar);
    uint64_t* yfull = reinterpret_cast<uint64_t*>(smem + C::kOffYfull);
    uint64_t* yempty = reinterpret_cast<uint64_t*>(smem + C::kOffYempty);
    double2* tpart = reinterpret_cast<double2*>(smem + C::kOffTpart);
    uint64_t* pready = reinterpret_cast<uint64_t*>(smem + C::kOffPready);
    int* sDone = reinterpret_cast<int*>(smem + C::kOffInts);   // chain: blocks of x done
    int* sF = sDone + 1;                                          // helpers: frontier view
    int* sLock = sDone + 2;
    int* sPub = sDone + 3;                                        // chain: blocks published
    double2* ring = reinterpret_cast<double2*>(smem + C::kOffRing);
    double2* pbuf = reinterpret_cast<double2*>(smem + C::kOffPbuf);
    double2* ybuf = reinterpret_cast<double2*>(smem + C::kOffYbuf);
    constexpr int kRingMask = C::kRing * B - 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int nblk = (int)a.nblk;
    const bool rev = a.rev != 0;
    auto phys = [&](int64_t i) -> int64_t { return rev ? n - 1 - i : i; };
    const int role = blockIdx.x < C::kCluster ? (int)blockIdx.x : -1;   // 0 chain, 1..3 lieutenants
    const bool chain = role == 0;

    if (tid == 0) {
        for (int s = 0; s < C::kStages; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, chain ? 2 + C::kTeam : 1);   // chain CTA: the y team's 2 warps + each team warp
        }
        for (int j = 0; j < C::kRing; j++) mbar_init(xbar + j, 1);
        for (int j = 0; j < C::kPbuf; j++) mbar_init(pbar + j, 1);
        for (int j = 0; j < C::kYbuf; j++) {
            mbar_init(yfull + j, 2);
            mbar_init(yempty + j, C::kTeam);
        }
        for (int j = 0; j < 2; j++) mbar_init(pready + j, C::kTeam);
        *sDone = 0;
        *sF = 0;
        *sLock = 0;
        *sPub = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();   // barriers and counters of every CTA initialised before any DSMEM access

    if (role >= 0) {
        const int nst = chain ? C::kStages : C::kLtStages;
        const size_t stsz = chain ? C::kChainStage : C::kLtStage;
        const int wprod = chain ? C::kWProducerChain : C::kCompute / 32;
        if (warp == wprod) {
            // ------------------------------------------------ producer: TMA staging
            if (lane == 0) {
                for (int k = 0; k < nblk; k++) {
                    const int s = k % nst;
                    if (k >= nst) mbar_wait(empty + s, (uint32_t)((k / nst - 1) & 1));
                    unsigned char* st = smem + stsz * s;
                    if (chain) {
                        while (ld_acquire(a.fflag + k) != epoch) __nanosleep(kProducerSleep);
                        if (trace) trace[(int64_t)k * kTrace + 5] = gtime();
                        fence_proxy_async();   // r_k (generic-proxy stores of a helper) -> TMA reads
                        const uint32_t nb = stage_near(nullptr, nullptr, nullptr, a.nbpA, a.ncolA, a.nvalA,
                                                       a.nlocA, k, C::kNloc, full + s, false);
                        mbar_expect_tx(full + s, (uint32_t)(C::kPK * 16 + 2 * B * B * 16 + B * 16) + nb);
                        bulk_g2s(st + C::kOffInv, a.dinv + (int64_t)k * C::kPK, C::kPK * 16, full + s);
                        bulk_g2s(st + C::kOffG, a.G + (int64_t)k * 2 * B * B, 2 * B * B * 16, full + s);
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
        } else if (chain && warp == C::kWPublisher) {
            // ------------------------------------------------ publisher: x blocks from the ring to
            // global memory (and through the iLUTP column permutation to the output), to the
            // lieutenants' rings (st.async, completing their mbarrier transactions), then the
            // gpu-scope frontier word
            uint32_t peer_ring[C::kLt], peer_xbar[C::kLt];
#pragma unroll
            for (int l = 0; l < C::kLt; l++) {
                peer_ring[l] = mapa(smem_u32(ring), (uint32_t)(l + 1));
                peer_xbar[l] = mapa(smem_u32(xbar), (uint32_t)(l + 1));
            }
            int published = 0;
            while (published < nblk) {
                const int d = ld_acq_cta(sDone);
                if (d > published) {
                    for (int j = published; j < d; j++) {
                        const int64_t i = (int64_t)j * B + lane;
                        const double2 v = ring[i & kRingMask];
#pragma unroll
                        for (int l = 0; l < C::kLt; l++)
                            st_async2(peer_ring[l] + (uint32_t)((i & kRingMask) * 16), v,
                                      peer_xbar[l] + (uint32_t)((j % C::kRing) * 8));
                        if (i < n) {
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
        } else if (chain && warp >= C::kTeamW0) {
            // ------------------------------------------------ chain team (4 warps):
            // x_k = y_k - sum_w [ G1_k[:, slice_w] x_{k-1}[slice_w] + G2_k[:, slice_w] x_{k-2}[slice_w] ]
            // Warp w owns 8 columns; the G2 term of block k+1 (which needs x_{k-1}) is formed
            // in step k's tail.  One named barrier per step; every team warp then reduces the
            // partials itself, so all of them hold x_k (lane = row) for the next step.
            const int tw = warp - C::kTeamW0;
            const int j0 = tw * C::kSlice;
            double2 g1[C::kSlice], g2[C::kSlice];
            auto load_g = [&](int k) {   // G1_k (stage k) and G2_{k+1} (stage k+1); release stage k
                const int s = k % C::kStages;
                mbar_wait(full + s, (uint32_t)((k / C::kStages) & 1));
                const double2* G1 = reinterpret_cast<const double2*>(smem + C::kChainStage * s + C::kOffG);
#pragma unroll
                for (int u = 0; u < C::kSlice; u++) g1[u] = G1[(j0 + u) * B + lane];
                if (k + 1 < nblk) {
                    const int s1 = (k + 1) % C::kStages;
                    mbar_wait(full + s1, (uint32_t)(((k + 1) / C::kStages) & 1));
                    const double2* G2 =
                        reinterpret_cast<const double2*>(smem + C::kChainStage * s1 + C::kOffG) + B * B;
#pragma unroll
                    for (int u = 0; u < C::kSlice; u++) g2[u] = G2[(j0 + u) * B + lane];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);   // this warp is done with stage k
            };
            double2 xk = make_double2(0.0, 0.0);      // x_{k-1}[lane]
            double2 carry = make_double2(0.0, 0.0);   // G2_k[lane, slice] x_{k-2}[slice]
            if (nblk > 0) load_g(0);
            for (int k = 0; k < nblk; k++) {
                const int yb = k % C::kYbuf;
                double2 xs[C::kSlice];
#pragma unroll
                for (int u = 0; u < C::kSlice; u++) {
                    xs[u].x = __shfl_sync(0xffffffffu, xk.x, j0 + u);
                    xs[u].y = __shfl_sync(0xffffffffu, xk.y, j0 + u);
                }
                double2 p0 = carry, p1 = make_double2(0.0, 0.0);
#pragma unroll
                for (int u = 0; u < C::kSlice; u += 2) {
                    p0 = cfma(p0, g1[u], xs[u]);
                    p1 = cfma(p1, g1[u + 1], xs[u + 1]);
                }
                tpart[((k & 1) * C::kTeam + tw) * B + lane] = cadd(p0, p1);
                __syncwarp();
                if (lane == 0) mbar_arrive(pready + (k & 1));   // this warp's partial is in tpart
                // tail (off the critical path): G2_{k+1} x_{k-1} for the next step
                double2 c0 = make_double2(0.0, 0.0), c1 = make_double2(0.0, 0.0);
                if (k + 1 < nblk) {
#pragma unroll
                    for (int u = 0; u < C::kSlice; u += 2) {
                        c0 = cfma(c0, g2[u], xs[u]);
                        c1 = cfma(c1, g2[u + 1], xs[u + 1]);
                    }
                }
                carry = cadd(c0, c1);
                if (k + 1 < nblk) load_g(k + 1);   // next G slices: overlaps the barrier wait
                mbar_wait(yfull + yb, (uint32_t)((k / C::kYbuf) & 1));   // y_k
                mbar_wait(pready + (k & 1), (uint32_t)((k >> 1) & 1));   // all team partials
                if (trace && tw == 0 && lane == 0) trace[(int64_t)k * kTrace + 0] = gtime();
                double2 sum = tpart[((k & 1) * C::kTeam + 0) * B + lane];
#pragma unroll
                for (int w = 1; w < C::kTeam; w++) sum = cadd(sum, tpart[((k & 1) * C::kTeam + w) * B + lane]);
                xk = csub(ybuf[yb * B + lane], sum);
                __syncwarp();
                if (lane == 0) mbar_arrive(yempty + yb);
                if (tw == 0) {
                    // the ring slot of block k held block k-8: the publisher must have copied it
                    if (k >= C::kRing)
                        while (ld_acq_cta(sPub) < k - C::kRing + 1) {
                        }
                    ring[((int64_t)k * B + lane) & kRingMask] = xk;
                    __syncwarp();
                    if (lane == 0) {
                        st_rel_cta(sDone, k + 1);   // publisher, y warps
                        if (trace) trace[(int64_t)k * kTrace + 3] = gtime();
                    }
                }
            }
        } else if (chain && warp >= C::kYW0) {
            // ------------------------------------------------ y warps: y_k = D_k^{-1} (r_k - A3_k x_{k-3} - partials)
            // 4 threads per row (r = row, q = column class): D_k^{-1}[r, j], j = q mod 4,
            // j <= r, lives in registers; one named barrier per block (the residual vector).
            // two y teams of 2 warps take the even / odd blocks (each has two chain steps)
            const int yteam = (warp - C::kYW0) >> 1;           // 0: even blocks, 1: odd blocks
            const int yt = ((warp - C::kYW0) & 1) * 32 + lane;   // 0 .. 63
            constexpr int kYT = 64;
            constexpr int kQ = kYT / B;                     // 2 threads per row
            const int r = yt / kQ, q = yt % kQ;
            double2* sR = reinterpret_cast<double2*>(smem + C::kOffR) + yteam * B;   // [2][B]
            for (int k = yteam; k < nblk; k += 2) {
                const int s = k % C::kStages, yb = k % C::kYbuf, pk = k % C::kPbuf;
                unsigned char* st = smem + C::kChainStage * s;
                mbar_wait(full + s, (uint32_t)((k / C::kStages) & 1));
                const double2* sInv = reinterpret_cast<const double2*>(st + C::kOffInv);
                double2 dv[B / kQ];
#pragma unroll
                for (int t = 0; t < B / kQ; t++) {
                    const int j = q + kQ * t;
                    dv[t] = j <= r ? sInv[j * B - (j * (j - 1)) / 2 + (r - j)] : make_double2(0.0, 0.0);
                }
                const double2 rf = reinterpret_cast<const double2*>(st + C::kOffRfar)[r];
                // list A: source distance 3 (x_{k-3}, in the ring once the team has done it)
                if (k >= 3)
                    while (ld_acq_cta(sDone) < k - 2) {
                    }
                if (trace && yt == 0) trace[(int64_t)k * kTrace + 2] = gtime();
                double2 acc = near_part<B, kQ>(reinterpret_cast<const int32_t*>(st + C::kOffAloc),
                                               reinterpret_cast<const int32_t*>(st + C::kOffAcol),
                                               reinterpret_cast<const double2*>(st + C::kOffAval), ring, r, q);
#pragma unroll
                for (int o = 1; o < kQ; o <<= 1) {
                    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                }
                if (yt == 0) mbar_expect_tx(pbar + pk, (uint32_t)(B * 16));
                mbar_wait(pbar + pk, (uint32_t)((k / C::kPbuf) & 1));   // lieutenants' partials
                if (trace && yt == 0) trace[(int64_t)k * kTrace + 6] = gtime();
                if (q == 0) sR[r] = csub(csub(rf, acc), pbuf[pk * B + r]);
                bar_named(2 + yteam * 2, kYT);   // the team's residual vector is complete
                double2 y0 = make_double2(0.0, 0.0), y1 = make_double2(0.0, 0.0);
#pragma unroll
                for (int t = 0; t < B / kQ; t += 2) {
                    y0 = cfma(y0, dv[t], sR[q + kQ * t]);
                    y1 = cfma(y1, dv[t + 1], sR[q + kQ * (t + 1)]);
                }
                double2 yv = cadd(y0, y1);
#pragma unroll
                for (int o = 1; o < kQ; o <<= 1) {
                    yv.x += __shfl_xor_sync(0xffffffffu, yv.x, o);
                    yv.y += __shfl_xor_sync(0xffffffffu, yv.y, o);
                }
                if (q == 0) {
                    if (k >= C::kYbuf) mbar_wait(yempty + yb, (uint32_t)((k / C::kYbuf - 1) & 1));
                    ybuf[yb * B + r] = yv;
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(yfull + yb);   // one arrival per y warp of the team (its 16 rows)
                    mbar_arrive(empty + s);
                    if (trace && yt == 0) trace[(int64_t)k * kTrace + 1] = gtime();
                }
                bar_named(2 + yteam * 2, kYT);   // sR is reused by the team's next block
            }
        } else if (!chain) {
            // ------------------------------------------------ lieutenants: list B partial sums
            const int l = role - 1;   // rows l, l+3, l+6, ...
            const uint32_t peer_pbuf = mapa(smem_u32(pbuf), 0u);
            const uint32_t peer_pbar = mapa(smem_u32(pbar), 0u);
            int xseen = 0;   // x blocks < xseen have landed in the ring
            const int r = l + C::kLt * (tid / C::kTPRl), q = tid % C::kTPRl;
            const bool rowok = r < B;
            if (warp < C::kCompute / 32) {
                for (int k = 0; k < nblk; k++) {
                    const int s = k % nst;
                    unsigned char* st = smem + stsz * s;
                    mbar_wait(full + s, (uint32_t)((k / nst) & 1));
                    // list B of block k reads x of blocks <= k - 4: consume their arrivals in
                    // order (each xbar phase exactly once)
                    for (; xseen <= k - 4; xseen++) {
                        const int j = xseen % C::kRing;
                        if (tid == 0) mbar_expect_tx(xbar + j, (uint32_t)(B * 16));
                        mbar_wait(xbar + j, (uint32_t)((xseen / C::kRing) & 1));
                    }
                    if (trace && tid == 0 && l == 0) trace[(int64_t)k * kTrace + 7] = gtime();
                    double2 acc = make_double2(0.0, 0.0);
                    if (rowok)
                        acc = near_part<B, C::kTPRl>(reinterpret_cast<const int32_t*>(st + C::kOffBloc),
                                                     reinterpret_cast<const int32_t*>(st + C::kOffBcol),
                                                     reinterpret_cast<const double2*>(st + C::kOffBval), ring, r, q);
#pragma unroll
                    for (int o = 1; o < C::kTPRl; o <<= 1) {
                        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                    }
                    if (rowok && q == 0) {
                        const int pk = k % C::kPbuf;
                        st_async2(peer_pbuf + (uint32_t)((pk * B + r) * 16), acc, peer_pbar + (uint32_t)(pk * 8));
                    }
                    bar_named(2, C::kCompute);
                    if (tid == 0) mbar_arrive(empty + s);
                }
                for (; xseen < nblk; xseen++) {   // drain the remaining arrivals before leaving
                    const int j = xseen % C::kRing;
                    if (tid == 0) mbar_expect_tx(xbar + j, (uint32_t)(B * 16));
                    mbar_wait(xbar + j, (uint32_t)((xseen / C::kRing) & 1));
                }
            }
        }
        // no CTA of the cluster leaves while a peer may still access its shared memory
        __syncwarp();
        cluster_sync();
        return;
    }

    // ================================================================ helper CTAs
    if (warp >= C::kFarWarps) return;
    const int H = gridDim.x - C::kCluster;
    int64_t* sRowP = reinterpret_cast<int64_t*>(smem + C::kOffRowP);
    int32_t* sRowL = reinterpret_cast<int32_t*>(smem + C::kOffRowL);
    for (int k = blockIdx.x - C::kCluster; k < nblk; k += H) {
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
        bar_named(1, C::kCompute);
        if (tid == 0) {
            st_release(a.fflag + k, epoch);
            if (trace) trace[(int64_t)k * kTrace + 4] = gtime();
        }
    }
}

template <int B>
cudaLaunchConfig_t launch_config(int grid, cudaLaunchAttribute* attr) {
    using C = Cfg<B>;
    cudaLaunchConfig_t cfg = {};
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C::kCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(C::kNT);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

template <int B>
void prepare(DevBlockTri& T) {
    using C = Cfg<B>;
    auto fn = k_chain_trsv<B>;
    SSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem));
    int dev = 0, sms = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // clusters of 4 (chain + 3 lieutenants, then helpers), one CTA per SM; every cluster
    // must be resident at once (the CTAs spin on one another)
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = launch_config<B>((sms / C::kCluster) * C::kCluster, attr);
    int clusters = 0;
    SSB_CUDA(cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg));
    SSB_CHECK(clusters >= 2, SS_ERR_CUDA, "block trsv: fewer than two co-resident clusters");
    const int64_t want = C::kCluster * ((T.nblk + 2 * C::kCluster - 1) / C::kCluster);   // >= 1 helper cluster
    T.grid = (int)std::min<int64_t>(want, (int64_t)C::kCluster * clusters);
    T.nt = C::kNT;
}

template <int B>
void launch(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    auto fn = k_chain_trsv<B>;
    if (T.grid == 0) prepare<B>(T);
    T.epoch++;
    TriArgs a = T.args();
    uint32_t ep = T.epoch;
    double2* xw = T.operm ? T.xwork : x;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = launch_config<B>(T.grid, attr);
    cfg.stream = s;
    SSB_CUDA(cudaLaunchKernelEx(&cfg, fn, a, b, x, xw, ep, trace));
    SSB_LAUNCHED();
}

}  // namespace

size_t block_trsv_packed(int B) { return (size_t)B * (B + 1) / 2; }

void block_trsv_prepare(DevBlockTri& T) {
    SSB_CHECK(T.B == 32, SS_ERR_ARG, "block substitution supports B = 32");
    prepare<32>(T);
}

void block_trsv(DevBlockTri& T, const double2* b, double2* x, cudaStream_t s, unsigned long long* trace) {
    if (T.n == 0) return;
    SSB_CHECK(T.B == 32, SS_ERR_ARG, "block substitution supports B = 32");
    launch<32>(T, b, x, s, trace);
}

}  // namespace ssb
