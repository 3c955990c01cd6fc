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
// This file: block substitution whose dependency chain is one 32x32 complex mat-vec per
// block on the chain CTA.  Rows are cut into blocks of B = 32 consecutive rows; in the
// kernel's index space (U reversed at setup, i' = n-1-i, so both factors are lower
// triangular)
//     x_k = D_k^{-1} ( b_k - sum_{j<k} T_kj x_j )
//         = y_k - sum_l q_{l,k} - G1_k x_{k-1} - G2_k x_{k-2}        (kDense = 2),
//     y_k = D_k^{-1} ( b_k - far_k ),  Gd_k = D_k^{-1} T_{k,k-d} (dense, precomputed),
//     q_{l,k} = D_k^{-1}[:, rows of l] (list B of lieutenant l applied to x),
// where "far" are the entries with source distance d >= Q_k and list B those with
// kDense < d < Q_k (setup.cpp::build_block_tri).  Only G1_k x_{k-1} is on the chain:
//   * chain CTA (cluster rank 0): three chain teams of 4 warps rotate over the blocks;
//     the team of block k prepares G1_k (registers), the carry G2_k x_{k-2} and y_k while
//     the other teams compute x_{k-2}, x_{k-1}; then x_{k-1}
//     (ring + mbarrier) -> G1_k x_{k-1} -> partials (mbarrier) -> x_k into the ring and,
//     by st.async, into the lieutenants' rings;
//   * lieutenants (cluster ranks 1..7, DSMEM): list B of rows l, l+7, ..., the early
//     part (d >= 4) once x_{k-4} has landed, the late part (d = 3) once x_{k-3} has, times
//     their columns of D_k^{-1}, st.async'd back to the chain CTA;
//   * helpers (the other SMs): the far entries streamed in 32-entry chunks as the
//     published frontier covers them; y_k published with a gpu-scope release flag;
//   * producer warps: TMA bulk copies (cp.async.bulk + mbarrier) of G1|G2 and y_k
//     (chain CTA) or list B and D_k^{-1} (lieutenants), stages ahead;
//   * publisher warp: copies finished x blocks from the ring to global memory (and
//     through the iLUTP column permutation to the output, x = Pi y) and advances the
//     frontier word (epoch << 32 | blocks done) with a gpu-scope release.
// One CTA per SM, clusters of 8; the grid never exceeds the co-resident cluster count, so
// the spin waits cannot deadlock.  Every reduction has a fixed order: the result is
// deterministic for a given layout.  DESIGN.md sec. 5 has the measurements.

#include "problem.h"

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
// arrive on a peer CTA's mbarrier (shared::cluster address), adding bytes to its expected
// transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx_remote(uint32_t addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes)
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
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {   // non-blocking
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
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

constexpr int kTrace = SS_TRACE_STAMPS;   // stamps per block when tracing (include/ss_b200.h)
// STAMP: the ss_debug_trace_trsv stamps (%globaltimer).  Built with -DSSB_TEAM_PROF instead,
// TPROF stamps clock64() at sub-steps of the chain team's warp 0 (scripts/trace_trsv.py --team).
#if defined(SSB_TEAM_PROF)
#define STAMP(k, i) ((void)0)
#define TPROF(k, i) \
    if (trace && tw == 0 && lane == 0) trace[(int64_t)(k) * kTrace + (i)] = clock64()
#define LPROF(k, i) ((void)0)
#elif defined(SSB_LT_PROF)   // the same for lieutenant 0's team thread 0
#define STAMP(k, i) ((void)0)
#define TPROF(k, i) ((void)0)
#define LPROF(k, i) \
    if (trace && tt == 0 && l == 0) trace[(int64_t)(k) * kTrace + (i)] = clock64()
#else
#define STAMP(k, i) (trace[(int64_t)(k) * kTrace + (i)] = gtime())
#define TPROF(k, i) ((void)0)
#define LPROF(k, i) ((void)0)
#endif
#ifndef SSB_LT_DINV_LDG
#define SSB_LT_DINV_LDG 0   // lieutenants read their columns of D_k^{-1} from global memory (L2), not staged
#endif
constexpr bool kLtDinvLdg = SSB_LT_DINV_LDG != 0;
#ifndef SSB_G3_WARPS
#define SSB_G3_WARPS 0   // with kDense = 3: G3_k x_{k-3} by the chain CTA's two idle warps (3, 4)
#endif
constexpr bool kG3Warps = SSB_G3_WARPS != 0;
#ifndef SSB_LT_GATE
#define SSB_LT_GATE 0   // lieutenants: the early part of block k waits for block k-1's late part (1) or its q (2)
#endif
constexpr int kLtGate = SSB_LT_GATE;
#ifndef SSB_LT_G3
#define SSB_LT_G3 0   // with kDense = 3: G3_k x_{k-3} by the lieutenants (columns l, l+7, ... of G3_k from L2), not the chain
#endif
constexpr bool kLtG3 = SSB_LT_G3 != 0;
#ifndef SSB_G3_LDG
#define SSB_G3_LDG 0   // with kDense = 3 and row-owning teams: G3_k x_{k-3} by four extra chain-CTA warps, G3 from L2
#endif
constexpr bool kG3Ldg = SSB_G3_LDG != 0;
constexpr int kChainDense = (kLtG3 || kG3Ldg) ? 2 : kDense;   // dense blocks the chain teams apply (G ring stage)
#ifndef SSB_TEST_NO_OPERAND_ZEROING
#define SSB_TEST_NO_OPERAND_ZEROING 0   // (test builds only: the pre-fix lieutenants, to show the stale-smem test fails on them)
#endif
constexpr bool kZeroOperands = SSB_TEST_NO_OPERAND_ZEROING == 0;
#ifndef SSB_ROWWARPS
#define SSB_ROWWARPS 0   // chain teams: warp w owns ROWS 8w .. 8w+7 (4 lanes per row, shuffle reduction) instead of columns
#endif
constexpr bool kRowWarps = SSB_ROWWARPS != 0;
#ifndef SSB_PUSH_SPLIT
#define SSB_PUSH_SPLIT 0   // lieutenants 0 .. SSB_PUSH_SPLIT-1 get x_k from team warp 0 (the rest from warp 1)
#endif
constexpr int kProducerSleep = 32;   // back-off of the producer polling a helper flag (ns)
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
    static constexpr int kLt = kLieutenants;
    static constexpr int kCluster = 1 + kLt;          // chain + lieutenants
    static constexpr int kCompute = 256;              // compute threads (8 warps)
    static constexpr int kNT = kG3Ldg ? 608 : 544;    // chain CTA: 17 warps (roles below; + warps 17, 18 with kG3Ldg)
    // chain CTA warp roles (warp w runs on SMSP w mod 4): producer 0, publisher 1, G producer
    // 2, chain teams 0, 1, 2 = warps 5 .. 8, 9 .. 12, 13 .. 16 (blocks k = team mod 3), one
    // warp of each team per SMSP (warps 3, 4 idle)
    static constexpr int kTeam = 4, kTeams = 3, kTeamW0 = 5;
    static constexpr int kWProducerChain = 0, kWPublisher = 1, kWGProducer = 2;
    static constexpr int kSlice = B / kTeam;          // columns of G per team warp
    static constexpr int kFarWarps = 16;              // helper warps streaming the far part
    static constexpr int kRPW = B / kFarWarps;        // far rows per helper warp
    static constexpr int kGrp = kRPW < 4 ? kRPW : 4;
    static constexpr int kGStages = 3;                // G1 | G2 | G3 ring (chain teams, a block ahead)
    static constexpr int kSStages = 16;               // y_k ring (the helpers' D_k^{-1} (b_k - far))
    static constexpr int kRing = 16;                  // chain CTA: x of the last 16 blocks
    static constexpr int kRingLt = 32;                // lieutenants: x of the last 32 blocks (Q <= 32)
    static constexpr int kPbuf = 4;                   // lieutenant partial-sum slots
    static constexpr int kPK = B * (B + 1) / 2;
    static constexpr int kCapB = near_cap_b(B);
    static constexpr int kNloc = near_nloc(B);        // per list: row starts | late-part starts
    static constexpr int kLate = B + 4;               // offset of the late-part starts

    static constexpr int kLtTeams = 4, kLtTeamT = 128;   // lieutenants: 4 teams of 4 warps (blocks k mod 4)
    static constexpr int kWProducerLt = kNT / 32 - 1;
    static constexpr int kTPRl = 16;                  // lieutenants: threads per row (early part)
    static constexpr int kTPRlate = 4;                //              and of them for the late part
    // chain CTA: a G ring (G1_k | G2_k | G3_k) and an S ring (y_k), filled independently (G is
    // static, y_k waits for the helpers)
    static constexpr size_t kGStage = (size_t)kChainDense * B * B * 16;
    static constexpr size_t kOffSR = kGStage * kGStages;
    static constexpr size_t kSStage = (size_t)B * 16;
    static constexpr size_t kChainRegion = kOffSR + kSStage * kSStages;
    // lieutenant stage: list B columns | values | row pointers
    static constexpr size_t kOffBcol = 0;
    static constexpr size_t kOffBval = kOffBcol + (size_t)kCapB * 4;
    static constexpr size_t kOffBloc = kOffBval + (size_t)kCapB * 16;
    static constexpr int kRowsL = lt_rows(B);         // rows of a block per lieutenant
    static constexpr size_t kOffBinv = kOffBloc + (size_t)kNloc * 4;   // D_k^{-1} (packed; shared in L2 by all)
    static constexpr size_t kLtStage = kOffBinv + (kLtDinvLdg ? 0 : (size_t)kPK * 16);
    static constexpr int kLtStages = kG3Warps ? 5 : 6;   // (the G3-warps variant needs 3 KB more)
    static constexpr size_t kOffLtRing = kLtStage * kLtStages;   // lieutenants' x ring
    static constexpr size_t kOffLtP = kOffLtRing + (size_t)kRingLt * B * 16;   // [kLtTeams][B] row partials
    static constexpr size_t kLtRegion = kOffLtP + (size_t)kLtTeams * B * 16;
    static constexpr size_t kStageRegion = kChainRegion > kLtRegion ? kChainRegion : kLtRegion;
    static constexpr size_t kOffRing = kStageRegion;
    static constexpr size_t kOffR = kOffRing + (size_t)kRing * B * 16;          // helpers: b_k - far
    static constexpr size_t kOffPbuf = kOffR + (size_t)B * 16;
    static constexpr size_t kOffTpart = kOffPbuf + (size_t)kPbuf * kLt * B * 16;   // [4][kTeam][B] partials
    static constexpr size_t kOffXw = kOffTpart + (size_t)4 * kTeam * B * 16;   // [kTeams kTeam][B] own x_k
    static constexpr size_t kOffRowP = kOffXw + (size_t)kTeams * kTeam * B * 16;
    static constexpr size_t kOffRowL = kOffRowP + (size_t)B * 8;
    static constexpr size_t kOffG3v = kOffRowL + (size_t)B * 4;                 // [4][B] G3_k x_{k-3}
    static constexpr size_t kOffG3p = kOffG3v + (kG3Warps ? (size_t)4 * B * 16 : 0);   // [2][B] its halves
    static constexpr size_t kOffBar = kOffG3p + (kG3Warps ? (size_t)2 * B * 16 : 0);
    // mbarriers: full/empty per S stage (lieutenants: per list B stage), full/empty per G
    // stage, xbar (lieutenant: x block landed), pbar (chain: partials landed), xfull (ring slot
    // holds x_k), pready (team partials), rfull (y_k staged), then int counters
    static constexpr int kNS = kSStages > kLtStages ? kSStages : kLtStages;
    static constexpr size_t kOffFull = kOffBar;
    static constexpr size_t kOffEmpty = kOffFull + 8 * kNS;
    static constexpr size_t kOffGfull = kOffEmpty + 8 * kNS;
    static constexpr size_t kOffGempty = kOffGfull + 8 * kGStages;
    static constexpr size_t kOffXbar = kOffGempty + 8 * kGStages;
    static constexpr size_t kOffPbar = kOffXbar + 8 * kRingLt;
    static constexpr size_t kOffXfull = kOffPbar + 8 * kPbuf;
    static constexpr size_t kOffPready = kOffXfull + 8 * kRing;
    static constexpr size_t kOffRfull = kOffPready + 8 * 4;
    static constexpr size_t kOffG3full = kOffRfull + 8 * kSStages;             // [4] G3 vector of block k ready
    static constexpr size_t kOffInts = kOffG3full + (kG3Warps ? 8 * 4 : 0);
    static constexpr size_t kOffLbar = kOffInts + 32;   // [4] (lieutenants) late part of block k done
    // kG3Ldg: partials of the four G3 warps, kG3Slots blocks deep.  Row-owning teams leave tpart and
    // pready unused (4 slots); column-owning teams leave the x_{k-3} copies (kOffXw) unused (3 slots)
    static constexpr int kG3Slots = kRowWarps ? 4 : 3;
    static constexpr size_t kOffG3Lp = kRowWarps ? kOffTpart : kOffXw;
    static constexpr size_t kOffG3Lfull = kRowWarps ? kOffPready : kOffLbar;   // (lbar: lieutenants only)
    static constexpr size_t kSmem = kOffInts + 64;
    static_assert((size_t)kG3Slots * 4 * B * 16 <= (kRowWarps ? (size_t)4 * kTeam * B * 16 : (size_t)kTeams * kTeam * B * 16), "G3 partial slots");
    static_assert(B == 32 && (kDense == 2 || kDense == 3), "the chain teams hold one row per lane, G1 .. G_kDense");
    static_assert(!kG3Warps || kDense == 3, "the G3 warps need G3 (kDense = 3)");
    static_assert(!kLtG3 || (kDense == 3 && !kG3Warps), "lieutenant G3 needs G3 (kDense = 3)");
    static_assert(!kG3Ldg || (kDense == 3 && !kG3Warps && !kLtG3), "G3-from-L2 warps: kDense = 3");
    static constexpr int kWG3 = 3;                    // G3 warps: 3, 4 (idle otherwise)
    static_assert(kCompute % B == 0 && B % kFarWarps == 0 && kRPW % kGrp == 0 && kFarWarps * 32 <= kNT, "layout");
    static constexpr int kHelperT = kFarWarps * 32;   // helper threads
    static constexpr int kYP = kHelperT / B;          // helper D^{-1} product: threads per row
    static_assert(kTeamW0 + kTeams * kTeam == 17 && 17 <= kNT / 32 && kCompute / 32 + 1 <= kNT / 32, "warp roles");
    static_assert(kTPRl * ((B + kLt - 1) / kLt) <= kLtTeamT && kLtTeams * kLtTeamT <= 32 * kWProducerLt &&
                      kLtTeams <= kLtStages,
                  "lieutenant rows / teams");
    static_assert(kSStage % 16 == 0 && kLtStage % 16 == 0 && kOffSR % 16 == 0 &&
                      kOffBval % 16 == 0 && kOffBloc % 16 == 0 && kOffBinv % 16 == 0 && kOffLtRing % 16 == 0,
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

// Entries [lo, hi) of one row of a staged list B, interleaved over the TPR threads of the
// row (thread q takes lo+q, lo+q+TPR, ...: the row's threads read consecutive entries),
// x from the lieutenant's ring.  Returns this thread's share (reduced by the caller).
template <int B, int TPR, int kRingBlocks>
__device__ __forceinline__ double2 near_range(const int32_t* col, const double2* val, const double2* ring, int lo,
                                              int hi, int q, double2 acc) {
    constexpr int kRingMask = kRingBlocks * B - 1;
    double2 acc2 = make_double2(0.0, 0.0);
    int e = lo + q;
    for (; e + TPR < hi; e += 2 * TPR) {
        const int c0 = col[e], c1 = col[e + TPR];
        const double2 v0 = val[e], v1 = val[e + TPR];
        acc = cfma(acc, v0, ring[c0 & kRingMask]);
        acc2 = cfma(acc2, v1, ring[c1 & kRingMask]);
    }
    if (e < hi) acc = cfma(acc, val[e], ring[col[e] & kRingMask]);
    return cadd(acc, acc2);
}

// Entries [lo, hi) of one row summed by ONE thread, 4 at a time with predicated
// (branch-free) loads, x from the ring.
template <int B, int kRingBlocks>
__device__ __forceinline__ double2 row_sum_1t(const int32_t* col, const double2* val, const double2* ring, int lo,
                                              int hi, double2 acc) {
    constexpr int kRingMask = kRingBlocks * B - 1;
    double2 acc2 = make_double2(0.0, 0.0);
    for (int e = lo; e < hi; e += 4) {
        int c[4];
        double2 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const bool ok = e + u < hi;
            const int ee = ok ? e + u : lo;
            c[u] = col[ee];
            v[u] = val[ee];
            v[u].x = ok ? v[u].x : 0.0;
            v[u].y = ok ? v[u].y : 0.0;
        }
        double2 xr[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {   // absent entries: zero the operand too (0 * NaN = NaN)
            xr[u] = ring[c[u] & kRingMask];
            xr[u].x = e + u < hi ? xr[u].x : 0.0;
            xr[u].y = e + u < hi ? xr[u].y : 0.0;
        }
        acc = cfma(acc, v[0], xr[0]);
        acc2 = cfma(acc2, v[1], xr[1]);
        acc = cfma(acc, v[2], xr[2]);
        acc2 = cfma(acc2, v[3], xr[3]);
    }
    return cadd(acc, acc2);
}

// Stage list g (TMA): entries [b0, b1) (columns, values; a multiple of 4) and row pointers,
// `extra` more bytes expected on the same barrier (one arrival).
__device__ __forceinline__ void stage_near(unsigned char* col_dst, unsigned char* val_dst, unsigned char* loc_dst,
                                           int64_t b0, int64_t b1, const int32_t* col, const double2* val,
                                           const int32_t* loc, int g, int nloc, uint64_t* bar, uint32_t extra = 0) {
    const uint32_t cnt = (uint32_t)(b1 - b0);
    mbar_expect_tx(bar, cnt * 20 + (uint32_t)nloc * 4 + extra);
    if (cnt) {
        bulk_g2s(col_dst, col + b0, cnt * 4, bar);
        bulk_g2s(val_dst, val + b0, cnt * 16, bar);
    }
    bulk_g2s(loc_dst, loc + (int64_t)g * nloc, (uint32_t)nloc * 4, bar);
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
    uint64_t* gfull = reinterpret_cast<uint64_t*>(smem + C::kOffGfull);
    uint64_t* gempty = reinterpret_cast<uint64_t*>(smem + C::kOffGempty);
    uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + C::kOffXbar);
    uint64_t* pbar = reinterpret_cast<uint64_t*>(smem + C::kOffPbar);
    uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + C::kOffXfull);
    uint64_t* rfull = reinterpret_cast<uint64_t*>(smem + C::kOffRfull);   // chain: r_k staged
    double2* tpart = reinterpret_cast<double2*>(smem + C::kOffTpart);
    uint64_t* pready = reinterpret_cast<uint64_t*>(smem + C::kOffPready);
    int* sF = reinterpret_cast<int*>(smem + C::kOffInts);      // helpers: frontier view
    int* sLock = sF + 1;
    int* sPub = sF + 2;                                           // chain: blocks published
    double2* ring = reinterpret_cast<double2*>(smem + C::kOffRing);
    double2* pbuf = reinterpret_cast<double2*>(smem + C::kOffPbuf);
    constexpr int kRingMask = C::kRing * B - 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = a.n;
    const int nblk = (int)a.nblk;
    const bool rev = a.rev != 0;
    auto phys = [&](int64_t i) -> int64_t { return rev ? n - 1 - i : i; };
    const int role = blockIdx.x < C::kCluster ? (int)blockIdx.x : -1;   // 0 chain, 1.. lieutenants
    const bool chain = role == 0;

    if (tid == 0) {
        for (int s = 0; s < C::kNS; s++) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, chain ? C::kTeam : 1);   // chain CTA: the warps of the block's team
        }
        for (int s = 0; s < C::kSStages; s++) mbar_init(rfull + s, 1);
        for (int s = 0; s < C::kGStages; s++) {
            mbar_init(gfull + s, 1);
            mbar_init(gempty + s, C::kTeam + (kG3Warps ? 2 : 0));   // the team of block k (+ the G3 warps)
        }
        for (int j = 0; j < C::kRingLt; j++) mbar_init(xbar + j, 1);
        for (int j = 0; j < C::kPbuf; j++) mbar_init(pbar + j, 1);
        for (int j = 0; j < C::kRing; j++) mbar_init(xfull + j, 32);   // the 32 lanes of the storing warp
        for (int j = 0; j < 4; j++) mbar_init(pready + j, C::kTeam * 32);   // every lane of a team
        if (!(kG3Ldg && !kRowWarps && chain))   // (the chain CTA of that variant keeps its G3 barriers there)
            for (int j = 0; j < 4; j++) mbar_init(reinterpret_cast<uint64_t*>(smem + C::kOffLbar) + j, 1);
        if (kG3Warps)
            for (int j = 0; j < 4; j++) mbar_init(reinterpret_cast<uint64_t*>(smem + C::kOffG3full) + j, 32);
        if (kG3Ldg && !kRowWarps && chain)   // every lane of the four G3 warps (re-initialises the chain CTA's unused lbar)
            for (int j = 0; j < C::kG3Slots; j++) mbar_init(reinterpret_cast<uint64_t*>(smem + C::kOffG3Lfull) + j, 128);
        *sF = 0;
        *sLock = 0;
        *sPub = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();   // barriers and counters of every CTA initialised before any DSMEM access

    if (role >= 0) {
        const int nst = chain ? C::kSStages : C::kLtStages;
        const size_t stsz = chain ? C::kSStage : C::kLtStage;
        unsigned char* const sbase = smem + (chain ? C::kOffSR : 0);
        const int wprod = chain ? C::kWProducerChain : C::kWProducerLt;
        if (warp == wprod) {
            // ------------------------------------------------ producer: TMA staging of the S ring
            // (chain: y_k once its helper flag is set, the 32 lanes polling 32 flags per round
            // trip; lieutenants: list B and D_k^{-1})
            if (chain) {
                int k = 0;
                while (k < nblk) {
                    const int kk = k + lane;
                    const bool ready = kk < nblk && ld_acquire(a.fflag + kk) == epoch;
                    const unsigned m = __ballot_sync(0xffffffffu, ready);
                    const int nready = m == 0xffffffffu ? 32 : __ffs(~m) - 1;   // consecutive from k
                    if (nready == 0) {
                        __nanosleep(kProducerSleep);
                        continue;
                    }
                    if (lane == 0) {
                        fence_proxy_async();   // y (generic-proxy stores of the helpers) -> TMA reads
                        for (int j = k; j < k + nready && j < nblk; j++) {
                            const int s = j % nst;
                            if (j >= nst) mbar_wait(empty + s, (uint32_t)((j / nst - 1) & 1));
                            if (trace) STAMP(j, 5);
                            mbar_expect_tx(rfull + s, (uint32_t)(B * 16));
                            bulk_g2s(sbase + stsz * s, a.yfar + (int64_t)j * B, B * 16, rfull + s);
                        }
                    }
                    __syncwarp();
                    k += nready;
                }
            } else if (lane == 0) {
                // lieutenants: the list bounds of block k+1 are loaded while block k's slot drains
                int64_t nb0 = 0, nb1 = 0;
                if (nblk > 0) {
                    nb0 = __ldg(a.nbpB + (role - 1));
                    nb1 = __ldg(a.nbpB + role);
                }
                for (int k = 0; k < nblk; k++) {
                    const int s = k % nst;
                    const int64_t b0 = nb0, b1 = nb1;
                    if (k + 1 < nblk) {
                        const int gn = (k + 1) * C::kLt + (role - 1);
                        nb0 = __ldg(a.nbpB + gn);
                        nb1 = __ldg(a.nbpB + gn + 1);
                    }
                    if (k >= nst) mbar_wait(empty + s, (uint32_t)((k / nst - 1) & 1));
                    unsigned char* st = sbase + stsz * s;
                    const int g = k * C::kLt + (role - 1);   // this lieutenant's rows of block k
                    stage_near(st + C::kOffBcol, st + C::kOffBval, st + C::kOffBloc, b0, b1, a.ncolB, a.nvalB,
                               a.nlocB, g, C::kNloc, full + s, kLtDinvLdg ? 0u : (uint32_t)(C::kPK * 16));
                    // the whole packed D_k^{-1}: the helper and all seven lieutenants read the same
                    // 8.4 KB, so DRAM sees it once (L2)
                    if (!kLtDinvLdg) bulk_g2s(st + C::kOffBinv, a.dinv + (int64_t)k * C::kPK, C::kPK * 16, full + s);
                }
            }
        } else if (chain && warp == C::kWGProducer) {
            // ------------------------------------------------ G producer: the teams' G ring
            if (lane == 0) {
                for (int k = 0; k < nblk; k++) {
                    const int s = k % C::kGStages;
                    if (k >= C::kGStages) mbar_wait(gempty + s, (uint32_t)((k / C::kGStages - 1) & 1));
                    mbar_expect_tx(gfull + s, (uint32_t)C::kGStage);
                    bulk_g2s(smem + C::kGStage * s, a.G + (int64_t)k * kDense * B * B, (uint32_t)C::kGStage,
                             gfull + s);
                }
            }
        } else if (chain && warp == C::kWPublisher) {
            // ------------------------------------------------ publisher: x blocks from the ring to
            // global memory (and through the iLUTP column permutation to the output), then the
            // gpu-scope frontier word
            // Blocks already complete are copied in one batch (up to 8) before the frontier
            // word is released; the output permutation of the next block is prefetched.
            auto perm_of = [&](int j) -> int64_t {
                const int64_t i = (int64_t)j * B + lane;
                return (a.operm && j < nblk && i < n) ? __ldg(a.operm + phys(i)) : 0;
            };
            int64_t op = perm_of(0);
            for (int j = 0; j < nblk;) {
                mbar_wait(xfull + j % C::kRing, (uint32_t)((j / C::kRing) & 1));
                const int j_end = min(nblk, j + 8);
                do {
                    const int64_t i = (int64_t)j * B + lane;
                    const double2 v = ring[i & kRingMask];
                    const int64_t opj = op;
                    op = perm_of(j + 1);
                    if (i < n) {
                        x[phys(i)] = v;
                        if (a.operm) out[opj] = v;
                    }
                    j++;
                } while (j < j_end && mbar_test(xfull + j % C::kRing, (uint32_t)((j / C::kRing) & 1)));
                __syncwarp();
                if (lane == 0) {
                    st_release64(a.xfront, ((unsigned long long)epoch << 32) | (unsigned)j);
                    st_rel_cta(sPub, j);
                }
            }
        } else if (chain && warp >= C::kTeamW0 && warp < C::kTeamW0 + C::kTeams * C::kTeam) {
            // ------------------------------------------------ chain teams 0, 1, 2 (blocks k = team
            // mod 3), 4 warps each:
            //     x_k = y_k - sum_w [ G1_k[:, w] x_{k-1}[w] + G2_k[:, w] x_{k-2}[w] + G3_k[:, w] x_{k-3}[w] ]
            // Warp w of a team owns 8 columns (slice w).  While the other teams compute x_{k-2},
            // x_{k-1}, the team of block k loads G1_k (registers) and forms the carry G2_k x_{k-2}
            // (the ring) + G3_k x_{k-3} (its own); then only x_{k-1} (from the ring, xfull) ->
            // G1_k x_{k-1} -> the
            // partials (pready, which also carries y_k) -> x_k is on the chain.  Every warp
            // reduces the partials itself; warp 0 stores x_k to the ring and releases xfull,
            // warp 1 pushes x_k to the lieutenants.
            const int team = (warp - C::kTeamW0) / C::kTeam;   // blocks k = team mod kTeams
            const int tw = (warp - C::kTeamW0) % C::kTeam;
            const int j0 = tw * C::kSlice;
            double2* xw = reinterpret_cast<double2*>(smem + C::kOffXw) + (warp - C::kTeamW0) * B;   // my x_{k-3}
            uint32_t peer_ring[C::kLt], peer_xbar[C::kLt];   // warp 1: the lieutenants' rings
#pragma unroll
            for (int l = 0; l < C::kLt; l++) {
                peer_ring[l] = mapa(smem_u32(smem + C::kOffLtRing), (uint32_t)(l + 1));
                peer_xbar[l] = mapa(smem_u32(xbar), (uint32_t)(l + 1));
            }
            if constexpr (kRowWarps) {
                // ---- row-owning variant: warp tw owns rows 8 tw .. 8 tw + 7, lane = (rr = lane & 7,
                // g = lane >> 3) takes columns g, g + 4, ..., g + 28 of its row; the four lanes of a
                // row reduce by shuffles (no partials in shared memory, no pready hand-off), lane
                // group g also adds q_g and q_{g+4} and pushes x_k to those lieutenants.
                static_assert(!kRowWarps || (kChainDense == 2 && B == 32 && C::kTeam == 4 && C::kLt <= 8), "row-owning teams");
                const int rr = lane & 7, g = lane >> 3, r = tw * 8 + rr;
                const int l0 = g, l1 = g + 4;   // this lane group's lieutenants (l1 only if < kLt)
                const uint32_t pr0 = mapa(smem_u32(smem + C::kOffLtRing), (uint32_t)(l0 + 1));
                const uint32_t pb0 = mapa(smem_u32(xbar), (uint32_t)(l0 + 1));
                const uint32_t pr1 = mapa(smem_u32(smem + C::kOffLtRing), (uint32_t)((l1 < C::kLt ? l1 : l0) + 1));
                const uint32_t pb1 = mapa(smem_u32(xbar), (uint32_t)((l1 < C::kLt ? l1 : l0) + 1));
                for (int k = team; k < nblk; k += C::kTeams) {
                    TPROF(k, 0);
                    if (k >= C::kRing)   // ring slot of block k held block k-kRing: published?
                        while (ld_acq_cta(sPub) < k - C::kRing + 1) {
                        }
                    TPROF(k, 8);
                    double2 g1[8];
                    double2 carry = make_double2(0.0, 0.0), carry2 = carry;
                    {
                        const int s = k % C::kGStages;
                        mbar_wait(gfull + s, (uint32_t)((k / C::kGStages) & 1));
                        TPROF(k, 9);
                        const double2* G = reinterpret_cast<const double2*>(smem + C::kGStage * s);
#pragma unroll
                        for (int u = 0; u < 8; u++) g1[u] = G[(g + 4 * u) * B + r];
                        TPROF(k, 10);
                        if (k >= 2) {
                            mbar_wait(xfull + (k - 2) % C::kRing, (uint32_t)(((k - 2) / C::kRing) & 1));   // x_{k-2}
                            TPROF(k, 12);
                            const double2* x2 = ring + (((int64_t)(k - 2) * B) & kRingMask);
#pragma unroll
                            for (int u = 0; u < 8; u += 2) {
                                carry = cfma(carry, G[B * B + (g + 4 * u) * B + r], x2[g + 4 * u]);
                                carry2 = cfma(carry2, G[B * B + (g + 4 * u + 4) * B + r], x2[g + 4 * u + 4]);
                            }
                        }
                        carry = cadd(carry, carry2);
                        if (kG3Ldg) {   // + G3_k[r, 8 g .. 8 g + 7] x_{k-3}[...] from G3 warp g (tpart region)
                            mbar_wait(reinterpret_cast<uint64_t*>(smem + C::kOffG3Lfull) + k % C::kG3Slots,
                                      (uint32_t)((k / C::kG3Slots) & 1));
                            carry = cadd(carry, reinterpret_cast<const double2*>(smem + C::kOffG3Lp)[((k % C::kG3Slots) * 4 + g) * B + r]);
                        }
                        TPROF(k, 13);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(gempty + s);
                    }
                    double2 yk;
                    {
                        const int s = k % C::kSStages;
                        mbar_wait(rfull + s, (uint32_t)((k / C::kSStages) & 1));
                        yk = reinterpret_cast<const double2*>(smem + C::kOffSR + C::kSStage * s)[r];
                        __syncwarp();
                        if (lane == 0) {
                            mbar_arrive(empty + s);
                            if (tw == 0) mbar_expect_tx(pbar + k % C::kPbuf, (uint32_t)(C::kLt * B * 16));   // the q_l of block k
                        }
                    }
                    TPROF(k, 1);
                    if (trace && tw == 0 && lane == 0) STAMP(k, 10);
                    // ---- the chain
                    double2 p0 = carry, p1 = make_double2(0.0, 0.0);
                    double2 p2 = make_double2(0.0, 0.0), p3 = make_double2(0.0, 0.0);
                    if (k >= 1) {
                        mbar_wait(xfull + (k - 1) % C::kRing, (uint32_t)(((k - 1) / C::kRing) & 1));   // x_{k-1}
                        const double2* xr = ring + (((int64_t)(k - 1) * B) & kRingMask);
                        TPROF(k, 2);
                        if (trace && tw == 0 && lane == 0) STAMP(k, 13);
#pragma unroll
                        for (int u = 0; u < 8; u += 4) {
                            p0 = cfma(p0, g1[u], xr[g + 4 * u]);
                            p1 = cfma(p1, g1[u + 1], xr[g + 4 * u + 4]);
                            p2 = cfma(p2, g1[u + 2], xr[g + 4 * u + 8]);
                            p3 = cfma(p3, g1[u + 3], xr[g + 4 * u + 12]);
                        }
                    }
                    double2 p = cadd(cadd(p0, p1), cadd(p2, p3));
                    TPROF(k, 3);
                    mbar_wait(pbar + k % C::kPbuf, (uint32_t)((k / C::kPbuf) & 1));   // the lieutenants' q_l
                    if (trace && tw == 0 && lane == 0) STAMP(k, 6);
                    p = cadd(p, pbuf[((k % C::kPbuf) * C::kLt + l0) * B + r]);
                    if (l1 < C::kLt) p = cadd(p, pbuf[((k % C::kPbuf) * C::kLt + l1) * B + r]);
                    TPROF(k, 4);
                    p.x += __shfl_xor_sync(0xffffffffu, p.x, 8);
                    p.y += __shfl_xor_sync(0xffffffffu, p.y, 8);
                    p.x += __shfl_xor_sync(0xffffffffu, p.x, 16);
                    p.y += __shfl_xor_sync(0xffffffffu, p.y, 16);
                    const double2 xk = csub(yk, p);
                    if (trace && tw == 0 && lane == 0) STAMP(k, 0);
                    TPROF(k, 5);
                    if (g == 0) {
                        ring[((int64_t)k * B + r) & kRingMask] = xk;
                        mbar_arrive(xfull + k % C::kRing);   // 8 lanes of each of the 4 warps: 32 arrivals
                    }
                    TPROF(k, 6);
                    if (trace && tw == 0 && lane == 0) STAMP(k, 3);
                    {
                        const uint32_t off = (uint32_t)((((int64_t)k * B + r) & (C::kRingLt * B - 1)) * 16);
                        const uint32_t bar = (uint32_t)((k % C::kRingLt) * 8);
                        if (tw == 0 && rr == 0) {   // the single arrival of each lieutenant's phase
                            mbar_arrive_expect_tx_remote(pb0 + bar, B * 16);
                            if (l1 < C::kLt) mbar_arrive_expect_tx_remote(pb1 + bar, B * 16);
                        }
                        st_async2(pr0 + off, xk, pb0 + bar);
                        if (l1 < C::kLt) st_async2(pr1 + off, xk, pb1 + bar);
                    }
                    if (trace && tw == 1 && lane == 0) STAMP(k, 8);
                    TPROF(k, 7);
                }
            } else {
            for (int k = team; k < nblk; k += C::kTeams) {
                const int pq = k & 3;
                TPROF(k, 0);
                // ---- off the chain (the other team is computing x_{k-1})
                if (tw == 0 && k >= C::kRing)   // ring slot of block k held block k-8: published?
                    while (ld_acq_cta(sPub) < k - C::kRing + 1) {
                    }
                TPROF(k, 8);
                double2 g1[C::kSlice];
                double2 carry = make_double2(0.0, 0.0);   // (G2_k x_{k-2} + G3_k x_{k-3})[lane, slice]
                {
                    const int s = k % C::kGStages;
                    mbar_wait(gfull + s, (uint32_t)((k / C::kGStages) & 1));
                    TPROF(k, 9);
                    const double2* G = reinterpret_cast<const double2*>(smem + C::kGStage * s);
#pragma unroll
                    for (int u = 0; u < C::kSlice; u++) g1[u] = G[(j0 + u) * B + lane];
                    TPROF(k, 10);
                    double2 c1 = make_double2(0.0, 0.0);
                    if constexpr (kG3Warps) {
                        // G3_k x_{k-3} from the G3 warps: warp 0 of the team adds it (once)
                        if (tw == 0 && k >= 3) {
                            mbar_wait(reinterpret_cast<uint64_t*>(smem + C::kOffG3full) + ((k - 3) & 3),
                                      (uint32_t)(((k - 3) >> 2) & 1));
                            c1 = reinterpret_cast<const double2*>(smem + C::kOffG3v)[((k - 3) & 3) * B + lane];
                        }
                    } else if constexpr (kChainDense >= 3) {
                        if (k >= 3) {   // x_{k-3}: this team's previous block
#pragma unroll
                            for (int u = 0; u < C::kSlice; u++)
                                c1 = cfma(c1, G[2 * B * B + (j0 + u) * B + lane], xw[j0 + u]);
                        }
                    }
                    TPROF(k, 11);
                    if (k >= 2) {
                        mbar_wait(xfull + (k - 2) % C::kRing, (uint32_t)(((k - 2) / C::kRing) & 1));   // x_{k-2}
                        TPROF(k, 12);
                        const double2* x2 = ring + (((int64_t)(k - 2) * B) & kRingMask);
#pragma unroll
                        for (int u = 0; u < C::kSlice; u++) carry = cfma(carry, G[B * B + (j0 + u) * B + lane], x2[j0 + u]);
                    }
                    carry = cadd(carry, c1);
                    if constexpr (kG3Ldg) {   // + the partial of G3 warp tw (columns 8 tw .. 8 tw + 7 of G3_k, lane = row)
                        mbar_wait(reinterpret_cast<uint64_t*>(smem + C::kOffG3Lfull) + k % C::kG3Slots,
                                  (uint32_t)((k / C::kG3Slots) & 1));
                        carry = cadd(carry, reinterpret_cast<const double2*>(smem + C::kOffG3Lp)[((k % C::kG3Slots) * 4 + tw) * B + lane]);
                    }
                    TPROF(k, 13);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(gempty + s);
                }
                // y_k (lane = row), staged by the producer once the helpers published it
                double2 yk;
                {
                    const int s = k % C::kSStages;
                    mbar_wait(rfull + s, (uint32_t)((k / C::kSStages) & 1));
                    yk = reinterpret_cast<const double2*>(smem + C::kOffSR + C::kSStage * s)[lane];
                    __syncwarp();
                    if (lane == 0) {
                        mbar_arrive(empty + s);
                        if (tw == 0) mbar_expect_tx(pbar + k % C::kPbuf, (uint32_t)(C::kLt * B * 16));   // the q_l of block k
                    }
                }
                TPROF(k, 1);
                if (trace && tw == 0 && lane == 0) STAMP(k, 10);
                // ---- the chain
                double2 xs[C::kSlice];
                if (k >= 1) {
                    mbar_wait(xfull + (k - 1) % C::kRing, (uint32_t)(((k - 1) / C::kRing) & 1));   // x_{k-1}
                    const double2* xr = ring + (((int64_t)(k - 1) * B) & kRingMask);
#pragma unroll
                    for (int u = 0; u < C::kSlice; u++) xs[u] = xr[j0 + u];
                } else {
#pragma unroll
                    for (int u = 0; u < C::kSlice; u++) xs[u] = make_double2(0.0, 0.0);
                }
                TPROF(k, 2);
                if (trace && tw == 0 && lane == 0) STAMP(k, 13);
                double2 p0 = carry, p1 = make_double2(0.0, 0.0);
                double2 p2 = make_double2(0.0, 0.0), p3 = make_double2(0.0, 0.0);
#pragma unroll
                for (int u = 0; u < C::kSlice; u += 4) {
                    p0 = cfma(p0, g1[u], xs[u]);
                    p1 = cfma(p1, g1[u + 1], xs[u + 1]);
                    p2 = cfma(p2, g1[u + 2], xs[u + 2]);
                    p3 = cfma(p3, g1[u + 3], xs[u + 3]);
                }
                tpart[(pq * C::kTeam + tw) * B + lane] = cadd(cadd(p0, p1), cadd(p2, p3));
                mbar_arrive(pready + pq);   // every lane, after its own partial
                TPROF(k, 3);
                // only warps 0 (ring) and 1 (lieutenants) need x_k (and, with kDense >= 3, every
                // warp for its x_{k-3} carry): the others go on to their next block
                if ((kChainDense < 3 || kG3Warps) && tw >= 2) continue;
                // y_k - sum_l q_l (the lieutenants' D_k^{-1}-multiplied partials), overlapping the
                // other warps' partials
#if !defined(SSB_NO_Q_WAIT)   // (timing experiment only: the chain without the q wait; wrong results)
                mbar_wait(pbar + k % C::kPbuf, (uint32_t)((k / C::kPbuf) & 1));
#endif
                if (trace && tw == 0 && lane == 0) STAMP(k, 6);
#pragma unroll
                for (int l = 0; l < C::kLt; l++) yk = csub(yk, pbuf[((k % C::kPbuf) * C::kLt + l) * B + lane]);
                mbar_wait(pready + pq, (uint32_t)((k >> 2) & 1));   // the team's partials
                TPROF(k, 4);
                if (trace && tw == 0 && lane == 0) STAMP(k, 0);
                double2 sum = tpart[(pq * C::kTeam + 0) * B + lane];
#pragma unroll
                for (int w = 1; w < C::kTeam; w++) sum = cadd(sum, tpart[(pq * C::kTeam + w) * B + lane]);
                const double2 xk = csub(yk, sum);
                TPROF(k, 5);
                // x_k to the lieutenants' rings (st.async completes 16 bytes of the peer's xbar):
                // warp 1 pushes to lieutenants [kPush0, kLt), warp 0 -- after releasing x_k in
                // the local ring for the next team -- to [0, kPush0)
                constexpr int kPush0 = SSB_PUSH_SPLIT;
                auto push = [&](int l0, int l1) {
                    const uint32_t off = (uint32_t)((((int64_t)k * B + lane) & (C::kRingLt * B - 1)) * 16);
                    const uint32_t bar = (uint32_t)((k % C::kRingLt) * 8);
#pragma unroll
                    for (int l = l0; l < l1; l++) {
                        if (lane == 0)   // the single arrival of the phase, expecting the block's bytes
                            mbar_arrive_expect_tx_remote(peer_xbar[l] + bar, B * 16);
                        st_async2(peer_ring[l] + off, xk, peer_xbar[l] + bar);
                    }
                };
                if (tw == 0) {
                    ring[((int64_t)k * B + lane) & kRingMask] = xk;
                    mbar_arrive(xfull + k % C::kRing);   // every lane releases its own x_k[lane]
                    TPROF(k, 6);
                    if (trace && lane == 0) STAMP(k, 3);
                    if constexpr (kPush0 > 0) push(0, kPush0);
                } else if (tw == 1) {
                    push(kPush0, C::kLt);
                    if (trace && lane == 0) STAMP(k, 8);
                }
                if constexpr (kChainDense >= 3 && !kG3Warps) {
                    xw[lane] = xk;   // my x_k: the carry of block k+3
                    __syncwarp();
                }
                TPROF(k, 7);
            }
            }
        } else if (kG3Ldg && chain && (warp == 3 || warp == 4 || warp >= 17)) {
            // ------------------------------------------------ G3-from-L2 warps (3, 4, 17, 18): warp h takes
            // columns 8 h .. 8 h + 7 of G3_k (lane = row) straight from global memory (L2-prefetched
            // 8 blocks ahead, registers double-buffered over two blocks), waits for x_{k-3} in the
            // chain ring and leaves its partial for lane group h of the teams (tpart region, 4 slots):
            // d = 3 never crosses DSMEM and adds nothing to the G ring.
            const int h = warp < 17 ? warp - 3 : warp - 15;
            uint64_t* g3f = reinterpret_cast<uint64_t*>(smem + C::kOffG3Lfull);
            const double2* gsrc = a.G + 2 * B * B + (h * 8) * B + lane;
            constexpr int64_t kStride = (int64_t)kDense * B * B;
            double2 ba[8], bb[8];
            auto load = [&](double2* buf, int k) {
#pragma unroll
                for (int u = 0; u < 8; u++) buf[u] = __ldg(gsrc + (int64_t)k * kStride + u * B);
                if (k + 8 < nblk) {
#pragma unroll
                    for (int u = 0; u < 8; u++)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(gsrc + (int64_t)(k + 8) * kStride + u * B));
                }
            };
            auto compute = [&](const double2* buf, int k) {
                double2 a0 = make_double2(0.0, 0.0), a1 = a0;
                if (k >= 3) {   // (blocks 0 .. 2 have no source: zero partials keep the slot phases in step)
                    mbar_wait(xfull + (k - 3) % C::kRing, (uint32_t)(((k - 3) / C::kRing) & 1));   // x_{k-3}
                    const double2* x3 = ring + (((int64_t)(k - 3) * B) & kRingMask) + h * 8;
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        a0 = cfma(a0, buf[u], x3[u]);
                        a1 = cfma(a1, buf[u + 1], x3[u + 1]);
                    }
                }
                reinterpret_cast<double2*>(smem + C::kOffG3Lp)[((k % C::kG3Slots) * 4 + h) * B + lane] = cadd(a0, a1);
                mbar_arrive(g3f + k % C::kG3Slots);   // every lane, after its own partial
            };
            if (nblk > 0) load(ba, 0);
            for (int k = 0; k < nblk; k += 2) {
                if (k + 1 < nblk) load(bb, k + 1);
                compute(ba, k);
                if (k + 2 < nblk) load(ba, k + 2);
                if (k + 1 < nblk) compute(bb, k + 1);
            }
        } else if (kG3Warps && chain && (warp == C::kWG3 || warp == C::kWG3 + 1)) {
            // ------------------------------------------------ G3 warps: G3_k x_{k-3} (dense, from the
            // G ring) as soon as x_{k-3} is in the ring, two halves of 16 columns, for the team
            // of block k (two steps of slack: off the chain and off the lieutenants' DSMEM path)
            const int h = warp - C::kWG3;
            double2* g3p = reinterpret_cast<double2*>(smem + C::kOffG3p);
            double2* g3v = reinterpret_cast<double2*>(smem + C::kOffG3v);
            uint64_t* g3full = reinterpret_cast<uint64_t*>(smem + C::kOffG3full);
            for (int k = 0; k < nblk; k++) {
                const int s = k % C::kGStages;
                mbar_wait(gfull + s, (uint32_t)((k / C::kGStages) & 1));
                if (k >= 3) {
                    const double2* G = reinterpret_cast<const double2*>(smem + C::kGStage * s) + 2 * B * B;
                    mbar_wait(xfull + (k - 3) % C::kRing, (uint32_t)(((k - 3) / C::kRing) & 1));   // x_{k-3}
                    const double2* x3 = ring + (((int64_t)(k - 3) * B) & kRingMask);
                    double2 a0 = make_double2(0.0, 0.0), a1 = a0;
#pragma unroll
                    for (int u = 0; u < 16; u += 2) {
                        a0 = cfma(a0, G[(h * 16 + u) * B + lane], x3[h * 16 + u]);
                        a1 = cfma(a1, G[(h * 16 + u + 1) * B + lane], x3[h * 16 + u + 1]);
                    }
                    g3p[h * B + lane] = cadd(a0, a1);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(gempty + s);
                bar_named(8, 64);   // both halves written
                if (h == 0 && k >= 3) {
                    g3v[((k - 3) & 3) * B + lane] = cadd(g3p[lane], g3p[B + lane]);
                    mbar_arrive(g3full + ((k - 3) & 3));
                }
                bar_named(8, 64);   // halves read before the next block overwrites them
            }
        } else if (!chain) {
            // ------------------------------------------------ lieutenants: list B partial sums
            // (source distance kDense+1 .. Q_k-1) of the rows l, l+kLt, ...; kLtTeams teams of
            // 4 warps take the blocks k mod kLtTeams.  The early part (distance >= kDense+2) is
            // summed once x_{k-kDense-2} has landed, the late part (kDense+1) once x_{k-kDense-1}
            // has.  x blocks land by
            // st.async from the chain team, which also makes each xbar phase's one arrival.
            // Each lieutenant sends q_l = D_k^{-1}[:, its rows] (its row partials), so the chain
            // only subtracts the three q_l from y_k = D_k^{-1} r_k.
            const int l = role - 1;
            uint64_t* lbar = reinterpret_cast<uint64_t*>(smem + C::kOffLbar);
            const uint32_t peer_pbuf = mapa(smem_u32(pbuf), 0u);
            const uint32_t peer_pbar = mapa(smem_u32(pbar), 0u);
            const double2* ltring = reinterpret_cast<const double2*>(smem + C::kOffLtRing);
            const int lteam = tid / C::kLtTeamT, tt = tid % C::kLtTeamT;
            double2* lp = reinterpret_cast<double2*>(smem + C::kOffLtP) + lteam * B;   // row partials
            int xseen = 0;   // x blocks < xseen have landed in the ring
            const int r = l + C::kLt * (tt / C::kTPRl), q = tt % C::kTPRl;
            const bool rowok = r < B;
            auto land = [&](int upto) {   // wait for the xbar phases of blocks xseen .. upto, in order
                for (; xseen <= upto; xseen++)
                    mbar_wait(xbar + xseen % C::kRingLt, (uint32_t)((xseen / C::kRingLt) & 1));
            };
            if (lteam < C::kLtTeams) {
                for (int k = lteam; k < nblk; k += C::kLtTeams) {
                    const int s = k % nst;
                    unsigned char* st = smem + stsz * s;
                    constexpr int kRows = C::kRowsL;
                    double2 dq[kRows];   // D_k^{-1}[tt, l + kLt m] (predicated: 0 above the diagonal)
                    if (kLtDinvLdg && tt < B) {   // from L2 (the helper of block k staged it long ago)
                        const double2* gInv = a.dinv + (int64_t)k * C::kPK;
#pragma unroll
                        for (int m = 0; m < kRows; m++) {
                            const int rr = m * C::kLt + l;
                            const bool ok = rr <= tt;
                            dq[m] = __ldg(gInv + (ok ? rr * B - (rr * (rr - 1)) / 2 + (tt - rr) : 0));
                            dq[m].x = ok ? dq[m].x : 0.0;
                            dq[m].y = ok ? dq[m].y : 0.0;
                        }
                    }
                    double2 g3[kRows];   // (kLtG3) G3_k[tt, l + kLt m]: prefetched into L2 now, loaded below
                    if (kLtG3 && tt < B && k + C::kLtTeams < nblk) {   // this team's next block: four steps ahead
                        const double2* gG3 = a.G + ((int64_t)(k + C::kLtTeams) * kDense + 2) * B * B + tt;
#pragma unroll
                        for (int m = 0; m < kRows; m++) {
                            const int c = m * C::kLt + l;
                            if (c < B) asm volatile("prefetch.global.L2 [%0];" ::"l"(gG3 + c * B));
                        }
                    }
                    LPROF(k, 0);
                    mbar_wait(full + s, (uint32_t)((k / nst) & 1));
                    LPROF(k, 1);
                    const bool tr0 = trace && tt == 0 && l == 0;
                    if (tr0) STAMP(k, 12);
                    const int32_t* loc = reinterpret_cast<const int32_t*>(st + C::kOffBloc);
                    const int32_t* col = reinterpret_cast<const int32_t*>(st + C::kOffBcol);
                    const double2* val = reinterpret_cast<const double2*>(st + C::kOffBval);
                    double2 acc = make_double2(0.0, 0.0);
                    land(k - kDense - 2);
                    if constexpr (kLtGate > 0) {   // block k-1's late part (same trigger x_{k-3}) first
                        if (k >= 1) mbar_wait(lbar + ((k - 1) & 3), (uint32_t)(((k - 1) >> 2) & 1));
                    }
                    LPROF(k, 2);
                    if (rowok) acc = near_range<B, C::kTPRl, C::kRingLt>(col, val, ltring, loc[r], loc[C::kLate + r], q, acc);
#pragma unroll
                    for (int o = 1; o < C::kTPRl; o <<= 1) {   // the early part, reduced before the late one lands
                        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                    }
                    if (q != 0) acc = make_double2(0.0, 0.0);
                    const int lt0 = rowok ? loc[C::kLate + r] : 0, lt1 = rowok ? loc[r + 1] : 0;   // late part
                    // the first 2 kTPRlate entries of the row's late part: columns and values now,
                    // x once it has landed (predicated: absent entries get value 0)
                    constexpr int kRM = C::kRingLt * B - 1;
                    int lc0 = 0, lc1 = 0;
                    double2 lv0 = make_double2(0.0, 0.0), lv1 = lv0;
                    bool lok0 = false, lok1 = false;   // the prefetched entries exist
                    auto pre = [&](int p0, int p1, int& c0, int& c1, double2& v0, double2& v1) {
                        const int e0 = p0 + q, e1 = e0 + C::kTPRlate;
                        const bool ok0 = e0 < p1, ok1 = e1 < p1;
                        lok0 = ok0;
                        lok1 = ok1;
                        c0 = col[ok0 ? e0 : 0];
                        c1 = col[ok1 ? e1 : 0];
                        v0 = val[ok0 ? e0 : 0];
                        v1 = val[ok1 ? e1 : 0];
                        v0.x = ok0 ? v0.x : 0.0;
                        v0.y = ok0 ? v0.y : 0.0;
                        v1.x = ok1 ? v1.x : 0.0;
                        v1.y = ok1 ? v1.y : 0.0;
                    };
                    if (rowok && q < C::kTPRlate) pre(lt0, lt1, lc0, lc1, lv0, lv1);
                    // and this thread's entries of D_k^{-1} for the q product below
                    if (!kLtDinvLdg && tt < B) {
                        const double2* sInv = reinterpret_cast<const double2*>(st + C::kOffBinv);
#pragma unroll
                        for (int m = 0; m < kRows; m++) {
                            const int rr = m * C::kLt + l;
                            const bool ok = rr <= tt;
                            dq[m] = sInv[ok ? rr * B - (rr * (rr - 1)) / 2 + (tt - rr) : 0];
                            dq[m].x = ok ? dq[m].x : 0.0;
                            dq[m].y = ok ? dq[m].y : 0.0;
                        }
                    }
                    if (kLtG3 && tt < B && k >= 3) {   // (L2 hits: prefetched at the top of the block)
                        const double2* gG3 = a.G + ((int64_t)k * kDense + 2) * B * B + tt;
#pragma unroll
                        for (int m = 0; m < kRows; m++) {
                            const int c = m * C::kLt + l;
                            g3[m] = c < B ? __ldg(gG3 + c * B) : make_double2(0.0, 0.0);
                        }
                    }
                    LPROF(k, 3);
                    if (tr0) STAMP(k, 11);
                    land(k - kDense - 1);
                    LPROF(k, 4);
                    if (tr0) STAMP(k, 7);
                    if (rowok && q < C::kTPRlate) {
                        // an absent entry reads a ring slot this launch may not have written yet (whatever
                        // the last kernel left in shared memory, possibly a NaN pattern): 0 * NaN = NaN, so
                        // the OPERAND is zeroed too, not only the value
                        double2 lx0 = ltring[lc0 & kRM], lx1 = ltring[lc1 & kRM];
                        if (kZeroOperands) {
                            lx0.x = lok0 ? lx0.x : 0.0;
                            lx0.y = lok0 ? lx0.y : 0.0;
                            lx1.x = lok1 ? lx1.x : 0.0;
                            lx1.y = lok1 ? lx1.y : 0.0;
                        }
                        acc = cfma(acc, lv0, lx0);
                        acc = cfma(acc, lv1, lx1);
                        for (int e = lt0 + q + 2 * C::kTPRlate; e < lt1; e += C::kTPRlate)   // long rows
                            acc = cfma(acc, val[e], ltring[col[e] & kRM]);
                    }
#pragma unroll
                    for (int o = 1; o < C::kTPRlate; o <<= 1) {
                        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
                        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
                    }
                    LPROF(k, 5);
                    if (rowok && q == 0) lp[r] = acc;
                    bar_named(2 + lteam, C::kLtTeamT);
                    if (kLtGate == 1 && tt == 0) mbar_arrive(lbar + (k & 3));
                    LPROF(k, 6);
                    // q_l = D_k^{-1}[:, rows of l] p_l: one thread per output row i (the team's first
                    // warp), the lieutenant's rows rr = l, l + kLt, ... <= i in order
                    if (tt < B) {
                        const int i = tt;
                        double2 qa = make_double2(0.0, 0.0), qb = make_double2(0.0, 0.0);
                        double2 pq[kRows];
#pragma unroll
                        for (int m = 0; m < kRows; m++) {
                            const int rr = m * C::kLt + l;
                            pq[m] = lp[rr < B ? rr : 0];   // (rr >= B: lp[0] is another lieutenant's row, never
                            if (kZeroOperands) {                // written here -- uninitialised shared memory; zeroed,
                                pq[m].x = rr < B ? pq[m].x : 0.0;   // because 0 * NaN = NaN)
                                pq[m].y = rr < B ? pq[m].y : 0.0;
                            }
                        }
#pragma unroll
                        for (int m = 0; m < kRows; m += 2) {
                            qa = cfma(qa, dq[m], pq[m]);
                            if (m + 1 < kRows) qb = cfma(qb, dq[m + 1], pq[m + 1]);
                        }
                        const int pk = k % C::kPbuf;
                        double2 qv = cadd(qa, qb);
                        if (kLtG3 && k >= 3) {   // + G3_k[:, my columns] x_{k-3}[my columns]: the only late term
                            land(k - 3);
                            if (tr0) STAMP(k, 14);
                            const double2* x3 = ltring + (((int64_t)(k - 3) * B) & kRM);
                            double2 qc = make_double2(0.0, 0.0);
#pragma unroll
                            for (int m = 0; m < kRows; m += 2) {
                                const int c0 = m * C::kLt + l, c1 = (m + 1) * C::kLt + l;
                                qv = cfma(qv, g3[m], x3[c0 < B ? c0 : 0]);
                                if (m + 1 < kRows) qc = cfma(qc, g3[m + 1], x3[c1 < B ? c1 : 0]);
                            }
                            qv = cadd(qv, qc);
                        }
                        st_async2(peer_pbuf + (uint32_t)(((pk * C::kLt + l) * B + i) * 16), qv,
                                  peer_pbar + (uint32_t)(pk * 8));
                        if (kLtGate == 2) {
                            __syncwarp();
                            if (tt == 0) mbar_arrive(lbar + (k & 3));
                        }
                        LPROF(k, 7);
                        if (tr0) STAMP(k, 9);
                        if (trace && tt == 0 && l == C::kLt - 1) STAMP(k, 2);
                    }
                    bar_named(2 + lteam, C::kLtTeamT);
                    LPROF(k, 8);
                    if (tt == 0) {
                        mbar_arrive(empty + s);

                    }
                }
                // before leaving, every x push to this CTA has landed: the last phase of each
                // xbar slot (earlier phases of a slot completed before it)
                if (xseen < nblk - C::kRingLt) xseen = nblk - C::kRingLt;
                land(nblk - 1);
            }
        }
        // no CTA of the cluster leaves while a peer may still access its shared memory
        __syncwarp();
        cluster_sync();
        return;
    }

    // ================================================================ helper CTAs
    // The far part of block k is cut into work items (row r, 32-entry chunk c), sorted at
    // setup by the newest source block they read (setup.cpp); warp w takes items w, w+16,
    // ..., kHU at a time (their column/value loads in flight together), waits once for the
    // newest source block of the batch, gathers x, and adds each item's warp sum to its
    // per-warp row partial (lane 0, item order: deterministic).  A block's long rows are so
    // spread over all 16 warps, and the items gated by the newest x blocks come last.
    if (warp >= C::kFarWarps) return;
#ifndef SSB_HU
#define SSB_HU 4   // far work items in flight per helper warp
#endif
    constexpr int kHU = SSB_HU;
    const int H = gridDim.x - C::kCluster;
    int64_t* sRowP = reinterpret_cast<int64_t*>(smem + C::kOffRowP);
    int32_t* sRowL = reinterpret_cast<int32_t*>(smem + C::kOffRowL);
    double2* sRf = reinterpret_cast<double2*>(smem + C::kOffR);   // b_k - far part
    const double2* hInv = reinterpret_cast<const double2*>(smem);  // D_k^{-1}, staged by TMA
    // per-warp row partials of the far sums, in the stage region after D_k^{-1} (helpers
    // use no stages)
    double2* hpart = reinterpret_cast<double2*>(smem + ((C::kPK * 16 + 127) & ~(size_t)127));
    static_assert(((C::kPK * 16 + 127) & ~(size_t)127) + (size_t)C::kFarWarps * B * 16 <= C::kStageRegion,
                  "helper partials fit the stage region");
    const int yi = tid / C::kYP, yp = tid % C::kYP;               // D^{-1} product: row, column class
    int hit = 0;                                                   // blocks done by this CTA
    for (int k = blockIdx.x - C::kCluster; k < nblk; k += H, hit++) {
        const int64_t row0 = (int64_t)k * B;
        if (tid == 0) {   // D_k^{-1} lands while the far part streams (full[0]: this CTA's barrier)
            mbar_expect_tx(full, (uint32_t)(C::kPK * 16));
            bulk_g2s(smem, a.dinv + (int64_t)k * C::kPK, C::kPK * 16, full);
        }
        if (warp == 0) {
            const int64_t i = row0 + lane;
            int64_t p0 = 0, l0 = 0;
            if (i < n) {
                p0 = a.farptr[i];
                l0 = a.farptr[i + 1] - p0;
            }
            sRowP[lane] = p0;
            sRowL[lane] = (int32_t)l0;
        }
        hpart[warp * B + lane] = make_double2(0.0, 0.0);
        const int64_t t0 = __ldg(a.itemptr + k), t1 = __ldg(a.itemptr + k + 1);
        bar_named(1, C::kHelperT);
#pragma unroll 1
        for (int64_t t = t0 + warp; t < t1; t += (int64_t)C::kFarWarps * kHU) {
            int32_t cc[kHU];
            double2 vv[kHU];
            int rr[kHU];
            int32_t need = -1;
#pragma unroll
            for (int u = 0; u < kHU; u++) {
                const int64_t tt = t + (int64_t)u * C::kFarWarps;
                const uint32_t it = tt < t1 ? __ldg(a.items + tt) : 0xffffffffu;
                rr[u] = it == 0xffffffffu ? -1 : (int)(it & (B - 1));
                cc[u] = -1;
                if (rr[u] >= 0) {
                    const int32_t pos = (int32_t)(it >> 5) * 32 + lane;
                    if (pos < sRowL[rr[u]]) {
                        cc[u] = ld_stream(a.fcol + sRowP[rr[u]] + pos);
                        vv[u] = ld_stream2(a.fval + sRowP[rr[u]] + pos);
                        need = max(need, cc[u]);
                    }
                }
            }
            need = __reduce_max_sync(0xffffffffu, need);
            if (need >= 0) helper_wait(need / B + 1, sF, sLock, a.xfront, epoch);
            double2 xv[kHU];
#pragma unroll
            for (int u = 0; u < kHU; u++)
                if (cc[u] >= 0) xv[u] = ld_cg2(x + phys(cc[u]));
#pragma unroll
            for (int u = 0; u < kHU; u++) {
                double2 acc = make_double2(0.0, 0.0);
                if (cc[u] >= 0) acc = cfma(acc, vv[u], xv[u]);
                acc = warp_sum2(acc);
                if (lane == 0 && rr[u] >= 0) hpart[warp * B + rr[u]] = cadd(hpart[warp * B + rr[u]], acc);
            }
        }
        bar_named(1, C::kHelperT);
        if (warp == 0) {   // lane = row: the 16 warp partials in order
            double2 sm = hpart[lane];
#pragma unroll
            for (int w = 1; w < C::kFarWarps; w++) sm = cadd(sm, hpart[w * B + lane]);
            const int64_t i = row0 + lane;
            sRf[lane] = (i < n) ? csub(__ldg(bvec + phys(i)), sm) : make_double2(0.0, 0.0);
        }
        bar_named(1, C::kHelperT);
        mbar_wait(full, (uint32_t)(hit & 1));
        double2 dv[B / C::kYP];   // D_k^{-1}[yi, yp + kYP m]
#pragma unroll
        for (int m = 0; m < B / C::kYP; m++) {
            const int j = yp + C::kYP * m;
            dv[m] = j <= yi ? hInv[j * B - (j * (j - 1)) / 2 + (yi - j)] : make_double2(0.0, 0.0);
        }
        // y_k = D_k^{-1} (b_k - far part): output row yi, columns j = yp, yp + kYP, ...
        {
            double2 ya = make_double2(0.0, 0.0);
#pragma unroll
            for (int m = 0; m < B / C::kYP; m++)
                if (yp + C::kYP * m <= yi) ya = cfma(ya, dv[m], sRf[yp + C::kYP * m]);
#pragma unroll
            for (int o = 1; o < C::kYP; o <<= 1) {
                ya.x += __shfl_xor_sync(0xffffffffu, ya.x, o);
                ya.y += __shfl_xor_sync(0xffffffffu, ya.y, o);
            }
            if (yp == 0) a.yfar[row0 + yi] = ya;
        }
        bar_named(1, C::kHelperT);
        if (tid == 0) {
            st_release(a.fflag + k, epoch);
            if (trace) STAMP(k, 4);
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
    // clusters of 8 (chain + 7 lieutenants, then helpers), one CTA per SM; every cluster
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
    using C = Cfg<B>;
    auto fn = k_chain_trsv<B>;
    if (T.grid == 0) prepare<B>(T);
    T.epoch++;
    TriArgs a = T.args();
    uint32_t ep = T.epoch;
    double2* xw = T.operm ? T.xwork : x;
    int grid = T.grid;
    if (T.sm_budget > 0)   // several problems share the GPU: whole clusters, chain + >= 1 helper cluster
        grid = std::min(grid, std::max(2 * C::kCluster, (T.sm_budget / C::kCluster) * C::kCluster));
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = launch_config<B>(grid, attr);
    cfg.stream = s;
    SSB_CUDA(cudaLaunchKernelEx(&cfg, fn, a, b, x, xw, ep, trace));
    SSB_LAUNCHED();
}

__global__ void __launch_bounds__(256, 1) k_poison_smem(int bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    for (int i = threadIdx.x * 16; i < bytes; i += 256 * 16)
        *reinterpret_cast<uint4*>(smem + i) = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
}

}  // namespace

// ss_debug_poison_smem: one CTA per SM (the full shared memory each, so they cannot share an SM),
// several waves so that every SM is covered whatever else is resident.
void poison_shared_memory(cudaStream_t s) {
    constexpr int kBytes = 232448 - 1024;
    SSB_CUDA(cudaFuncSetAttribute(k_poison_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes));
    int dev = 0, sms = 0;
    SSB_CUDA(cudaGetDevice(&dev));
    SSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    k_poison_smem<<<4 * sms, 256, kBytes, s>>>(kBytes);
    SSB_CUDA(cudaGetLastError());
    SSB_LAUNCHED();
}

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
