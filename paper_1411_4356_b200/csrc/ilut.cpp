// ilut.cpp -- dual-threshold incomplete LU with column pivoting (ILUTP) of L~_RCM (setup,
// host, multi-threaded).
//
// PAPER.md:94 (sec. II): "an incomplete LU factorization with dual-threshold and pivoting
// (iLUTP) ... a drop tolerance d and allowed fill-in p are specified such that all fill-in
// smaller than d times the infinity-norm of a row are dropped, and at most only
// p NNZ(L~) fill-in elements are allowed".  Row-wise (IKJ) ILUTP as in the paper's
// reference [saad:2003]; the exact rules (R4-R7, R13 in DESIGN.md):
//   tau_i = d * max_j |a_ij|; a value z is dropped iff |z|^2 < tau_i^2;
//   multiplier w_k <- w_k * (1/u_kk), 1/u = (ur, -ui)/(ur^2+ui^2), dropped by the same
//   test before it is used; update w_j <- w_j - w_k u_kj (no FMA: -ffp-contract=off);
//   after elimination the L part and the strict U part of the row each keep at most
//   floor(p * nnz(a_i) / 2) entries of largest |.|^2 (ties: smaller position);
//   pivoting: A Pi = L U; the largest kept U entry |w_t|^2 (ties: smaller position)
//   replaces the diagonal when permtol^2 |w_t|^2 > |w_i|^2 -- positions i and t are
//   exchanged for this and all later rows; a zero pivot left after that becomes tau_i
//   (error if tau_i = 0).  permtol = 0 is plain ILUT.
//
// B200-first change vs. a serial ILUTP: rows are factorised by a pool of host threads.
// A column's position can only change at a step s <= its position (step s exchanges
// positions s and t >= s), so every position below the published frontier F (rows < F
// finished) is final.  A thread claims the next row, keeps its working row in ORIGINAL
// columns, and eliminates the positions < F in increasing order as F advances (the U
// rows it needs are published by then); once F reaches its row it drops, caps,
// pivots and publishes (F = i + 1).  The operands and their order are those of the
// serial algorithm, so the factors are bit-identical for any thread count.  U rows are
// kept in original columns while factoring (later exchanges move positions > i) and
// converted to final positions at the end.
//
// The chain of row hand-offs (row i needs U row i-1) is the critical path, so the work
// between "F reaches i" and "U row i published" is kept small: the row's positions live in
// a bitmap (elimination order = ascending set bits, no heaps), the U candidates are
// snapshotted while the last kSnapAhead rows are still being finished elsewhere and kept
// current by the late updates, the cap is a counting selection over binary orders of
// magnitude, the U row is published in position order as selected, and the L row, the
// clearing of the work row and the arena page faults are done after publication.  Each
// thread keeps two rows in flight (RowWork): while the row it publishes next waits for the
// frontier, it eliminates ahead in the next one (SSB_ILUT_ROWS=1: one row).
// SSB_ILUT_PROF=1 prints the per-row time of each phase.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <thread>

#if defined(__x86_64__)
#include <immintrin.h>
#define SSB_PAUSE() _mm_pause()
#else
#define SSB_PAUSE() std::this_thread::yield()
#endif
// spin, and give the core away now and then (another thread may own the next row)
#define SSB_BACKOFF(cnt)                                 \
    do {                                                 \
        if (((++(cnt)) & 255) == 0) std::this_thread::yield(); \
        else SSB_PAUSE();                                \
    } while (0)

#include "problem.h"

namespace ssb {

namespace {

inline double mag2(double2 z) { return z.x * z.x + z.y * z.y; }

// append-only storage whose blocks never move (other threads read published rows)
struct Arena {
    static constexpr int64_t kBlock = 1 << 20;
    std::vector<std::unique_ptr<int32_t[]>> cblocks;
    std::vector<std::unique_ptr<double2[]>> vblocks;
    int64_t used = kBlock, size = 0;
    int64_t touched = 0;   // entries of the current block whose pages were written
    void grow(int64_t len) {
        size = std::max(kBlock, len);
        cblocks.emplace_back(new int32_t[size]);
        vblocks.emplace_back(new double2[size]);
        used = touched = 0;
    }
    void reserve(int64_t len, int32_t*& c, double2*& v) {
        if (cblocks.empty() || used + len > size) grow(len);
        c = cblocks.back().get() + used;
        v = vblocks.back().get() + used;
        used += len;
    }
    // take the page faults of the next `ahead` entries now (off the critical path)
    void prefault(int64_t ahead) {
        if (cblocks.empty() || used + ahead > size) grow(ahead);
        const int64_t end = std::min(size, used + ahead);
        int32_t* c = cblocks.back().get();
        double2* v = vblocks.back().get();
        for (int64_t e = std::max(touched, used); e < end; e += 256) v[e] = make_double2(0.0, 0.0);   // 4 KB
        for (int64_t e = std::max(touched, used); e < end; e += 1024) c[e] = 0;
        touched = std::max(touched, end);
    }
};

struct RowRef {
    const int32_t* c = nullptr;   // int32: n < 2^31 (checked), fewer bytes per re-read U row
    const double2* v = nullptr;
    int64_t len = 0;
};

struct Ent {
    int64_t j;   // position
    int64_t c;   // original column
    double2 v;
    double m;
};

struct Shared {
    const HostCSR& A;
    double drop_tol, fill_factor, permtol;
    int64_t n;
    std::atomic<int64_t> next{0};
    std::atomic<int64_t> front{0};                    // rows < front are published
    std::atomic<int64_t> swap_version{0};             // bumped by every column exchange
    std::unique_ptr<std::pair<int64_t, int64_t>[]> swap_log;   // exchange v: positions (s, t)
    std::unique_ptr<std::atomic<int64_t>[]> perm;     // position -> original column
    std::unique_ptr<std::atomic<int64_t>[]> iperm;    // original column -> position
    std::vector<RowRef> Lrow, Urow;                   // L: positions; U: original columns
    std::atomic<int> error_row{-1};
    std::atomic<int32_t> repaired{0}, swaps{0};
    int rows_per_thread = 2;                          // SSB_ILUT_ROWS (1 or 2)
    int64_t snap_ahead = 2;                           // kSnapAhead (SSB_ILUT_SNAP)
    bool prof = false;                                // SSB_ILUT_PROF: per-phase times (stderr)
    std::atomic<int64_t> t_elim{0}, t_spin{0}, t_wait{0}, t_fin{0}, n_late{0}, t_post{0}, n_cand{0}, n_lcand{0},
        t_fcand{0}, t_fsel{0}, n_kept{0}, n_snap{0};
    explicit Shared(const HostCSR& a) : A(a) {}
};

constexpr int64_t kSnapAhead = 2;   // snapshot the U candidates once F >= i - kSnapAhead (SSB_ILUT_SNAP)

// next set bit of b in [from, lim), else lim
inline int64_t next_bit(const uint64_t* b, int64_t from, int64_t lim) {
    if (from >= lim) return lim;
    int64_t wi = from >> 6;
    uint64_t x = b[wi] & (~0ull << (from & 63));
    for (;;) {
        if (x) {
            const int64_t p = (wi << 6) + __builtin_ctzll(x);
            return p < lim ? p : lim;
        }
        if ((++wi << 6) >= lim) return lim;
        x = b[wi];
    }
}

// the k-th largest of m[0..cnt) (1 <= k < cnt; all m > 0): one counting pass over binary
// orders of magnitude, then a selection inside the one bucket that holds it
inline double kth_largest(const double* m, size_t cnt, int64_t k, std::vector<double>& tmp) {
    constexpr int kBins = 128;
    uint32_t hist[kBins] = {};
    auto bexp = [](double x) {
        uint64_t b;
        std::memcpy(&b, &x, 8);
        return (int)(b >> 52);   // x >= 0: sign bit clear
    };
    int emax = 0;
    for (size_t t = 0; t < cnt; t++) emax = std::max(emax, bexp(m[t]));
    auto bin = [&](double x) { return std::min(kBins - 1, emax - bexp(x)); };   // 0 = largest
    for (size_t t = 0; t < cnt; t++) hist[bin(m[t])]++;
    int b = 0;
    int64_t above = 0;
    while (above + hist[b] < k) above += hist[b++];
    tmp.clear();
    for (size_t t = 0; t < cnt; t++)
        if (bin(m[t]) == b) tmp.push_back(m[t]);
    const int64_t r = k - above;   // 1 <= r <= hist[b]
    std::nth_element(tmp.begin(), tmp.begin() + (r - 1), tmp.end(), std::greater<double>());
    return tmp[r - 1];
}

using clk = std::chrono::steady_clock;
inline int64_t ns_between(clk::time_point a, clk::time_point b) {
    return (int64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
}

// One row in factorisation: its work row, position bitmap, U-candidate snapshot and
// progress.  A thread holds up to two (worker below): the row it will publish next
// and, while that one waits for the frontier, the next row it claimed.
struct RowWork {
    Shared& S;
    const int64_t n;
    std::vector<double2> w;        // indexed by ORIGINAL column
    std::vector<uint8_t> present;
    // the row's columns by POSITION: bit p set = the column at position p is in the row.
    // Positions are eliminated in increasing order by scanning the bits (fill from U row k
    // lies at positions > k), the U part is the bits >= i.
    std::vector<uint64_t> bits;
    uint64_t* bt;
    std::vector<int64_t> nz;
    std::vector<Ent> lbuf, buf;
    std::vector<double> mk, km;
    // U candidates of the row (positions > i): snapshot taken while the last rows before i are
    // finished by other threads; afterwards only the entries the late U rows touch change
    std::vector<int32_t> sidx;   // column -> snapshot index
    std::vector<int64_t> s_pos, s_col;
    std::vector<double> s_m;
    std::vector<uint8_t> s_bin;   // histogram bin of s_m, kNotKept if dropped
    std::vector<int32_t> ties;
    bool snapped = false;
    // histogram of the kept (not dropped) snapshot magnitudes over binary orders of
    // magnitude below the row's scale, maintained with s_m: the cap's bucket is known
    // without a pass
    static constexpr int kHB = 128;
    static constexpr uint8_t kNotKept = 255;
    uint32_t shist[kHB];
    // the row
    bool active = false;
    int64_t i = -1, lfil = 0, cursor = 0, my_version = 0, lo, hi = -1;
    double rowmax2 = 0.0, tau2 = 0.0;
    int cur_base = 0;
    // profile (SSB_ILUT_PROF)
    clk::time_point tp0;
    int64_t p_elim = 0, p_late = 0, p_wait = 0, p_fin = 0, p_post = 0, p_cand = 0, p_lcand = 0;
    int64_t p_fcand = 0, p_fsel = 0, p_kept = 0, p_snap = 0;

    enum { kWorked, kIdle, kReady, kError };

    explicit RowWork(Shared& s)
        : S(s), n(s.n), w(s.n, make_double2(0.0, 0.0)), present(s.n, 0), bits(((size_t)s.n >> 6) + 2, 0),
          sidx(s.n, -1), lo(s.n) {
        bt = bits.data();
        nz.reserve(4096);
        buf.reserve(4096);
        lbuf.reserve(4096);
    }
    bool kept(double m) const { return m != 0.0 && !(m < tau2); }
    int hbin(double m) const {
        uint64_t b;
        std::memcpy(&b, &m, 8);
        return std::min(kHB - 1, std::max(0, cur_base - (int)(b >> 52)));
    }
    void setbit(int64_t p) {
        bt[p >> 6] |= 1ull << (p & 63);
        lo = std::min(lo, p);
        hi = std::max(hi, p);
    }
    void clear_bits() {
        if (hi >= lo) std::memset(bt + (lo >> 6), 0, (size_t)((hi >> 6) - (lo >> 6) + 1) * sizeof(uint64_t));
        lo = n;
        hi = -1;
    }
    void take_snapshot() {
        std::memset(shist, 0, sizeof(shist));
        for (int64_t pp = next_bit(bt, i + 1, hi + 1); pp <= hi; pp = next_bit(bt, pp + 1, hi + 1)) {
            const int64_t c = S.perm[pp].load(std::memory_order_relaxed);
            const double m = mag2(w[c]);
            sidx[c] = (int32_t)s_col.size();
            s_pos.push_back(pp);
            s_col.push_back(c);
            s_m.push_back(m);
            const uint8_t bn = kept(m) ? (uint8_t)hbin(m) : kNotKept;
            s_bin.push_back(bn);
            if (bn != kNotKept) shist[bn]++;
        }
        snapped = true;
    }
    void drop_snapshot() {
        for (int64_t c : s_col) sidx[c] = -1;
        s_pos.clear();
        s_col.clear();
        s_m.clear();
        s_bin.clear();
        snapped = false;
    }

    // w <- w - wk * (U row k), new fill recorded; with a snapshot (SN) also keep the
    // magnitudes of the U candidates (positions > i) current
    template <bool SN>
    void update_row(const RowRef& U, double2 wk) {
        const int32_t* __restrict uc = U.c;
        const double2* __restrict uv = U.v;
        double2* __restrict wp = w.data();
        uint8_t* __restrict pr = present.data();
        const int64_t len = U.len;
        for (int64_t q = 1; q < len; q++) {
            const int64_t c = uc[q];
            if (__builtin_expect(!pr[c], 0)) {   // fill: position > k (see above)
                pr[c] = 1;
                wp[c] = make_double2(0.0, 0.0);
                nz.push_back(c);
                const int64_t pc = S.iperm[c].load(std::memory_order_relaxed);
                setbit(pc);
                if (SN && pc > i) {
                    sidx[c] = (int32_t)s_col.size();
                    s_pos.push_back(pc);
                    s_col.push_back(c);
                    s_m.push_back(0.0);
                    s_bin.push_back(kNotKept);
                }
            }
            const double2 u = uv[q];
            const double px = wk.x * u.x - wk.y * u.y;
            const double py = wk.x * u.y + wk.y * u.x;
            double2 t = wp[c];
            t.x = t.x - px;
            t.y = t.y - py;
            wp[c] = t;
            if (SN) {
                const int32_t si = sidx[c];
                if (si >= 0) {
                    const double mn = mag2(t);
                    const uint8_t bo = s_bin[si], bn = kept(mn) ? (uint8_t)hbin(mn) : kNotKept;
                    if (bo != kNotKept) shist[bo]--;
                    if (bn != kNotKept) shist[bn]++;
                    s_m[si] = mn;
                    s_bin[si] = bn;
                }
            }
        }
    }

    void begin(int64_t row) {
        active = true;
        i = row;
        if (S.prof) tp0 = clk::now();
        const int64_t r0 = S.A.rowptr[i], r1 = S.A.rowptr[i + 1];
        lfil = (int64_t)(S.fill_factor * (double)(r1 - r0) / 2.0);
        rowmax2 = 0.0;
        nz.clear();
        lbuf.clear();
        // positions are read after the version: a later exchange is seen as a new version.
        // A position read while an exchange of step s >= f0 is under way may be stale, but
        // then both its old and new value are >= f0, hence cursor <= f0 below.
        const int64_t f0 = S.front.load(std::memory_order_acquire);
        my_version = S.swap_version.load(std::memory_order_acquire);
        for (int64_t q = r0; q < r1; q++) {
            const int64_t c = S.A.col[q];
            const double m = mag2(S.A.val[q]);
            if (m > rowmax2) rowmax2 = m;
            w[c] = S.A.val[q];
            present[c] = 1;
            nz.push_back(c);
            setbit(S.iperm[c].load(std::memory_order_relaxed));
        }
        cursor = std::min(lo, f0);   // the row's positions < cursor are eliminated (or dropped)
        tau2 = S.drop_tol * S.drop_tol * rowmax2;
        uint64_t b;
        std::memcpy(&b, &rowmax2, 8);
        cur_base = (int)(b >> 52) + 32;   // bin 0: >= 2^32 rowmax2 (and everything larger)
    }

    // eliminate final positions < min(F, i) in increasing order as F advances, at most
    // max_elims of them.  Positions only change through column exchanges (step s exchanges
    // s and t >= s >= F), which bump swap_version before the frontier moves on (logging the
    // two positions); the two bits of every exchange seen are then re-derived.
    int advance(int64_t max_elims) {
        // after a breakdown some rows are drained unpublished: never eliminate against them
        if (S.error_row.load(std::memory_order_acquire) >= 0) return kError;
        const int64_t f = S.front.load(std::memory_order_acquire);
        const int64_t ver = S.swap_version.load(std::memory_order_acquire);
        if (ver != my_version) {
            if (snapped) drop_snapshot();
            // exchange v swapped positions s and t (both >= the frontier then, so >=
            // cursor): re-derive those two bits from the columns now there.  This also
            // repairs a fill bit set from a position read while the exchange was under
            // way; later exchanges re-derive their own positions when they are seen.
            for (int64_t v = my_version; v < ver; v++) {
                for (const int64_t pp : {S.swap_log[v].first, S.swap_log[v].second}) {
                    if (pp < cursor) continue;
                    if (present[S.perm[pp].load(std::memory_order_relaxed)]) setbit(pp);
                    else bt[pp >> 6] &= ~(1ull << (pp & 63));
                }
            }
            my_version = ver;
        }
        const int64_t lim = std::min(f, i);
        int64_t k = next_bit(bt, cursor, lim);
        if (k >= lim) {
            cursor = std::max(cursor, lim);
            if (S.error_row.load(std::memory_order_relaxed) >= 0) return kError;
            if (f >= i) return kReady;
            if (!snapped && f >= i - S.snap_ahead) {
                take_snapshot();
                return kWorked;
            }
            return kIdle;
        }
        const bool late = S.prof && f >= i - 1;
        const clk::time_point tl = late ? clk::now() : clk::time_point();
        for (int64_t done = 0; k < lim && done < max_elims; k = next_bit(bt, cursor, lim), done++) {
            cursor = k + 1;
            const int64_t ck = S.perm[k].load(std::memory_order_relaxed);
            const RowRef& U = S.Urow[k];
            const double2 ukk = U.v[0];
            const double d = ukk.x * ukk.x + ukk.y * ukk.y;
            const double2 inv = make_double2(ukk.x / d, -ukk.y / d);
            const double2 wk0 = w[ck];
            const double2 wk = make_double2(wk0.x * inv.x - wk0.y * inv.y, wk0.x * inv.y + wk0.y * inv.x);
            if (mag2(wk) < tau2) {
                w[ck] = make_double2(0.0, 0.0);
                continue;
            }
            w[ck] = wk;
            lbuf.push_back(Ent{k, ck, wk, mag2(wk)});
            if (snapped) update_row<true>(U, wk);
            else update_row<false>(U, wk);
        }
        if (k >= lim) cursor = std::max(cursor, lim);
        if (late) p_late += ns_between(tl, clk::now());
        return kWorked;
    }

    // F == i: cap, pivot and publish U row i, then (off the critical path) the L row
    void finish(Arena& La, Arena& Ua, uint32_t& spins) {
        const double pt2 = S.permtol * S.permtol;
        // wait until every earlier row is published (then nobody else exchanges columns)
        const clk::time_point tp1 = S.prof ? clk::now() : clk::time_point();
        while (S.front.load(std::memory_order_acquire) < i) {
            if (S.error_row.load(std::memory_order_relaxed) >= 0) break;
            SSB_BACKOFF(spins);
        }
        const clk::time_point tp2 = S.prof ? clk::now() : clk::time_point();
        if (S.error_row.load(std::memory_order_relaxed) >= 0) {   // drain after a breakdown
            for (int64_t c : nz) {
                present[c] = 0;
                w[c] = make_double2(0.0, 0.0);
            }
            clear_bits();
            drop_snapshot();
            // nothing is published (no null rows, no frontier move): every waiter and every
            // advance() leaves on error_row
            active = false;
            return;
        }

        // U part: the row's positions > i (current: no exchange is pending now).  With a
        // snapshot (kept current by update_row since) nothing is re-read.
        const clk::time_point tq0 = S.prof ? clk::now() : clk::time_point();
        const int64_t cdiag = S.perm[i].load(std::memory_order_relaxed);
        double2 di = present[cdiag] ? w[cdiag] : make_double2(0.0, 0.0);
        if (S.prof) p_snap += snapped;
        if (!snapped) take_snapshot();
        int64_t nkept = 0;
        for (int t = 0; t < kHB; t++) nkept += shist[t];
        const clk::time_point tq1 = S.prof ? clk::now() : clk::time_point();
        if (S.prof) p_kept += nkept;
        buf.clear();
        const size_t ns = s_m.size();
        const uint8_t* sb = s_bin.data();
        if (nkept <= lfil) {
            for (size_t t = 0; t < ns; t++)
                if (sb[t] != kNotKept) buf.push_back(Ent{s_pos[t], s_col[t], w[s_col[t]], s_m[t]});
        } else if (lfil > 0) {   // keep the lfil largest (ties: smaller position)
            int hb = 0;
            int64_t above = 0;
            while (above + shist[hb] < lfil) above += shist[hb++];
            mk.clear();
            for (size_t t = 0; t < ns; t++)
                if (sb[t] == hb) mk.push_back(s_m[t]);
            const int64_t r = lfil - above;   // 1 <= r <= shist[hb]
            std::nth_element(mk.begin(), mk.begin() + (r - 1), mk.end(), std::greater<double>());
            const double mth = mk[r - 1];
            ties.clear();
            for (size_t t = 0; t < ns; t++) {   // bins < hb: larger than anything in hb
                if (sb[t] < hb) {
                    buf.push_back(Ent{s_pos[t], s_col[t], w[s_col[t]], s_m[t]});
                } else if (sb[t] == hb) {
                    const double m = s_m[t];
                    if (m > mth) buf.push_back(Ent{s_pos[t], s_col[t], w[s_col[t]], m});
                    else if (m == mth) ties.push_back((int32_t)t);
                }
            }
            const int64_t need = lfil - (int64_t)buf.size();
            if ((int64_t)ties.size() > need) {
                std::sort(ties.begin(), ties.end(), [&](int32_t x, int32_t y) { return s_pos[x] < s_pos[y]; });
                ties.resize(need);
            }
            for (int32_t t : ties) buf.push_back(Ent{s_pos[t], s_col[t], w[s_col[t]], s_m[t]});
        }
        if (S.prof) {
            const auto tq2 = clk::now();
            p_fcand += ns_between(tq0, tq1);
            p_fsel += ns_between(tq1, tq2);
        }
        // pivot: largest kept entry (ties: smaller position) against the diagonal
        int64_t tb = -1;
        double mb = -1.0;
        for (int64_t t = 0; t < (int64_t)buf.size(); t++)
            if (buf[t].m > mb || (buf[t].m == mb && buf[t].j < buf[tb].j)) {
                mb = buf[t].m;
                tb = t;
            }
        int64_t cnew = cdiag;
        if (tb >= 0 && pt2 * mb > mag2(di)) {
            const int64_t tpos = buf[tb].j, ct = buf[tb].c;
            const double2 old = di;
            di = buf[tb].v;
            cnew = ct;
            S.perm[i].store(ct, std::memory_order_relaxed);
            S.perm[tpos].store(cdiag, std::memory_order_relaxed);
            S.iperm[ct].store(i, std::memory_order_relaxed);
            S.iperm[cdiag].store(tpos, std::memory_order_relaxed);
            const int64_t v = S.swap_version.load(std::memory_order_relaxed);   // one writer at a time
            S.swap_log[v] = {i, tpos};
            S.swap_version.store(v + 1, std::memory_order_release);
            if (old.x != 0.0 || old.y != 0.0) {
                buf[tb] = Ent{tpos, cdiag, old, mag2(old)};
            } else {
                buf[tb] = buf.back();
                buf.pop_back();
            }
            S.swaps.fetch_add(1, std::memory_order_relaxed);
        }
        if (di.x == 0.0 && di.y == 0.0) {
            if (tau2 == 0.0) {
                int expected = -1;
                S.error_row.compare_exchange_strong(expected, (int)i);
            }
            di = make_double2(S.drop_tol * std::sqrt(rowmax2), 0.0);
            S.repaired.fetch_add(1, std::memory_order_relaxed);
        }
        {   // publish U row i in any order (consumers scatter by column; assembly sorts)
            int32_t* c;
            double2* v;
            Ua.reserve((int64_t)buf.size() + 1, c, v);
            c[0] = (int32_t)cnew;
            v[0] = di;
            for (size_t t = 0; t < buf.size(); t++) {
                c[t + 1] = (int32_t)buf[t].c;
                v[t + 1] = buf[t].v;
            }
            S.Urow[i] = RowRef{c, v, (int64_t)buf.size() + 1};
        }
        S.front.store(i + 1, std::memory_order_release);
        const clk::time_point tp3 = S.prof ? clk::now() : clk::time_point();
        // off the critical path (later rows need only U rows)
        // L part: multipliers kept, nonzero, above the threshold; cap; by position
        // (lbuf is in elimination order = ascending position; w at eliminated positions is
        // final, so e.v / e.m are the values the serial algorithm caps)
        buf.clear();
        for (const Ent& e : lbuf)
            if (e.m != 0.0 && !(e.m < tau2)) buf.push_back(e);
        if ((int64_t)buf.size() > lfil) {   // lfil largest, ties: smaller position (= earlier)
            if (lfil == 0) {
                buf.clear();
            } else {
                km.clear();
                for (const Ent& e : buf) km.push_back(e.m);
                const double mth = kth_largest(km.data(), km.size(), lfil, mk);
                int64_t need = lfil;
                for (const Ent& e : buf) need -= e.m > mth;
                size_t o = 0;
                for (size_t t = 0; t < buf.size(); t++) {
                    const Ent& e = buf[t];
                    if (e.m > mth || (e.m == mth && need-- > 0)) buf[o++] = e;
                }
                buf.resize(o);
            }
        }
        {
            int32_t* c;
            double2* v;
            La.reserve((int64_t)buf.size(), c, v);
            for (size_t t = 0; t < buf.size(); t++) {
                c[t] = (int32_t)buf[t].j;
                v[t] = buf[t].v;
            }
            S.Lrow[i] = RowRef{c, v, (int64_t)buf.size()};
        }
        // (w needs no clearing: every read of w is of a present column, and a column becomes
        // present by an assignment -- the row of A or a zero for new fill)
        for (int64_t c : nz) present[c] = 0;
        Ua.prefault(4096);
        if (S.prof) p_cand += hi - i;   // span of the U part (positions)
        clear_bits();
        drop_snapshot();
        if (S.prof) {
            p_post += ns_between(tp3, clk::now());
            p_lcand += (int64_t)lbuf.size();
            p_elim += ns_between(tp0, tp1);
            p_wait += ns_between(tp1, tp2);
            p_fin += ns_between(tp2, tp3);
        }
        active = false;
    }

    void flush_profile(int64_t spin) {
        if (!S.prof) return;
        S.t_elim += p_elim - spin;
        S.t_spin += spin;
        S.t_wait += p_wait;
        S.t_fin += p_fin;
        S.n_late += p_late;
        S.t_post += p_post;
        S.n_cand += p_cand;
        S.n_lcand += p_lcand;
        S.t_fcand += p_fcand;
        S.t_fsel += p_fsel;
        S.n_kept += p_kept;
        S.n_snap += p_snap;
    }
};

// A thread owns the row it will publish next (pri) and, while pri waits for the frontier,
// works ahead on the next row it claims (sec), a few eliminations at a time so that pri
// is served as soon as the frontier reaches it.  Rows are claimed in increasing order, so
// the row at the frontier is always some thread's pri (no deadlock).
void worker(Shared& S, Arena& La, Arena& Ua) {
    const int rows_per_thread = S.rows_per_thread;
    std::unique_ptr<RowWork> A(new RowWork(S)), B(rows_per_thread > 1 ? new RowWork(S) : nullptr);
    RowWork* pri = A.get();
    RowWork* sec = B.get();
    auto claim = [&](RowWork* r) {
        const int64_t row = S.next.fetch_add(1, std::memory_order_relaxed);
        if (row >= S.n) return false;
        r->begin(row);
        return true;
    };
    uint32_t spins = 0;
    int64_t p_spin = 0;
    bool more = claim(pri);
    while (pri->active) {
        const int st = pri->advance(INT64_MAX);
        if (st == RowWork::kReady || st == RowWork::kError) {
            pri->finish(La, Ua, spins);
            spins = 0;
            if (sec && sec->active) std::swap(pri, sec);
            else if (more) more = claim(pri);
            continue;
        }
        if (st == RowWork::kWorked) continue;
        // pri idle: work ahead on the next row
        if (sec && !sec->active && more) more = claim(sec);
        if (sec && sec->active && sec->advance(2) == RowWork::kWorked) continue;
        if (S.prof) {
            const auto a = clk::now();
            SSB_BACKOFF(spins);
            p_spin += ns_between(a, clk::now());
        } else {
            SSB_BACKOFF(spins);
        }
    }
    A->flush_profile(p_spin);
    if (B) B->flush_profile(0);
}

}  // namespace

void ilut_factor(const HostCSR& A, double drop_tol, double fill_factor, double permtol, int threads, HostCSR& L,
                 HostCSR& U, std::vector<int64_t>& colperm, IlutStats& st) {
    const int64_t n = A.n;
    SSB_CHECK(n < (int64_t)INT32_MAX, SS_ERR_ARG, "ILUT: n must be < 2^31");
    SSB_CHECK(drop_tol >= 0.0 && fill_factor >= 0.0 && permtol >= 0.0, SS_ERR_ARG,
              "drop_tol, fill_factor and permtol must be >= 0");
    // the frontier hand-off spins: never more threads than cores (oversubscribed, a waiting
    // thread can hold the core the row owner needs -- measured 27x slower at 24 on 16)
    const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
    const int cap = std::getenv("SSB_ILUT_MAXTHREADS") ? std::max(1, std::atoi(std::getenv("SSB_ILUT_MAXTHREADS"))) : hw;
    if (threads <= 0) threads = hw;
    if (threads > cap) threads = cap;
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n / 64));
    Shared S(A);
    S.drop_tol = drop_tol;
    S.fill_factor = fill_factor;
    S.permtol = permtol;
    S.n = n;
    S.prof = std::getenv("SSB_ILUT_PROF") != nullptr;
    if (const char* e = std::getenv("SSB_ILUT_SNAP")) S.snap_ahead = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("SSB_ILUT_ROWS")) S.rows_per_thread = std::max(1, std::min(2, std::atoi(e)));
    const auto tw0 = std::chrono::steady_clock::now();
    S.swap_log.reset(new std::pair<int64_t, int64_t>[n + 1]);   // at most one exchange per row
    S.perm.reset(new std::atomic<int64_t>[n]);
    S.iperm.reset(new std::atomic<int64_t>[n]);
    for (int64_t c = 0; c < n; c++) {
        S.perm[c].store(c, std::memory_order_relaxed);
        S.iperm[c].store(c, std::memory_order_relaxed);
    }
    S.Lrow.assign(n, RowRef{});
    S.Urow.assign(n, RowRef{});
    std::vector<Arena> La(threads), Ua(threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; t++) pool.emplace_back(worker, std::ref(S), std::ref(La[t]), std::ref(Ua[t]));
    worker(S, La[0], Ua[0]);
    for (auto& th : pool) th.join();
    if (S.prof) {
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - tw0).count();
        std::fprintf(stderr,
                     "ilut prof: n %lld threads %d wall %.3f s | per row (us): elim %.2f spin %.2f "
                     "wait %.2f finish %.2f (U candidates %.2f cap %.2f) post %.2f | eliminations after F >= i-1 %.2f | "
                     "U span %.0f kept %.0f, L %.0f | snapshot rows %.3f\n",
                     (long long)n, threads, wall, S.t_elim * 1e-3 / n, S.t_spin * 1e-3 / n, S.t_wait * 1e-3 / n,
                     S.t_fin * 1e-3 / n, S.t_fcand * 1e-3 / n, S.t_fsel * 1e-3 / n, S.t_post * 1e-3 / n,
                     S.n_late * 1e-3 / n, (double)S.n_cand / n, (double)S.n_kept / n, (double)S.n_lcand / n,
                     (double)S.n_snap / n);
    }
    const int bad = S.error_row.load();
    SSB_CHECK(bad < 0, SS_ERR_BREAKDOWN, "ILUT: zero pivot at row " + std::to_string(bad) + " with drop_tol = 0");
    colperm.resize(n);
    for (int64_t p = 0; p < n; p++) colperm[p] = S.perm[p].load(std::memory_order_relaxed);
    // assemble CSR in row order; U from original columns to final positions (strict part
    // re-sorted by position, diagonal first)
    L.n = U.n = n;
    L.rowptr.assign(n + 1, 0);
    U.rowptr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; i++) {
        L.rowptr[i + 1] = L.rowptr[i] + S.Lrow[i].len;
        U.rowptr[i + 1] = U.rowptr[i] + S.Urow[i].len;
    }
    L.col.resize(L.rowptr[n]);
    L.val.resize(L.rowptr[n]);
    U.col.resize(U.rowptr[n]);
    U.val.resize(U.rowptr[n]);
    std::vector<std::thread> asm_pool;
    const int nt = std::max(1, threads);
    for (int t = 0; t < nt; t++)
        asm_pool.emplace_back([&, t] {
            std::vector<std::pair<int64_t, double2>> tmp;
            for (int64_t i = n * t / nt; i < n * (t + 1) / nt; i++) {
                for (int64_t q = 0; q < S.Lrow[i].len; q++) L.col[L.rowptr[i] + q] = S.Lrow[i].c[q];
                std::memcpy(&L.val[L.rowptr[i]], S.Lrow[i].v, S.Lrow[i].len * sizeof(double2));
                const RowRef& R = S.Urow[i];
                const int64_t o = U.rowptr[i];
                if (R.len == 0) continue;
                U.col[o] = S.iperm[R.c[0]].load(std::memory_order_relaxed);
                U.val[o] = R.v[0];
                // published in position order of step i; a later exchange may have moved some
                bool sorted = true;
                int64_t prev = -1;
                for (int64_t q = 1; q < R.len; q++) {
                    const int64_t pq = S.iperm[R.c[q]].load(std::memory_order_relaxed);
                    U.col[o + q] = pq;
                    U.val[o + q] = R.v[q];
                    sorted &= pq > prev;
                    prev = pq;
                }
                if (sorted) continue;
                tmp.clear();
                for (int64_t q = 1; q < R.len; q++) tmp.emplace_back(U.col[o + q], U.val[o + q]);
                std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
                for (size_t q = 0; q < tmp.size(); q++) {
                    U.col[o + 1 + q] = tmp[q].first;
                    U.val[o + 1 + q] = tmp[q].second;
                }
            }
        });
    for (auto& th : asm_pool) th.join();
    st.repaired = S.repaired.load();
    st.swaps = S.swaps.load();
    st.threads = threads;
}

}  // namespace ssb
