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
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>

#if defined(__x86_64__)
#include <immintrin.h>
#define SSB_PAUSE() _mm_pause()
#else
#define SSB_PAUSE() std::this_thread::yield()
#endif

#include "problem.h"

namespace ssb {

namespace {

inline double mag2(double2 z) { return z.x * z.x + z.y * z.y; }

// append-only storage whose blocks never move (other threads read published rows)
struct Arena {
    static constexpr int64_t kBlock = 1 << 20;
    std::vector<std::unique_ptr<int64_t[]>> cblocks;
    std::vector<std::unique_ptr<double2[]>> vblocks;
    int64_t used = kBlock;
    void reserve(int64_t len, int64_t*& c, double2*& v) {
        if (cblocks.empty() || used + len > kBlock) {
            int64_t sz = std::max(kBlock, len);
            cblocks.emplace_back(new int64_t[sz]);
            vblocks.emplace_back(new double2[sz]);
            used = 0;
        }
        c = cblocks.back().get() + used;
        v = vblocks.back().get() + used;
        used += len;
    }
};

struct RowRef {
    const int64_t* c = nullptr;
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
    std::unique_ptr<std::atomic<int64_t>[]> perm;     // position -> original column
    std::unique_ptr<std::atomic<int64_t>[]> iperm;    // original column -> position
    std::vector<RowRef> Lrow, Urow;                   // L: positions; U: original columns
    std::atomic<int> error_row{-1};
    std::atomic<int32_t> repaired{0}, swaps{0};
    explicit Shared(const HostCSR& a) : A(a) {}
};

void worker(Shared& S, Arena& La, Arena& Ua) {
    const int64_t n = S.n;
    std::vector<double2> w(n, make_double2(0.0, 0.0));   // indexed by ORIGINAL column
    std::vector<uint8_t> present(n, 0);
    std::vector<int64_t> nz, heap;
    std::vector<std::pair<int64_t, int64_t>> pending;   // min-heap of (position when keyed, column)
    std::vector<Ent> lbuf, buf;
    nz.reserve(4096);
    pending.reserve(4096);
    heap.reserve(4096);
    buf.reserve(4096);
    lbuf.reserve(4096);
    auto cmp_heap = [](int64_t a, int64_t b) { return a > b; };   // min-heap of positions
    auto cmp_pend = [](const std::pair<int64_t, int64_t>& a, const std::pair<int64_t, int64_t>& b) {
        return a.first > b.first;
    };
    auto by_mag = [](const Ent& a, const Ent& b) { return a.m > b.m || (a.m == b.m && a.j < b.j); };
    auto by_pos = [](const Ent& a, const Ent& b) { return a.j < b.j; };
    const double pt2 = S.permtol * S.permtol;

    for (;;) {
        const int64_t i = S.next.fetch_add(1, std::memory_order_relaxed);
        if (i >= n) break;
        const int64_t r0 = S.A.rowptr[i], r1 = S.A.rowptr[i + 1];
        const int64_t lfil = (int64_t)(S.fill_factor * (double)(r1 - r0) / 2.0);
        double rowmax2 = 0.0;
        nz.clear();
        pending.clear();
        heap.clear();
        lbuf.clear();
        for (int64_t q = r0; q < r1; q++) {
            const int64_t c = S.A.col[q];
            const double m = mag2(S.A.val[q]);
            if (m > rowmax2) rowmax2 = m;
            w[c] = S.A.val[q];
            present[c] = 1;
            nz.push_back(c);
            pending.emplace_back(S.iperm[c].load(std::memory_order_relaxed), c);
        }
        std::make_heap(pending.begin(), pending.end(), cmp_pend);
        int64_t my_version = -1;   // forces a re-key on the first pass
        const double tau2 = S.drop_tol * S.drop_tol * rowmax2;

        // eliminate final positions < min(F, i) in increasing order as F advances.  Pending
        // columns are keyed by their position; positions only change through column
        // exchanges, which bump swap_version before the frontier moves on, so the keys are
        // refreshed only when that happens (rare).
        for (;;) {
            const int64_t f = S.front.load(std::memory_order_acquire);
            const int64_t ver = S.swap_version.load(std::memory_order_acquire);
            if (ver != my_version) {
                for (auto& e : pending) e.first = S.iperm[e.second].load(std::memory_order_relaxed);
                std::make_heap(pending.begin(), pending.end(), cmp_pend);
                my_version = ver;
            }
            const int64_t lim = std::min(f, i);
            while (!pending.empty() && pending.front().first < lim) {
                heap.push_back(pending.front().first);
                std::push_heap(heap.begin(), heap.end(), cmp_heap);
                std::pop_heap(pending.begin(), pending.end(), cmp_pend);
                pending.pop_back();
            }
            if (heap.empty()) {
                if (f >= i) break;
                if (S.error_row.load(std::memory_order_relaxed) >= 0) break;
                SSB_PAUSE();
                continue;
            }
            while (!heap.empty()) {
                std::pop_heap(heap.begin(), heap.end(), cmp_heap);
                const int64_t k = heap.back();
                heap.pop_back();
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
                for (int64_t q = 1; q < U.len; q++) {
                    const int64_t c = U.c[q];
                    const double2 u = U.v[q];
                    if (!present[c]) {
                        present[c] = 1;
                        w[c] = make_double2(0.0, 0.0);
                        nz.push_back(c);
                        const int64_t p = S.iperm[c].load(std::memory_order_relaxed);
                        if (p < lim) {
                            heap.push_back(p);
                            std::push_heap(heap.begin(), heap.end(), cmp_heap);
                        } else {
                            pending.emplace_back(p, c);
                            std::push_heap(pending.begin(), pending.end(), cmp_pend);
                        }
                    }
                    const double px = wk.x * u.x - wk.y * u.y;
                    const double py = wk.x * u.y + wk.y * u.x;
                    w[c].x = w[c].x - px;
                    w[c].y = w[c].y - py;
                }
            }
        }
        // wait until every earlier row is published (then nobody else exchanges columns)
        while (S.front.load(std::memory_order_acquire) < i) {
            if (S.error_row.load(std::memory_order_relaxed) >= 0) break;
            SSB_PAUSE();
        }
        if (S.error_row.load(std::memory_order_relaxed) >= 0) {   // drain after a breakdown
            for (int64_t c : nz) {
                present[c] = 0;
                w[c] = make_double2(0.0, 0.0);
            }
            S.Lrow[i] = RowRef{};
            S.Urow[i] = RowRef{};
            S.front.store(i + 1, std::memory_order_release);
            continue;
        }

        // L part: multipliers kept, nonzero, above the threshold; cap; by position
        buf.clear();
        for (const Ent& e : lbuf) {
            const double m = mag2(w[e.c]);
            if (m != 0.0 && !(m < tau2)) buf.push_back(Ent{e.j, e.c, w[e.c], m});
        }
        if ((int64_t)buf.size() > lfil) {
            std::nth_element(buf.begin(), buf.begin() + lfil, buf.end(), by_mag);
            buf.resize(lfil);
        }
        std::sort(buf.begin(), buf.end(), by_pos);
        {
            int64_t* c;
            double2* v;
            La.reserve((int64_t)buf.size(), c, v);
            for (size_t t = 0; t < buf.size(); t++) {
                c[t] = buf[t].j;
                v[t] = buf[t].v;
            }
            S.Lrow[i] = RowRef{c, v, (int64_t)buf.size()};
        }
        // U part: positions > i (pending holds exactly the columns at positions >= i)
        const int64_t cdiag = S.perm[i].load(std::memory_order_relaxed);
        double2 di = present[cdiag] ? w[cdiag] : make_double2(0.0, 0.0);
        buf.clear();
        for (const auto& e : pending) {
            const int64_t c = e.second;
            if (c == cdiag) continue;
            const double m = mag2(w[c]);
            if (m != 0.0 && !(m < tau2)) buf.push_back(Ent{S.iperm[c].load(std::memory_order_relaxed), c, w[c], m});
        }
        if ((int64_t)buf.size() > lfil) {
            std::nth_element(buf.begin(), buf.begin() + lfil, buf.end(), by_mag);
            buf.resize(lfil);
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
            S.swap_version.fetch_add(1, std::memory_order_release);
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
        std::sort(buf.begin(), buf.end(), by_pos);
        {
            int64_t* c;
            double2* v;
            Ua.reserve((int64_t)buf.size() + 1, c, v);
            c[0] = cnew;
            v[0] = di;
            for (size_t t = 0; t < buf.size(); t++) {
                c[t + 1] = buf[t].c;
                v[t + 1] = buf[t].v;
            }
            S.Urow[i] = RowRef{c, v, (int64_t)buf.size() + 1};
        }
        for (int64_t c : nz) {
            present[c] = 0;
            w[c] = make_double2(0.0, 0.0);
        }
        S.front.store(i + 1, std::memory_order_release);
    }
}

}  // namespace

void ilut_factor(const HostCSR& A, double drop_tol, double fill_factor, double permtol, int threads, HostCSR& L,
                 HostCSR& U, std::vector<int64_t>& colperm, IlutStats& st) {
    const int64_t n = A.n;
    SSB_CHECK(drop_tol >= 0.0 && fill_factor >= 0.0 && permtol >= 0.0, SS_ERR_ARG,
              "drop_tol, fill_factor and permtol must be >= 0");
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n / 64));
    Shared S(A);
    S.drop_tol = drop_tol;
    S.fill_factor = fill_factor;
    S.permtol = permtol;
    S.n = n;
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
                std::memcpy(&L.col[L.rowptr[i]], S.Lrow[i].c, S.Lrow[i].len * sizeof(int64_t));
                std::memcpy(&L.val[L.rowptr[i]], S.Lrow[i].v, S.Lrow[i].len * sizeof(double2));
                const RowRef& R = S.Urow[i];
                const int64_t o = U.rowptr[i];
                if (R.len == 0) continue;
                U.col[o] = S.iperm[R.c[0]].load(std::memory_order_relaxed);
                U.val[o] = R.v[0];
                tmp.clear();
                for (int64_t q = 1; q < R.len; q++)
                    tmp.emplace_back(S.iperm[R.c[q]].load(std::memory_order_relaxed), R.v[q]);
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
