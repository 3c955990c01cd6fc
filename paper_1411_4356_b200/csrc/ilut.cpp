// ilut.cpp -- dual-threshold incomplete LU of L~_RCM (setup, host, multi-threaded).
//
// PAPER.md:94 (sec. II): "an incomplete LU factorization with dual-threshold ... a drop
// tolerance d and allowed fill-in p are specified such that all fill-in smaller than d
// times the infinity-norm of a row are dropped, and at most only p NNZ(L~) fill-in
// elements are allowed".  Row-wise (IKJ) ILUT as in the paper's reference [saad:2003];
// the exact rules (R4-R7 in DESIGN.md):
//   tau_i = d * max_j |a_ij|; a value z is dropped iff |z|^2 < tau_i^2;
//   multiplier w_k <- w_k * (1/u_kk), 1/u = (ur, -ui)/(ur^2+ui^2), dropped by the same
//   test before it is used; update w_j <- w_j - w_k u_kj (no FMA: -ffp-contract=off);
//   after elimination the L part and the strict U part of the row each keep at most
//   floor(p * nnz(a_i) / 2) entries of largest |.|^2 (ties: smaller column);
//   the diagonal is never dropped, an exactly-zero pivot becomes tau_i (error if 0).
//
// B200-first change vs. a serial ILUT: rows are factorised by a pool of host threads
// in a software pipeline.  Row i only needs the finished U rows k < i that appear in
// its elimination, so a thread claims the next row from an atomic counter and spins
// on the per-row "published" flag of each U row it consumes.  Rows are claimed in
// increasing order, hence every awaited row is already owned by a running thread (no
// deadlock), and the arithmetic of every row is identical to the serial algorithm
// (same operands, same order) -- the factors are bit-identical for any thread count.
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
    int64_t total = 0;
    // reserve len contiguous slots; returns pointers
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
        total += len;
    }
};

struct RowRef {
    const int64_t* c = nullptr;
    const double2* v = nullptr;
    int64_t len = 0;
};

struct Ent {
    int64_t j;
    double2 v;
    double m;
};

struct Shared {
    const HostCSR& A;
    double drop_tol, fill_factor;
    int64_t n;
    std::atomic<int64_t> next{0};
    std::unique_ptr<std::atomic<uint8_t>[]> ready;
    std::vector<RowRef> Lrow, Urow;
    std::atomic<int> error_row{-1};
    std::atomic<int32_t> repaired{0};
    explicit Shared(const HostCSR& a) : A(a) {}
};

void worker(Shared& S, Arena& La, Arena& Ua) {
    const int64_t n = S.n;
    std::vector<double2> w(n, make_double2(0.0, 0.0));
    std::vector<uint8_t> present(n, 0);
    std::vector<int64_t> nz;
    nz.reserve(4096);
    std::vector<int64_t> heap;
    heap.reserve(4096);
    std::vector<Ent> buf;
    buf.reserve(4096);
    auto cmp_heap = [](int64_t a, int64_t b) { return a > b; };   // min-heap
    auto by_mag = [](const Ent& a, const Ent& b) { return a.m > b.m || (a.m == b.m && a.j < b.j); };
    auto by_col = [](const Ent& a, const Ent& b) { return a.j < b.j; };

    for (;;) {
        const int64_t i = S.next.fetch_add(1, std::memory_order_relaxed);
        if (i >= n) break;
        if (S.error_row.load(std::memory_order_relaxed) >= 0) {   // drain: publish empty rows
            S.ready[i].store(1, std::memory_order_release);
            continue;
        }
        const int64_t r0 = S.A.rowptr[i], r1 = S.A.rowptr[i + 1];
        const int64_t lfil = (int64_t)(S.fill_factor * (double)(r1 - r0) / 2.0);
        double rowmax2 = 0.0;
        nz.clear();
        heap.clear();
        for (int64_t q = r0; q < r1; q++) {
            const int64_t j = S.A.col[q];
            const double m = mag2(S.A.val[q]);
            if (m > rowmax2) rowmax2 = m;
            w[j] = S.A.val[q];
            present[j] = 1;
            nz.push_back(j);
            if (j < i) {
                heap.push_back(j);
                std::push_heap(heap.begin(), heap.end(), cmp_heap);
            }
        }
        if (!present[i]) {
            present[i] = 1;
            w[i] = make_double2(0.0, 0.0);
            nz.push_back(i);
        }
        const double tau2 = S.drop_tol * S.drop_tol * rowmax2;

        while (!heap.empty()) {
            std::pop_heap(heap.begin(), heap.end(), cmp_heap);
            const int64_t k = heap.back();
            heap.pop_back();
            while (!S.ready[k].load(std::memory_order_acquire)) SSB_PAUSE();
            const RowRef& U = S.Urow[k];
            if (U.len == 0) continue;   // only during error drain
            const double2 ukk = U.v[0];
            const double d = ukk.x * ukk.x + ukk.y * ukk.y;
            const double2 inv = make_double2(ukk.x / d, -ukk.y / d);
            const double2 wk0 = w[k];
            const double2 wk = make_double2(wk0.x * inv.x - wk0.y * inv.y, wk0.x * inv.y + wk0.y * inv.x);
            if (mag2(wk) < tau2) {
                w[k] = make_double2(0.0, 0.0);
                continue;
            }
            w[k] = wk;
            for (int64_t q = 1; q < U.len; q++) {
                const int64_t j = U.c[q];
                const double2 u = U.v[q];
                if (!present[j]) {
                    present[j] = 1;
                    w[j] = make_double2(0.0, 0.0);
                    nz.push_back(j);
                    if (j < i) {
                        heap.push_back(j);
                        std::push_heap(heap.begin(), heap.end(), cmp_heap);
                    }
                }
                const double px = wk.x * u.x - wk.y * u.y;
                const double py = wk.x * u.y + wk.y * u.x;
                w[j].x = w[j].x - px;
                w[j].y = w[j].y - py;
            }
        }

        // L part
        buf.clear();
        for (int64_t j : nz)
            if (j < i) {
                const double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) buf.push_back(Ent{j, w[j], m});
            }
        if ((int64_t)buf.size() > lfil) {
            std::nth_element(buf.begin(), buf.begin() + lfil, buf.end(), by_mag);
            buf.resize(lfil);
        }
        std::sort(buf.begin(), buf.end(), by_col);
        {
            int64_t* c;
            double2* v;
            La.reserve((int64_t)buf.size(), c, v);
            for (size_t t = 0; t < buf.size(); t++) { c[t] = buf[t].j; v[t] = buf[t].v; }
            S.Lrow[i] = RowRef{c, v, (int64_t)buf.size()};
        }
        // diagonal
        double2 di = w[i];
        if (di.x == 0.0 && di.y == 0.0) {
            if (tau2 == 0.0) {
                int expected = -1;
                S.error_row.compare_exchange_strong(expected, (int)i);
            }
            di = make_double2(S.drop_tol * std::sqrt(rowmax2), 0.0);
            S.repaired.fetch_add(1, std::memory_order_relaxed);
        }
        // strict U part
        buf.clear();
        for (int64_t j : nz)
            if (j > i) {
                const double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) buf.push_back(Ent{j, w[j], m});
            }
        if ((int64_t)buf.size() > lfil) {
            std::nth_element(buf.begin(), buf.begin() + lfil, buf.end(), by_mag);
            buf.resize(lfil);
        }
        std::sort(buf.begin(), buf.end(), by_col);
        {
            int64_t* c;
            double2* v;
            Ua.reserve((int64_t)buf.size() + 1, c, v);
            c[0] = i;
            v[0] = di;
            for (size_t t = 0; t < buf.size(); t++) { c[t + 1] = buf[t].j; v[t + 1] = buf[t].v; }
            S.Urow[i] = RowRef{c, v, (int64_t)buf.size() + 1};
        }
        S.ready[i].store(1, std::memory_order_release);
        for (int64_t j : nz) {
            present[j] = 0;
            w[j] = make_double2(0.0, 0.0);
        }
    }
}

}  // namespace

void ilut_factor(const HostCSR& A, double drop_tol, double fill_factor, int threads, HostCSR& L, HostCSR& U,
                 IlutStats& st) {
    const int64_t n = A.n;
    SSB_CHECK(drop_tol >= 0.0 && fill_factor >= 0.0, SS_ERR_ARG, "drop_tol and fill_factor must be >= 0");
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    threads = (int)std::min<int64_t>(threads, std::max<int64_t>(1, n / 64));
    Shared S(A);
    S.drop_tol = drop_tol;
    S.fill_factor = fill_factor;
    S.n = n;
    S.ready.reset(new std::atomic<uint8_t>[n]);
    for (int64_t i = 0; i < n; i++) S.ready[i].store(0, std::memory_order_relaxed);
    S.Lrow.assign(n, RowRef{});
    S.Urow.assign(n, RowRef{});
    std::vector<Arena> La(threads), Ua(threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; t++) pool.emplace_back(worker, std::ref(S), std::ref(La[t]), std::ref(Ua[t]));
    worker(S, La[0], Ua[0]);
    for (auto& th : pool) th.join();
    const int bad = S.error_row.load();
    SSB_CHECK(bad < 0, SS_ERR_BREAKDOWN,
              "ILUT: zero pivot at row " + std::to_string(bad) + " with drop_tol = 0");
    // assemble CSR in row order
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
    for (int64_t i = 0; i < n; i++) {
        std::memcpy(&L.col[L.rowptr[i]], S.Lrow[i].c, S.Lrow[i].len * sizeof(int64_t));
        std::memcpy(&L.val[L.rowptr[i]], S.Lrow[i].v, S.Lrow[i].len * sizeof(double2));
        std::memcpy(&U.col[U.rowptr[i]], S.Urow[i].c, S.Urow[i].len * sizeof(int64_t));
        std::memcpy(&U.val[U.rowptr[i]], S.Urow[i].v, S.Urow[i].len * sizeof(double2));
    }
    st.repaired = S.repaired.load();
    st.threads = threads;
}

}  // namespace ssb
