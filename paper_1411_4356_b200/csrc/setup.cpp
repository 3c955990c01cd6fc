// setup.cpp -- one-time setup of a built Liouvillian: RCM order, permuted L~_RCM,
// ILUT factors, substitution schedules and their device layout (timed separately from
// the GMRES hot path, as the north star asks).
//
// sec. III: RCM of L~ + L~^T applied as a symmetric permutation;
// sec. II: bandwidth B = ub + lb + 1 reported before / after;
// sec. II: ILUT(d, p).
#include <algorithm>
#include <chrono>
#include <exception>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "problem.h"

namespace ssb {

namespace {

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

int64_t bandwidth(const HostCSR& A) {
    int64_t ub = 0, lb = 0;
    for (int64_t i = 0; i < A.n; i++)
        for (int64_t q = A.rowptr[i]; q < A.rowptr[i + 1]; q++) {
            int64_t d = A.col[q] - i;
            ub = std::max(ub, d);
            lb = std::max(lb, -d);
        }
    return ub + lb + 1;
}

void download(const DevCSR& D, HostCSR& H, cudaStream_t s) {
    H.n = D.n;
    H.rowptr.resize(D.n + 1);
    std::vector<int32_t> c32(D.nnz);
    H.val.resize(D.nnz);
    SSB_CUDA(cudaMemcpyAsync(H.rowptr.data(), D.rowptr, (D.n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(c32.data(), D.col, D.nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaMemcpyAsync(H.val.data(), D.val, D.nnz * sizeof(double2), cudaMemcpyDeviceToHost, s));
    SSB_CUDA(cudaStreamSynchronize(s));
    H.col.assign(c32.begin(), c32.end());
}

void upload(const HostCSR& H, DevCSR& D, cudaStream_t s) {
    D.release();
    D.alloc_rowptr(H.n);
    D.alloc_entries(H.nnz());
    std::vector<int32_t> c32(H.col.begin(), H.col.end());
    SSB_CUDA(cudaMemcpyAsync(D.rowptr, H.rowptr.data(), (H.n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.col, c32.data(), c32.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.val, H.val.data(), H.val.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaStreamSynchronize(s));
}

// A_new[k][*] = A[perm[k]][perm^{-1}(*)], columns re-sorted
HostCSR permute(const HostCSR& A, const std::vector<int64_t>& perm) {
    const int64_t n = A.n;
    std::vector<int64_t> iperm(n);
    for (int64_t k = 0; k < n; k++) iperm[perm[k]] = k;
    HostCSR B;
    B.n = n;
    B.rowptr.assign(n + 1, 0);
    for (int64_t k = 0; k < n; k++) B.rowptr[k + 1] = B.rowptr[k] + (A.rowptr[perm[k] + 1] - A.rowptr[perm[k]]);
    B.col.resize(A.nnz());
    B.val.resize(A.nnz());
    std::vector<std::pair<int64_t, double2>> tmp;
    for (int64_t k = 0; k < n; k++) {
        const int64_t o = perm[k];
        tmp.clear();
        for (int64_t q = A.rowptr[o]; q < A.rowptr[o + 1]; q++) tmp.emplace_back(iperm[A.col[q]], A.val[q]);
        std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        int64_t p = B.rowptr[k];
        for (auto& e : tmp) {
            B.col[p] = e.first;
            B.val[p] = e.second;
            p++;
        }
    }
    return B;
}

// B = A^T, columns ascending in every row of B.  skip_first: leave out the first stored
// entry of every row of A (the diagonal of a diagonal-first U factor).
HostCSR transpose(const HostCSR& A, bool skip_first) {
    const int64_t n = A.n;
    HostCSR B;
    B.n = n;
    B.rowptr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; i++)
        for (int64_t q = A.rowptr[i] + (skip_first ? 1 : 0); q < A.rowptr[i + 1]; q++) B.rowptr[A.col[q] + 1]++;
    for (int64_t j = 0; j < n; j++) B.rowptr[j + 1] += B.rowptr[j];
    B.col.resize(B.rowptr[n]);
    B.val.resize(B.rowptr[n]);
    std::vector<int64_t> next(B.rowptr.begin(), B.rowptr.end() - 1);
    for (int64_t i = 0; i < n; i++)
        for (int64_t q = A.rowptr[i] + (skip_first ? 1 : 0); q < A.rowptr[i + 1]; q++) {
            const int64_t t = next[A.col[q]]++;
            B.col[t] = i;
            B.val[t] = A.val[q];
        }
    return B;
}

// B[j][*] = A[rows[j]][*] (rows reordered, columns unchanged)
HostCSR permute_rows(const HostCSR& A, const std::vector<int64_t>& rows) {
    const int64_t n = A.n;
    HostCSR B;
    B.n = n;
    B.rowptr.assign(n + 1, 0);
    for (int64_t j = 0; j < n; j++) B.rowptr[j + 1] = B.rowptr[j] + (A.rowptr[rows[j] + 1] - A.rowptr[rows[j]]);
    B.col.resize(A.nnz());
    B.val.resize(A.nnz());
    for (int64_t j = 0; j < n; j++) {
        const int64_t o = rows[j];
        std::copy(A.col.begin() + A.rowptr[o], A.col.begin() + A.rowptr[o + 1], B.col.begin() + B.rowptr[j]);
        std::copy(A.val.begin() + A.rowptr[o], A.val.begin() + A.rowptr[o + 1], B.val.begin() + B.rowptr[j]);
    }
    return B;
}

template <class Fn>
void parallel_for(int64_t n, int threads, Fn fn, int64_t grain = 1024) {
    threads = (int)std::max<int64_t>(1, std::min<int64_t>(threads, n / grain + 1));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; t++) {
        const int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        pool.emplace_back([=, &fn] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

void build_sell(const HostCSR& H, DevCSR& D, cudaStream_t s) {
    const int64_t n = H.n, ns = (n + 31) / 32;
    std::vector<int64_t> sptr(ns + 1, 0), lrows;
    for (int64_t sl = 0; sl < ns; sl++) {
        int64_t w = 1;
        for (int64_t r = sl * 32; r < std::min(n, sl * 32 + 32); r++) {
            const int64_t len = H.rowptr[r + 1] - H.rowptr[r];
            if (len > kSellLong) lrows.push_back(r);
            else w = std::max(w, len);
        }
        sptr[sl + 1] = sptr[sl] + 32 * w;
    }
    const int64_t tot = sptr[ns];
    hvec<int32_t> c(tot);
    hvec<double2> v(tot);
    const int threads = (int)std::max(1u, std::thread::hardware_concurrency());
    parallel_for(ns, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t sl = lo; sl < hi; sl++) {
            const int64_t w = (sptr[sl + 1] - sptr[sl]) / 32;
            for (int r = 0; r < 32; r++) {
                const int64_t i = sl * 32 + r;
                const int64_t len = i < n ? H.rowptr[i + 1] - H.rowptr[i] : 0;
                const bool lng = len > kSellLong;
                for (int64_t e = 0; e < w; e++) {
                    const int64_t t = sptr[sl] + 32 * e + r;
                    if (!lng && e < len) {
                        c[t] = (int32_t)H.col[H.rowptr[i] + e];
                        v[t] = H.val[H.rowptr[i] + e];
                    } else {
                        c[t] = (lng && e == 0) ? -1 : 0;
                        v[t] = make_double2(0.0, 0.0);
                    }
                }
            }
        }
    }, 256);
    D.nslices = ns;
    D.nlong = (int64_t)lrows.size();
    D.sell_entries = tot;
    SSB_CUDA(cudaMalloc(&D.sptr, (ns + 1) * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&D.scol, std::max<int64_t>(1, tot) * sizeof(int32_t)));
    SSB_CUDA(cudaMalloc(&D.sval, std::max<int64_t>(1, tot) * sizeof(double2)));
    SSB_CUDA(cudaMalloc(&D.lrows, std::max<int64_t>(1, D.nlong) * sizeof(int64_t)));
    SSB_CUDA(cudaMemcpyAsync(D.sptr, sptr.data(), (ns + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.scol, c.data(), tot * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(D.sval, v.data(), tot * sizeof(double2), cudaMemcpyHostToDevice, s));
    if (D.nlong)
        SSB_CUDA(cudaMemcpyAsync(D.lrows, lrows.data(), D.nlong * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaStreamSynchronize(s));
}

namespace {

// Row-level dependency levels of the substitution (diagnostic: the length of the
// chain a row-level schedule would walk).
int64_t count_levels(const HostCSR& F, bool upper) {   // F: strict triangle
    const int64_t n = F.n;
    std::vector<int32_t> lev(n, 0);
    int32_t maxl = 0;
    auto row = [&](int64_t i) {
        int32_t l = 0;
        for (int64_t q = F.rowptr[i]; q < F.rowptr[i + 1]; q++) l = std::max(l, lev[F.col[q]] + 1);
        lev[i] = l;
        maxl = std::max(maxl, l);
    };
    if (!upper)
        for (int64_t i = 0; i < n; i++) row(i);
    else
        for (int64_t i = n - 1; i >= 0; i--) row(i);
    return n ? (int64_t)maxl + 1 : 0;
}

// Block layout of one triangular factor for trsv.cu, given as its STRICT triangle F (CSR,
// columns ascending) and its diagonal (diag = nullptr: unit).  Kernel index space: a
// lower factor as is; an upper one reversed (i' = n-1-i), which turns it into a lower one.  Row i' of block k splits
// its strict entries (ascending kernel column) into "far" (source block <= k-Q), "near"
// (source blocks k-Q+1 .. k-1) and in-block.  Far entries form a CSR; the near entries
// of a block form one list (rows in order, start padded to 4 entries for TMA, row
// pointers relative to the block start); the in-block entries and the diagonal (1 for
// L, u_ii for U) form the dense block D_k, whose inverse is stored packed (lower,
// column-major; column j = rows j..B-1).  The last block is padded with identity rows.
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

void build_block_tri(const HostCSR& F, const double2* diag, bool upper, int B, int q_max, int threads,
                     DevBlockTri& T, cudaStream_t s) {
    T.release();
    const bool prof = std::getenv("SSB_SETUP_PROF") != nullptr;
    double tpf[8] = {now_ms()};
    double t_copy = 0;
    const int64_t n = F.n;
    const int64_t nblk = (n + B - 1) / B;
    const int64_t PK = (int64_t)block_trsv_packed(B);
    T.n = n;
    T.B = B;
    T.nblk = nblk;
    T.rev = upper ? 1 : 0;
    // strict entries of kernel row ip in ascending kernel column: for L the CSR row; for U
    // the reversed strict part of row n-1-ip.
    auto row_range = [&](int64_t ip, int64_t& q0, int64_t& q1) {
        const int64_t i = upper ? n - 1 - ip : ip;
        q0 = F.rowptr[i];
        q1 = F.rowptr[i + 1];
    };
    auto kcol = [&](int64_t q) -> int64_t { return upper ? n - 1 - F.col[q] : F.col[q]; };
    auto entry = [&](int64_t q0, int64_t q1, int64_t t) -> int64_t { return upper ? q1 - 1 - t : q0 + t; };

    // per row: entries per source distance d = k - source block (d = 1 .. kMaxQ-1; d >= kMaxQ
    // counted together); the near window Q (near = d < Q, far = d >= Q) is the largest
    // Q <= Qmax whose per-block near lists fit the shared-memory stage (kNearCap)
    constexpr int kMaxQ = 32;
    std::vector<int64_t> dcnt((size_t)n * kMaxQ, 0);   // [row][d], d = 0 means ">= kMaxQ"
    std::vector<int64_t> nin(n);                        // strict entries left of the block
    parallel_for(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t ip = lo; ip < hi; ip++) {
            int64_t q0, q1;
            row_range(ip, q0, q1);
            const int64_t k = ip / B, kb = k * B;
            int64_t c = 0;
            for (int64_t t = 0; t < q1 - q0; t++) {
                const int64_t j = kcol(entry(q0, q1, t));
                if (j >= kb) break;
                const int64_t d = k - j / B;
                dcnt[(size_t)ip * kMaxQ + (d < kMaxQ ? d : 0)]++;
                c++;
            }
            nin[ip] = c;
        }
    });
    // Split of the entries left of block k by source distance d (problem.h, trsv.cu):
    //   d = 1 .. kDense       -> dense G_d = D_k^{-1} T_{k,k-d} (the chain teams)
    //   kDense < d < Q_k      -> list B (the lieutenant CTAs of the chain's cluster; lieutenant
    //                            l holds the rows r = l mod kLieutenants of the block); the
    //                            d = kDense+1 entries of each row (the last ones) form its late part
    //   d >= Q_k              -> far (the helper CTAs)
    // Q_k is the largest Q <= Qmax (>= kDense+1) whose per-lieutenant lists fit their stages.
    // A row's entries in ascending column: far | list B (late part last) | G_kDense .. G_1 | block.
    constexpr int kD1 = kDense + 1;
    const int qmax = std::max(kD1, std::min(kMaxQ, q_max));
    // per-lieutenant entry budget of a block: the stage capacity, or less (SSB_TRSV_LTCAP) to
    // keep heavy blocks from making their lieutenants late (the rest goes to the helpers)
    const int ltcap = std::min(near_cap_b(B), env_int("SSB_TRSV_LTCAP", near_cap_b(B)));
    std::vector<int> qk(nblk, qmax);
    parallel_for(nblk, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; k++) {
            int q = qmax;
            for (; q > kD1; q--) {
                int64_t cb[kLieutenants] = {};
                for (int64_t ip = k * B; ip < std::min(n, (k + 1) * B); ip++)
                    for (int d = kD1; d < q; d++) cb[(ip - k * B) % kLieutenants] += dcnt[(size_t)ip * kMaxQ + d];
                bool fit = true;
                for (int l = 0; l < kLieutenants; l++) fit = fit && cb[l] + 3 <= ltcap;
                if (fit) break;
            }
            qk[k] = q;
        }
    }, 16);
    int qmin = qmax;
    for (int64_t k = 0; k < nblk; k++) qmin = std::min(qmin, qk[k]);
    T.Q = qmin;
    // per row: far / list B (its late part) / dense G_d entries
    std::vector<int64_t> cnt(n), bcnt(n), blate(n), gcnt((size_t)n * kDense);
    for (int64_t ip = 0; ip < n; ip++) {
        const int q = qk[ip / B];
        int64_t nbb = 0, ng = 0;
        for (int d = kD1; d < q; d++) nbb += dcnt[(size_t)ip * kMaxQ + d];
        for (int d = 1; d <= kDense; d++) ng += (gcnt[(size_t)ip * kDense + d - 1] = dcnt[(size_t)ip * kMaxQ + d]);
        bcnt[ip] = nbb;
        blate[ip] = q > kD1 ? dcnt[(size_t)ip * kMaxQ + kD1] : 0;
        cnt[ip] = nin[ip] - ng - nbb;
    }
    std::vector<int64_t>().swap(dcnt);
    std::vector<int64_t> farptr(n + 1, 0);
    for (int64_t i = 0; i < n; i++) farptr[i + 1] = farptr[i] + cnt[i];
    // list B: per (block, lieutenant) a padded start, per row a local pointer and the local
    // start of its late part
    struct NearHost {
        std::vector<int64_t> bp, row;   // list starts [nblk*G+1], global row starts [n]
        std::vector<int32_t> loc;       // [nblk*G][2(B+4)]
    };
    const int NL = near_nloc(B);
    auto layout = [&](const std::vector<int64_t>& c, const std::vector<int64_t>& late, int G, NearHost& H) {
        H.bp.assign(nblk * G + 1, 0);
        H.row.assign(n, 0);
        H.loc.assign((size_t)nblk * G * NL, 0);
        for (int64_t k = 0; k < nblk; k++)
            for (int g = 0; g < G; g++) {
                const int64_t idx = k * G + g;
                int32_t* loc = &H.loc[(size_t)idx * NL];
                int64_t off = 0;
                for (int r = 0; r < B; r++) {
                    const int64_t ip = k * B + r;
                    loc[r] = (int32_t)off;
                    loc[B + 4 + r] = (int32_t)off;
                    if (ip < n && r % G == g) {
                        H.row[ip] = H.bp[idx] + off;
                        off += c[ip];
                        loc[B + 4 + r] = (int32_t)(off - late[ip]);
                    }
                }
                for (int r = B; r < B + 4; r++) loc[r] = loc[B + 4 + r] = (int32_t)off;
                H.bp[idx + 1] = H.bp[idx] + ((off + 3) & ~(int64_t)3);
            }
    };
    constexpr int G = kLieutenants;
    NearHost HB;
    layout(bcnt, blate, G, HB);
    const int64_t nf = farptr[n], nB = HB.bp[nblk * G];
    T.nnz_far = nf;
    T.nnz_near = 0;
    for (int64_t i = 0; i < n; i++) T.nnz_near += nin[i] - cnt[i];
    T.nnz_strict = F.nnz();

    // far work items of each block for the helper CTAs: item (r, c) = far entries 32c ..
    // 32c+31 of the block's row r, keyed by the source block of its last (newest) entry and
    // sorted by that key (then c, r), so that a block's long rows are spread over all helper
    // warps and the items waiting for the newest x blocks come last
    static_assert(sizeof(uint32_t) == 4, "item encoding (c << 5) | r needs B = 32");
    SSB_CHECK(B == 32, SS_ERR_ARG, "far work items encode the row in 5 bits (B = 32)");
    std::vector<int64_t> itemptr(nblk + 1, 0);
    for (int64_t k = 0; k < nblk; k++) {
        int64_t c = 0;
        for (int64_t ip = k * B; ip < std::min(n, (k + 1) * B); ip++) c += (cnt[ip] + 31) / 32;
        itemptr[k + 1] = itemptr[k] + c;
    }
    hvec<uint32_t> items(std::max<int64_t>(1, itemptr[nblk]));
    parallel_for(nblk, threads, [&](int64_t lo, int64_t hi) {
        std::vector<std::pair<int64_t, uint32_t>> key;
        for (int64_t k = lo; k < hi; k++) {
            key.clear();
            for (int64_t ip = k * B; ip < std::min(n, (k + 1) * B); ip++) {
                int64_t q0, q1;
                row_range(ip, q0, q1);
                const uint32_t r = (uint32_t)(ip - k * B);
                for (int64_t c = 0; c * 32 < cnt[ip]; c++) {
                    const int64_t last = std::min(cnt[ip], 32 * c + 32) - 1;   // far entries lead the row
                    const int64_t src = kcol(entry(q0, q1, last)) / B;
                    key.emplace_back((src << 32) | (c << 5) | r, (uint32_t)((c << 5) | r));
                }
            }
            std::sort(key.begin(), key.end());
            for (size_t t = 0; t < key.size(); t++) items[itemptr[k] + t] = key[t].second;
        }
    }, 64);

    auto upload_near = [&](const NearHost& H, int64_t total, NearDev& D) {
        SSB_CUDA(cudaMalloc(&D.bp, H.bp.size() * sizeof(int64_t)));
        SSB_CUDA(cudaMalloc(&D.col, std::max<int64_t>(4, total) * sizeof(int32_t)));
        SSB_CUDA(cudaMalloc(&D.val, std::max<int64_t>(4, total) * sizeof(double2)));
        SSB_CUDA(cudaMalloc(&D.loc, H.loc.size() * sizeof(int32_t)));
        SSB_CUDA(cudaMemsetAsync(D.col, 0, std::max<int64_t>(4, total) * sizeof(int32_t), s));   // padding
        SSB_CUDA(cudaMemcpyAsync(D.bp, H.bp.data(), H.bp.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(D.loc, H.loc.data(), H.loc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    };
    SSB_CUDA(cudaMalloc(&T.farptr, (n + 1) * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&T.fcol, std::max<int64_t>(1, nf) * sizeof(int32_t)));
    SSB_CUDA(cudaMalloc(&T.fval, std::max<int64_t>(1, nf) * sizeof(double2)));
    upload_near(HB, nB, T.nearB);
    SSB_CUDA(cudaMalloc(&T.dinv, std::max<int64_t>(1, nblk * PK) * sizeof(double2)));

    SSB_CUDA(cudaMalloc(&T.G, std::max<int64_t>(1, nblk * kDense * B * B) * sizeof(double2)));
    SSB_CUDA(cudaMalloc(&T.yfar, std::max<int64_t>(1, nblk * B) * sizeof(double2)));
    SSB_CUDA(cudaMalloc(&T.fflag, std::max<int64_t>(1, nblk) * sizeof(uint32_t)));
    SSB_CUDA(cudaMalloc(&T.xfront, sizeof(unsigned long long)));
    SSB_CUDA(cudaMemsetAsync(T.fflag, 0, std::max<int64_t>(1, nblk) * sizeof(uint32_t), s));
    SSB_CUDA(cudaMemsetAsync(T.xfront, 0, sizeof(unsigned long long), s));
    SSB_CUDA(cudaMemcpyAsync(T.farptr, farptr.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMalloc(&T.itemptr, (nblk + 1) * sizeof(int64_t)));
    SSB_CUDA(cudaMalloc(&T.items, items.size() * sizeof(uint32_t)));
    SSB_CUDA(cudaMemcpyAsync(T.itemptr, itemptr.data(), (nblk + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(T.items, items.data(), items.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaStreamSynchronize(s));

    // entries, in block chunks of ~2^26 (bounded host staging); the rows of a chunk of
    // blocks map to contiguous ranges of the far CSR and of list B
    tpf[1] = now_ms();
    const int64_t kChunk = (int64_t)1 << 26;
    hvec<int32_t> fc, bc;   // filled in parallel below (no serial zeroing of GBs)
    hvec<double2> fv, bv;
    auto frow = [&](int64_t k) { return farptr[std::min(n, k * B)]; };
    for (int64_t k0 = 0; k0 < nblk;) {
        int64_t k1 = k0 + 1;
        while (k1 < nblk && (frow(k1 + 1) - frow(k0)) + (HB.bp[(k1 + 1) * G] - HB.bp[k0 * G]) <= kChunk)
            k1++;
        const int64_t r0 = k0 * B, r1 = std::min(n, k1 * B);
        const int64_t fb = farptr[r0], flen = farptr[r1] - fb;
        const int64_t bb = HB.bp[k0 * G], blen = HB.bp[k1 * G] - bb;
        fc.resize(flen);
        fv.resize(flen);
        bc.resize(blen);
        bv.resize(blen);
        for (int64_t idx = k0 * G; idx < k1 * G; idx++)   // list padding (multiple of 4 entries)
            for (int64_t e = HB.bp[idx] + HB.loc[(size_t)idx * NL + B]; e < HB.bp[idx + 1]; e++) {
                bc[e - bb] = 0;
                bv[e - bb] = make_double2(0.0, 0.0);
            }
        parallel_for(r1 - r0, threads, [&](int64_t lo, int64_t hi) {
            for (int64_t ip = r0 + lo; ip < r0 + hi; ip++) {
                int64_t q0, q1;
                row_range(ip, q0, q1);
                // row layout (ascending column = descending distance): far | list B | dense | block
                int64_t t = 0;
                for (int64_t u = 0; u < cnt[ip]; u++, t++) {
                    const int64_t q = entry(q0, q1, t);
                    fc[farptr[ip] - fb + u] = (int32_t)kcol(q);
                    fv[farptr[ip] - fb + u] = F.val[q];
                }
                for (int64_t u = 0; u < bcnt[ip]; u++, t++) {
                    const int64_t q = entry(q0, q1, t);
                    bc[HB.row[ip] - bb + u] = (int32_t)kcol(q);
                    bv[HB.row[ip] - bb + u] = F.val[q];
                }
            }
        });
        const double tc0 = now_ms();
        if (flen) {
            SSB_CUDA(cudaMemcpyAsync(T.fcol + fb, fc.data(), flen * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            SSB_CUDA(cudaMemcpyAsync(T.fval + fb, fv.data(), flen * sizeof(double2), cudaMemcpyHostToDevice, s));
        }
        if (blen > 0) {
            SSB_CUDA(cudaMemcpyAsync(T.nearB.col + bb, bc.data(), blen * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            SSB_CUDA(cudaMemcpyAsync(T.nearB.val + bb, bv.data(), blen * sizeof(double2), cudaMemcpyHostToDevice, s));
        }
        // on the problem's stream, complete before the staging buffers are refilled: a plain
        // cudaMemcpy from pageable memory runs on the legacy stream and may still be in flight
        // when it returns, unordered with a non-blocking stream (concurrent sweep points)
        SSB_CUDA(cudaStreamSynchronize(s));
        t_copy += now_ms() - tc0;
        k0 = k1;
    }
    tpf[2] = now_ms();

    // dense diagonal blocks -> explicit inverses D_k^{-1}, and Gd_k = D_k^{-1} T_{k,k-d} for
    // d = 1 .. kDense (column-major, G1 first per block), in block chunks
    const int64_t kBlkChunk = std::max<int64_t>(1, ((int64_t)1 << 27) / ((PK + kDense * (int64_t)B * B) * 16));
    std::vector<double2> ibuf, gbuf;
    for (int64_t k0 = 0; k0 < nblk; k0 += kBlkChunk) {
        const int64_t k1 = std::min(nblk, k0 + kBlkChunk);
        ibuf.assign((k1 - k0) * PK, make_double2(0.0, 0.0));
        gbuf.assign((k1 - k0) * kDense * B * B, make_double2(0.0, 0.0));
        parallel_for(k1 - k0, threads, [&](int64_t lo, int64_t hi) {
            std::vector<double2> D((size_t)B * B), X((size_t)B * B), inv(B), N1((size_t)B * B);
            for (int64_t k = k0 + lo; k < k0 + hi; k++) {
                std::fill(D.begin(), D.end(), make_double2(0.0, 0.0));
                const int64_t kb = k * B;
                for (int r = 0; r < B; r++) {
                    const int64_t ip = kb + r;
                    if (ip >= n) {
                        D[(size_t)r * B + r] = make_double2(1.0, 0.0);
                        continue;
                    }
                    int64_t q0, q1;
                    row_range(ip, q0, q1);
                    for (int64_t t = nin[ip]; t < q1 - q0; t++) {
                        const int64_t q = entry(q0, q1, t);
                        D[(size_t)r * B + (kcol(q) - kb)] = F.val[q];
                    }
                    const int64_t i = upper ? n - 1 - ip : ip;
                    D[(size_t)r * B + r] = diag ? diag[i] : make_double2(1.0, 0.0);
                }
                for (int r = 0; r < B; r++) {
                    const double2 d = D[(size_t)r * B + r];
                    const double m = d.x * d.x + d.y * d.y;
                    inv[r] = make_double2(d.x / m, -d.y / m);
                }
                // X = D^{-1}, column by column (forward substitution on unit vectors)
                for (int j = 0; j < B; j++) {
                    X[(size_t)j * B + j] = inv[j];
                    for (int i = j + 1; i < B; i++) {
                        double2 acc = make_double2(0.0, 0.0);
                        for (int m = j; m < i; m++) acc = cadd(acc, cmul(D[(size_t)i * B + m], X[(size_t)m * B + j]));
                        X[(size_t)i * B + j] = cmul(make_double2(-acc.x, -acc.y), inv[i]);
                    }
                }
                double2* out = &ibuf[(size_t)(k - k0) * PK];
                for (int j = 0; j < B; j++) {
                    const int64_t cs = (int64_t)j * B - ((int64_t)j * (j - 1)) / 2;
                    for (int i = j; i < B; i++) out[cs + (i - j)] = X[(size_t)i * B + j];
                }
                // Nd = T_{k,k-d}: the distance-d entries of the block's rows; Gd = X Nd.  Row
                // layout (ascending column): far | list B | d = kDense | .. | d = 1 | in-block
                for (int d = 1; d <= kDense; d++) {
                    if (k < d) continue;
                    std::fill(N1.begin(), N1.end(), make_double2(0.0, 0.0));
                    const int64_t kbd = (k - d) * B;
                    bool any = false;
                    for (int r = 0; r < B; r++) {
                        const int64_t ip = kb + r;
                        if (ip >= n) continue;
                        int64_t q0, q1;
                        row_range(ip, q0, q1);
                        int64_t t1 = nin[ip];
                        for (int e = 1; e < d; e++) t1 -= gcnt[(size_t)ip * kDense + e - 1];
                        const int64_t t0 = t1 - gcnt[(size_t)ip * kDense + d - 1];
                        for (int64_t t = t0; t < t1; t++) {
                            const int64_t q = entry(q0, q1, t);
                            N1[(size_t)r * B + (kcol(q) - kbd)] = F.val[q];
                            any = true;
                        }
                    }
                    if (!any) continue;
                    // column-major (the chain teams: lane = row, a warp per 8 columns)
                    double2* g = &gbuf[((size_t)(k - k0) * kDense + (d - 1)) * B * B];
                    for (int j = 0; j < B; j++)
                        for (int i = 0; i < B; i++) {
                            double2 acc = make_double2(0.0, 0.0);
                            for (int m = 0; m <= i; m++)
                                acc = cadd(acc, cmul(X[(size_t)i * B + m], N1[(size_t)m * B + j]));
                            g[(size_t)j * B + i] = acc;
                        }
                }
            }
        }, 4);
        SSB_CUDA(cudaMemcpyAsync(T.dinv + k0 * PK, ibuf.data(), (k1 - k0) * PK * sizeof(double2),
                                 cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaMemcpyAsync(T.G + k0 * kDense * B * B, gbuf.data(), (k1 - k0) * kDense * B * B * sizeof(double2),
                                 cudaMemcpyHostToDevice, s));
        SSB_CUDA(cudaStreamSynchronize(s));   // (as above: the problem's stream, buffers reused)
    }
    SSB_CUDA(cudaStreamSynchronize(s));
    block_trsv_prepare(T);
    if (prof)
        std::fprintf(stderr, "build_block_tri(%s): layout %.0f ms, entries %.0f ms (copies %.0f), dense blocks %.0f ms\n",
                     upper ? "U" : "L", tpf[1] - tpf[0], tpf[2] - tpf[1], t_copy, now_ms() - tpf[2]);
}

// Tuning knobs of the block substitution: rows per block and CTA size.

}  // namespace

void setup_problem(Problem& P, double drop_tol, double fill_factor, double permtol, int threads,
                   ss_setup_info* info) {
    cudaStream_t s = P.stream;
    SSB_CUDA(cudaSetDevice(P.device));   // every allocation below (and the helper thread's) on P's device
    P.have_setup = false;
    const double t0 = now_ms();
    HostCSR nat;
    download(P.nat, nat, s);
    P.bw_nat = bandwidth(nat);
    P.perm = rcm_order(nat.n, nat.rowptr, nat.col);
    HostCSR A = permute(nat, P.perm);
    P.bw_rcm = bandwidth(A);
    const double t1 = now_ms();
    // column-oriented iLUTP (R16): the row-wise iLUTP of L~_RCM^T,
    //   L~_RCM^T Pi = L' U'   <=>   Pi^T L~_RCM = U'^T L'^T
    IlutStats st;
    {
        const HostCSR At = transpose(A, false);
        ilut_factor(At, drop_tol, fill_factor, permtol, threads, P.hL, P.hU, P.colperm, st);
    }
    const double t2 = now_ms();
    // the hot path solves the row-permuted system A' x = b', A' = Pi^T L~_RCM (row j of A' is
    // row colperm[j] of L~_RCM), preconditioned by M'^{-1} = L'^{-T} U'^{-T}: the same Krylov
    // space as M^{-1} L~_RCM with M = Pi U'^T L'^T, and no permutation left in the loop
    const int64_t n = P.n;
    {
        const HostCSR Ar = permute_rows(A, P.colperm);
        upload(Ar, P.A, s);
        build_sell(Ar, P.A, s);
    }
    P.rowperm.resize(n);
    P.rhs_pos = -1;
    for (int64_t j = 0; j < n; j++) {
        P.rowperm[j] = P.perm[P.colperm[j]];   // natural index of row j of A'
        if (P.rowperm[j] == 0) P.rhs_pos = j;  // b = (w, 0, ...): w sits in row 0 of L~
    }
    if (!P.d_perm) SSB_CUDA(cudaMalloc(&P.d_perm, n * sizeof(int64_t)));
    if (!P.d_rowperm) SSB_CUDA(cudaMalloc(&P.d_rowperm, n * sizeof(int64_t)));
    SSB_CUDA(cudaMemcpyAsync(P.d_perm, P.perm.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SSB_CUDA(cudaMemcpyAsync(P.d_rowperm, P.rowperm.data(), n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (threads <= 0) threads = (int)std::max(1u, std::thread::hardware_concurrency());
    const int B = env_int("SSB_TRSV_B", 32);
    const int QMAX = env_int("SSB_TRSV_Q", 32);
    const int QMAX_U = env_int("SSB_TRSV_QU", QMAX);   // (the upper factor's window, if different)
    // the two substitutions: first U'^T (lower, the pivots on its diagonal), then L'^T (unit upper)
    HostCSR F1, F2;
    std::vector<double2> d1(n);
    {
        std::thread tt([&] { F2 = transpose(P.hL, false); });
        F1 = transpose(P.hU, true);
        for (int64_t i = 0; i < n; i++) d1[i] = P.hU.val[P.hU.rowptr[i]];
        tt.join();
    }
    int64_t levL = 0, levU = 0;
    std::thread lev([&] { levL = count_levels(F1, false); });   // diagnostics, off the path
    std::thread levu([&] { levU = count_levels(F2, true); });
    try {
        // the two factors' layouts are independent: build them concurrently (host work of
        // one overlaps the other's copies)
        std::exception_ptr errL;
        std::thread tl([&] {
            try {
                SSB_CUDA(cudaSetDevice(P.device));   // the current device is per host thread
                build_block_tri(F1, d1.data(), false, B, QMAX, threads, P.L, s);
            } catch (...) {
                errL = std::current_exception();
            }
        });
        try {
            build_block_tri(F2, nullptr, true, B, QMAX_U, threads, P.U, s);
        } catch (...) {
            tl.join();
            throw;
        }
        tl.join();
        if (errL) std::rethrow_exception(errL);
    } catch (...) {
        lev.join();
        levu.join();
        throw;
    }
    lev.join();
    levu.join();
    P.L.sm_budget = P.U.sm_budget = P.sm_budget;
    P.L.nlev = levL;
    P.U.nlev = levU;
    const double t3 = now_ms();
    P.have_setup = true;
    P.have_solution = false;
    if (info) {
        info->nnz_L = P.hL.nnz();
        info->nnz_U = P.hU.nnz();
        info->fill = (double)(P.hL.nnz() + P.hU.nnz()) / (double)P.nnz;
        info->bandwidth_nat = P.bw_nat;
        info->bandwidth_rcm = P.bw_rcm;
        info->levels_L = P.L.nlev;
        info->levels_U = P.U.nlev;
        info->pivots_repaired = st.repaired;
        info->pivot_swaps = st.swaps;
        info->threads = st.threads;
        info->trsv_block = B;
        info->trsv_grid = P.L.grid;
        info->trsv_q_L = P.L.Q;
        info->trsv_q_U = P.U.Q;
        info->rcm_ms = t1 - t0;
        info->ilut_ms = t2 - t1;
        info->upload_ms = t3 - t2;
    }
}

}  // namespace ssb
