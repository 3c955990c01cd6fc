// rcm.cpp -- reverse Cuthill-McKee ordering of pattern(L~ + L~^T) (setup, host).
//
// PAPER.md:98 (sec. III): breadth-first search from a node of lowest degree (degree =
// number of nonzeros of the row), neighbours of each node visited from lowest to
// highest degree, repeated for every connected component, order reversed; computed
// on the symmetrised structure L~ + L~^T.  Tie-breaking (reading R3):
// equal degrees -> smaller original index, for component starts and for neighbours.
// The paper notes "RCM reordering itself is a serial algorithm": this
// is a single-threaded O(nnz log d) host pass, timed separately by ss_setup.
#include <algorithm>
#include <numeric>

#include "problem.h"

namespace ssb {

std::vector<int64_t> rcm_order(int64_t n, const std::vector<int64_t>& rowptr, const hvec<int64_t>& col) {
    // transpose pattern (counting sort by column)
    std::vector<int64_t> tptr(n + 1, 0), tcol(col.size());
    for (int64_t c : col) tptr[c + 1]++;
    for (int64_t i = 0; i < n; i++) tptr[i + 1] += tptr[i];
    {
        std::vector<int64_t> pos(tptr.begin(), tptr.end() - 1);
        for (int64_t i = 0; i < n; i++)
            for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) tcol[pos[col[q]]++] = i;
    }
    // union rows (both sorted ascending) -> symmetric pattern S
    std::vector<int64_t> sptr(n + 1, 0);
    std::vector<int64_t> scol;
    scol.reserve(col.size() * 2);
    for (int64_t i = 0; i < n; i++) {
        int64_t a = rowptr[i], ae = rowptr[i + 1], b = tptr[i], be = tptr[i + 1];
        while (a < ae || b < be) {
            int64_t v;
            if (b >= be || (a < ae && col[a] < tcol[b])) v = col[a++];
            else if (a >= ae || tcol[b] < col[a]) v = tcol[b++];
            else { v = col[a]; a++; b++; }
            scol.push_back(v);
        }
        sptr[i + 1] = (int64_t)scol.size();
    }
    std::vector<int64_t> deg(n);
    for (int64_t i = 0; i < n; i++) deg[i] = sptr[i + 1] - sptr[i];
    // global order of nodes by (degree, index)
    std::vector<int64_t> by(n);
    std::iota(by.begin(), by.end(), 0);
    std::stable_sort(by.begin(), by.end(), [&](int64_t x, int64_t y) { return deg[x] < deg[y]; });
    std::vector<int64_t> rank(n);
    for (int64_t r = 0; r < n; r++) rank[by[r]] = r;

    std::vector<char> seen(n, 0);
    std::vector<int64_t> q;
    q.reserve(n);
    std::vector<int64_t> kids;
    for (int64_t r = 0; r < n; r++) {
        const int64_t s0 = by[r];
        if (seen[s0]) continue;
        seen[s0] = 1;
        size_t head = q.size();
        q.push_back(s0);
        while (head < q.size()) {
            const int64_t v = q[head++];
            kids.clear();
            for (int64_t p = sptr[v]; p < sptr[v + 1]; p++) {
                const int64_t u = scol[p];
                if (u != v && !seen[u]) {
                    seen[u] = 1;
                    kids.push_back(u);
                }
            }
            std::sort(kids.begin(), kids.end(), [&](int64_t x, int64_t y) { return rank[x] < rank[y]; });
            q.insert(q.end(), kids.begin(), kids.end());
        }
    }
    std::reverse(q.begin(), q.end());
    return q;
}

}  // namespace ssb
