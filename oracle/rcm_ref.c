/*
 * oracle/rcm_ref.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Second, independently written reverse Cuthill-McKee (sec. III)
 * used to cross-check oracle/rcm.py bit-exactly and to order large inputs.
 * Same rule (R3), different construction:
 *   - a global rank of every node by (degree, index) is built with a stable
 *     counting sort on the degree;
 *   - the BFS is run level set by level set; the unvisited neighbours of each
 *     node of the current level are appended in increasing rank (insertion
 *     sort on rank);
 *   - components are started from the lowest-ranked unvisited node;
 *   - the Cuthill-McKee sequence is finally reversed.
 * Input: a structurally symmetric CSR pattern (rowptr/colidx, int64).
 * Output: perm[new] = old.
 */
#include <stdint.h>
#include <stdlib.h>

int oracle_rcm(int64_t n, const int64_t *rowptr, const int64_t *colidx, int64_t *perm)
{
    int64_t *deg = malloc(n * sizeof(int64_t));
    int64_t *rank = malloc(n * sizeof(int64_t));
    int64_t *byrank = malloc(n * sizeof(int64_t));
    char *seen = calloc(n, 1);
    int64_t *cm = malloc(n * sizeof(int64_t));
    if (!deg || !rank || !byrank || !seen || !cm) return -1;

    int64_t maxdeg = 0;
    for (int64_t i = 0; i < n; i++) {
        deg[i] = rowptr[i + 1] - rowptr[i];
        if (deg[i] > maxdeg) maxdeg = deg[i];
    }
    int64_t *cnt = calloc(maxdeg + 2, sizeof(int64_t));
    if (!cnt) return -1;
    for (int64_t i = 0; i < n; i++) cnt[deg[i] + 1]++;
    for (int64_t d = 1; d <= maxdeg + 1; d++) cnt[d] += cnt[d - 1];
    for (int64_t i = 0; i < n; i++) {          /* stable: index order within a degree */
        int64_t r = cnt[deg[i]]++;
        rank[i] = r;
        byrank[r] = i;
    }
    free(cnt);

    int64_t filled = 0;
    for (int64_t r0 = 0; r0 < n; r0++) {
        int64_t s = byrank[r0];
        if (seen[s]) continue;
        seen[s] = 1;
        cm[filled++] = s;
        int64_t lev_begin = filled - 1, lev_end = filled;
        while (lev_begin < lev_end) {
            for (int64_t t = lev_begin; t < lev_end; t++) {
                int64_t v = cm[t];
                int64_t first_new = filled;
                for (int64_t q = rowptr[v]; q < rowptr[v + 1]; q++) {
                    int64_t u = colidx[q];
                    if (u == v || seen[u]) continue;
                    seen[u] = 1;
                    /* insertion by rank among this node's new children */
                    int64_t pos = filled++;
                    while (pos > first_new && rank[cm[pos - 1]] > rank[u]) { cm[pos] = cm[pos - 1]; pos--; }
                    cm[pos] = u;
                }
            }
            lev_begin = lev_end;
            lev_end = filled;
        }
    }
    for (int64_t k = 0; k < n; k++) perm[k] = cm[n - 1 - k];
    free(deg); free(rank); free(byrank); free(seen); free(cm);
    return filled == n ? 0 : -2;
}
