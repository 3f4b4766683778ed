/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY. A plain, slow, obviously-correct CPU
 * reference for what the GPU path computes. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with paper_1501_05387_b200/.
 *
 * What it computes is the PLAIN DEFINITION the method reaches exactly
 * (DESIGN.md "Oracle"):
 *
 *   oracle_bfs  -- depth[v] = number of edges on a shortest src->v path that
 *                  follows CSR out-edges, -1 if unreachable; pred[v] = the
 *                  vertex that first discovered v in FIFO order, pred[src] =
 *                  src (reading A-1), -1 if unreachable (A-2).
 *                  Paper: BFS labels are "the distance from the source" and
 *                  pred "the predecessor vertex's ID" (PAPER.md P:892-897,
 *                  P:910-912, §5.1). Algorithm: the textbook FIFO queue BFS.
 *
 *   oracle_sssp -- dist[v] = min over src->v paths of the sum of the integer
 *                  edge weights, UINT32_MAX if unreachable (A-2); weights are
 *                  non-negative (§4.1 "We assume weights between
 *                  nodes are all non-negative, which permits the use of
 *                  Dijkstra's algorithm"). Algorithm: textbook Dijkstra with
 *                  a binary heap and lazy deletion, accumulated in uint64.
 *                  pred[v] = the vertex whose relaxation last lowered dist[v]
 *                  (a tight parent), pred[src] = src.
 *
 *   oracle_bc   -- bc[v] = sum over the given sources s of Brandes's dependency
 *                  delta_s(v) = sum over t != s, v of sigma_st(v) / sigma_st,
 *                  with shortest = fewest CSR out-edges (no halving).
 *                  Paper §5.3 names Brandes's formulation
 *                  ("a forward BFS pass to accumulate sigma values for each
 *                  node, and a backward BFS pass to compute centrality
 *                  values"). Algorithm: Brandes 2001, Algorithm 1, as printed
 *                  (FIFO BFS with a stack S and predecessor lists P[w]; then
 *                  pop w, delta[v] += sigma[v]/sigma[w] * (1 + delta[w]) for
 *                  v in P[w]; bc[w] += delta[w] for w != s), in double.
 *
 *   oracle_cc   -- comp[v] = the smallest vertex id of v's (weakly) connected
 *                  component, edges taken as undirected; returns the number
 *                  of components in *ncomp. Paper §5.4: "labels
 *                  the vertices in each connected component in a graph with a
 *                  unique component ID". Algorithm: textbook disjoint-set
 *                  union (union by size, path halving) over every CSR edge,
 *                  then the minimum id of each set.
 *
 * Return codes: 0 ok, 1 bad argument (src out of range / n <= 0),
 * 2 out of memory, 3 a distance does not fit in uint32 (reading A-19).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int oracle_bfs(int64_t n, const int64_t *R, const int32_t *C, int32_t src,
               int32_t *depth, int32_t *pred)
{
    if (n <= 0 || src < 0 || src >= n) return 1;
    int32_t *queue = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!queue) return 2;
    for (int64_t v = 0; v < n; ++v) {
        depth[v] = -1;
        if (pred) pred[v] = -1;
    }
    int64_t head = 0, tail = 0;
    depth[src] = 0;
    if (pred) pred[src] = src;
    queue[tail++] = src;
    while (head < tail) {
        int32_t u = queue[head++];
        for (int64_t e = R[u]; e < R[u + 1]; ++e) {
            int32_t v = C[e];
            if (depth[v] == -1) {
                depth[v] = depth[u] + 1;
                if (pred) pred[v] = u;
                queue[tail++] = v;
            }
        }
    }
    free(queue);
    return 0;
}

/* ---- binary min-heap of (key = dist, vertex) with lazy deletion ---------- */
typedef struct { uint64_t d; int32_t v; } heap_item;

static void heap_push(heap_item *h, int64_t *size, heap_item x)
{
    int64_t i = (*size)++;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p].d <= x.d) break;
        h[i] = h[p];
        i = p;
    }
    h[i] = x;
}

static heap_item heap_pop(heap_item *h, int64_t *size)
{
    heap_item top = h[0];
    heap_item last = h[--(*size)];
    int64_t i = 0, s = *size;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, c = i;
        uint64_t cd = last.d;
        if (l < s && h[l].d < cd) { c = l; cd = h[l].d; }
        if (r < s && h[r].d < cd) { c = r; }
        if (c == i) break;
        h[i] = h[c];
        i = c;
    }
    if (s > 0) h[i] = last;
    return top;
}

int oracle_sssp(int64_t n, const int64_t *R, const int32_t *C, const uint32_t *W,
                int32_t src, uint32_t *dist_out, int32_t *pred)
{
    if (n <= 0 || src < 0 || src >= n || !W) return 1;
    int64_t m = R[n];
    uint64_t *dist = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
    /* every successful relaxation pushes one item: at most m + 1 live items */
    heap_item *heap = (heap_item *)malloc((size_t)(m + 1) * sizeof(heap_item));
    if (!dist || !done || !heap) { free(dist); free(done); free(heap); return 2; }
    const uint64_t INF = UINT64_MAX;
    for (int64_t v = 0; v < n; ++v) {
        dist[v] = INF;
        if (pred) pred[v] = -1;
    }
    int64_t size = 0;
    dist[src] = 0;
    if (pred) pred[src] = src;
    heap_item s0 = {0, src};
    heap_push(heap, &size, s0);
    while (size > 0) {
        heap_item it = heap_pop(heap, &size);
        int32_t u = it.v;
        if (done[u] || it.d != dist[u]) continue; /* stale entry */
        done[u] = 1;
        for (int64_t e = R[u]; e < R[u + 1]; ++e) {
            int32_t v = C[e];
            uint64_t nd = dist[u] + (uint64_t)W[e];
            if (nd < dist[v]) {
                dist[v] = nd;
                if (pred) pred[v] = u;
                heap_item x = {nd, v};
                heap_push(heap, &size, x);
            }
        }
    }
    int rc = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (dist[v] == INF) dist_out[v] = UINT32_MAX;
        else if (dist[v] >= (uint64_t)UINT32_MAX) { rc = 3; dist_out[v] = UINT32_MAX; }
        else dist_out[v] = (uint32_t)dist[v];
    }
    free(dist); free(done); free(heap);
    return rc;
}

int oracle_bc(int64_t n, const int64_t *R, const int32_t *C, const int32_t *sources, int64_t nsrc,
              double *bc)
{
    if (n <= 0 || nsrc < 0) return 1;
    for (int64_t i = 0; i < nsrc; ++i)
        if (sources[i] < 0 || sources[i] >= n) return 1;
    int64_t m = R[n];
    int32_t *S = (int32_t *)malloc((size_t)n * sizeof(int32_t));      /* stack (= BFS order) */
    int64_t *dist = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    double *sigma = (double *)malloc((size_t)n * sizeof(double));
    double *delta = (double *)malloc((size_t)n * sizeof(double));
    int64_t *phead = (int64_t *)malloc((size_t)n * sizeof(int64_t));  /* P[w]: linked lists */
    int64_t *pnext = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    int32_t *pv = (int32_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    if (!S || !dist || !sigma || !delta || !phead || !pnext || !pv) {
        free(S); free(dist); free(sigma); free(delta); free(phead); free(pnext); free(pv);
        return 2;
    }
    for (int64_t v = 0; v < n; ++v) bc[v] = 0.0;
    for (int64_t i = 0; i < nsrc; ++i) {
        int32_t s = sources[i];
        int64_t np = 0, top = 0, head = 0;
        for (int64_t v = 0; v < n; ++v) {
            phead[v] = -1;
            sigma[v] = 0.0;
            dist[v] = -1;
        }
        sigma[s] = 1.0;
        dist[s] = 0;
        /* the queue is S itself: S[head..top) are enqueued, S[0..top) is the stack */
        S[top++] = s;
        while (head < top) {
            int32_t v = S[head++];
            for (int64_t e = R[v]; e < R[v + 1]; ++e) {
                int32_t w = C[e];
                if (dist[w] < 0) {             /* w found for the first time? */
                    S[top++] = w;
                    dist[w] = dist[v] + 1;
                }
                if (dist[w] == dist[v] + 1) {  /* shortest path to w via v? */
                    sigma[w] += sigma[v];
                    pv[np] = v;                /* append v to P[w] */
                    pnext[np] = phead[w];
                    phead[w] = np++;
                }
            }
        }
        for (int64_t v = 0; v < n; ++v) delta[v] = 0.0;
        while (top > 0) {                      /* S returns vertices in order of non-increasing distance */
            int32_t w = S[--top];
            for (int64_t k = phead[w]; k >= 0; k = pnext[k]) {
                int32_t v = pv[k];
                delta[v] += sigma[v] / sigma[w] * (1.0 + delta[w]);
            }
            if (w != s) bc[w] += delta[w];
        }
    }
    free(S); free(dist); free(sigma); free(delta); free(phead); free(pnext); free(pv);
    return 0;
}

static int32_t uf_find(int32_t *parent, int32_t x)
{
    while (parent[x] != x) {
        parent[x] = parent[parent[x]]; /* path halving */
        x = parent[x];
    }
    return x;
}

int oracle_cc(int64_t n, const int64_t *R, const int32_t *C, int32_t *comp, int64_t *ncomp)
{
    if (n <= 0) return 1;
    int32_t *parent = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int64_t *size = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    int32_t *minid = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    if (!parent || !size || !minid) { free(parent); free(size); free(minid); return 2; }
    for (int64_t v = 0; v < n; ++v) { parent[v] = (int32_t)v; size[v] = 1; }
    for (int64_t u = 0; u < n; ++u)
        for (int64_t e = R[u]; e < R[u + 1]; ++e) {
            int32_t a = uf_find(parent, (int32_t)u), b = uf_find(parent, C[e]);
            if (a == b) continue;
            if (size[a] < size[b]) { int32_t t = a; a = b; b = t; }
            parent[b] = a;               /* union by size */
            size[a] += size[b];
        }
    for (int64_t v = 0; v < n; ++v) minid[v] = INT32_MAX;
    int64_t k = 0;
    for (int64_t v = 0; v < n; ++v) {   /* increasing v: the first member seen is the minimum */
        int32_t r = uf_find(parent, (int32_t)v);
        if (minid[r] == INT32_MAX) { minid[r] = (int32_t)v; ++k; }
        comp[v] = minid[r];
    }
    *ncomp = k;
    free(parent); free(size); free(minid);
    return 0;
}
