/*
 * oracle/tc_oracle.c -- CPU oracle for exact triangle counting.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1804_06926_b200/) never imports, links or calls it,
 * and this file shares no source, header, table or helper with the CUDA path.
 *
 * Plain, slow, obviously-correct C.  Integer arithmetic only (there is no
 * floating point anywhere on the path: PAPER.md never rounds).
 * Citations: "P:n" = /root/reference/PAPER.md line n.
 *
 * What it computes (the plain definition):
 *   T(G) = |{ {a,b,c} : {a,b},{b,c},{a,c} in E }|,
 *   E    = { {u,v} : u != v and (u,v) or (v,u) is an input arc },
 *   t(v) = number of those triangles that contain v.
 *
 * How (the paper's own CPU baseline, Schank-Wagner "forward", P:577-579,
 * P:301-306 §3.2; Alg. 2 P:333-366 in its step order):
 *   1. clean      -- arcs read as undirected, self-loops dropped, duplicates
 *                    collapsed (Table 1 caption P:604-606; DESIGN reading R1).
 *   2. orient     -- "Form_Filtered_Edge_List" (Alg. 2): keep each
 *                    undirected edge once, from lower to higher (degree, id)
 *                    rank (DESIGN reading R2: direction per north_star,
 *                    tie-break by smaller id exactly as P:521-522).
 *   3. intersect  -- "Compute_Intersection": for every kept edge
 *                    (u,v) the matches w of N+(u) and N+(v) ("Let the
 *                    intersections between the neighbor lists of u and v be
 *                    (w_1..w_N) ... the number of triangles formed with e is N",
 *                    P:315-321), by a plain two-pointer merge of sorted lists.
 *   4. reduce     -- "Count = Reduce(IntersectList)", uint64.
 *
 * Per-vertex counts: each match w of edge (u,v) is the triangle {u,v,w}; it
 * adds one to t(u), t(v) and t(w) (clustering-coefficient use).
 *
 * oracle_vertex_triangles() is the per-vertex DEFINITION written out
 * (t(v) = number of edges among N(v)) for sampled checks at full size.
 *
 * Error behaviour: functions return a negative int on bad input (an arc id
 * >= n) or allocation failure; nothing is ever partially trusted.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return (x > y) - (x < y);
}

/*
 * Step 1: clean.  Input: any CSR of n vertices (arcs u -> col[k] for
 * rowptr[u] <= k < rowptr[u+1]).  Output: the simple undirected graph as a
 * symmetric CSR with each row sorted ascending: out_rowptr[n+1],
 * out_col[capacity 2*rowptr[n]].  Returns the number of stored arcs (= 2m),
 * or -1 if an arc points outside [0,n), -2 on allocation failure.
 */
int64_t oracle_clean(uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                     uint64_t *out_rowptr, uint32_t *out_col) {
    uint64_t M = rowptr[n];
    uint64_t *pairs = (uint64_t *)malloc((M ? M : 1) * sizeof(uint64_t));
    if (!pairs) return -2;
    uint64_t k = 0;
    for (uint64_t u = 0; u < n; u++) {
        for (uint64_t e = rowptr[u]; e < rowptr[u + 1]; e++) {
            uint64_t v = col[e];
            if (v >= n) { free(pairs); return -1; }
            if (v == u) continue;                     /* self-loop dropped */
            uint64_t a = u < v ? u : v, b = u < v ? v : u;
            pairs[k++] = (a << 32) | b;               /* undirected edge {a,b} */
        }
    }
    qsort(pairs, k, sizeof(uint64_t), cmp_u64);
    uint64_t m = 0;                                   /* duplicates collapsed */
    for (uint64_t i = 0; i < k; i++)
        if (m == 0 || pairs[i] != pairs[m - 1]) pairs[m++] = pairs[i];

    uint64_t *deg = (uint64_t *)calloc(n + 1, sizeof(uint64_t));
    if (!deg) { free(pairs); return -2; }
    for (uint64_t i = 0; i < m; i++) {
        deg[pairs[i] >> 32]++;
        deg[pairs[i] & 0xffffffffu]++;
    }
    out_rowptr[0] = 0;
    for (uint64_t v = 0; v < n; v++) out_rowptr[v + 1] = out_rowptr[v] + deg[v];
    for (uint64_t v = 0; v < n; v++) deg[v] = out_rowptr[v];   /* reuse as cursor */
    for (uint64_t i = 0; i < m; i++) {
        uint32_t a = (uint32_t)(pairs[i] >> 32), b = (uint32_t)(pairs[i] & 0xffffffffu);
        out_col[deg[a]++] = b;
        out_col[deg[b]++] = a;
    }
    for (uint64_t v = 0; v < n; v++)
        qsort(out_col + out_rowptr[v], out_rowptr[v + 1] - out_rowptr[v],
              sizeof(uint32_t), cmp_u32);
    free(deg);
    free(pairs);
    return (int64_t)(2 * m);
}

/* rank(u) < rank(v) with rank = (d, id) compared lexicographically. */
static int rank_less(const uint64_t *rowptr, uint64_t u, uint64_t v) {
    uint64_t du = rowptr[u + 1] - rowptr[u], dv = rowptr[v + 1] - rowptr[v];
    return du < dv || (du == dv && u < v);
}

/*
 * Step 2: orient ("Form_Filtered_Edge_List", Alg. 2; filter rule
 * P:520-523).  Input: a clean symmetric CSR with sorted rows (oracle_clean's
 * output).  Output: N+(u) = { v in N(u) : rank(u) < rank(v) } in
 * off_plus[n+1] / col_plus[capacity rowptr[n]/2], each row ascending because
 * N(u) is.  Returns m (the number of kept edges).
 */
int64_t oracle_orient(uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                      uint64_t *off_plus, uint32_t *col_plus) {
    uint64_t k = 0;
    off_plus[0] = 0;
    for (uint64_t u = 0; u < n; u++) {
        for (uint64_t e = rowptr[u]; e < rowptr[u + 1]; e++)
            if (rank_less(rowptr, u, col[e])) col_plus[k++] = col[e];
        off_plus[u + 1] = k;
    }
    return (int64_t)k;
}

/*
 * Steps 3+4: for each kept edge (u,v), merge N+(u) and N+(v); every common
 * element w is one triangle {u,v,w}; Count = sum.
 * per_vertex (nullable, n entries, zeroed here) receives t(v).
 */
uint64_t oracle_forward(uint64_t n, const uint64_t *off_plus, const uint32_t *col_plus,
                        uint64_t *per_vertex) {
    if (per_vertex) memset(per_vertex, 0, n * sizeof(uint64_t));
    uint64_t T = 0;
    int64_t nn = (int64_t)n;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : T)
    for (int64_t uu = 0; uu < nn; uu++) {
        uint64_t u = (uint64_t)uu;
        for (uint64_t e = off_plus[u]; e < off_plus[u + 1]; e++) {
            uint64_t v = col_plus[e];
            uint64_t i = off_plus[u], iend = off_plus[u + 1];
            uint64_t j = off_plus[v], jend = off_plus[v + 1];
            while (i < iend && j < jend) {
                uint32_t a = col_plus[i], b = col_plus[j];
                if (a < b) {
                    i++;
                } else if (a > b) {
                    j++;
                } else {                               /* w = a is in both lists */
                    T++;
                    if (per_vertex) {
#pragma omp atomic
                        per_vertex[u]++;
#pragma omp atomic
                        per_vertex[v]++;
#pragma omp atomic
                        per_vertex[a]++;
                    }
                    i++;
                    j++;
                }
            }
        }
    }
    return T;
}

/*
 * Whole oracle: clean -> orient -> intersect -> reduce.
 * stats (nullable, 8 entries): [0] m (undirected edges), [1] W =
 * sum over kept edges of d+(u)+d+(v) (merge work), [2] SSD = sum d(v)^2
 * (Fig. ssd), [3] sum_v d-(v)*d+(v), [4] max d+, [5] max d,
 * [6] wedges = sum C(d(v),2), [7] unused (0).
 * Returns 0 and writes *total, or a negative error from oracle_clean.
 */
int oracle_count(uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                 uint64_t *total, uint64_t *per_vertex, uint64_t *stats) {
    uint64_t M = rowptr[n];
    uint64_t *crow = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    uint32_t *ccol = (uint32_t *)malloc((M ? 2 * M : 1) * sizeof(uint32_t));
    uint64_t *orow = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    uint32_t *ocol = (uint32_t *)malloc((M ? M : 1) * sizeof(uint32_t));
    if (!crow || !ccol || !orow || !ocol) {
        free(crow); free(ccol); free(orow); free(ocol);
        return -2;
    }
    int64_t arcs = oracle_clean(n, rowptr, col, crow, ccol);
    if (arcs < 0) {
        free(crow); free(ccol); free(orow); free(ocol);
        return (int)arcs;
    }
    int64_t m = oracle_orient(n, crow, ccol, orow, ocol);
    *total = oracle_forward(n, orow, ocol, per_vertex);
    if (stats) {
        memset(stats, 0, 8 * sizeof(uint64_t));
        stats[0] = (uint64_t)m;
        for (uint64_t u = 0; u < n; u++) {
            uint64_t dp = orow[u + 1] - orow[u];
            uint64_t d = crow[u + 1] - crow[u];
            for (uint64_t e = orow[u]; e < orow[u + 1]; e++) {
                uint64_t v = ocol[e];
                stats[1] += dp + (orow[v + 1] - orow[v]);
            }
            stats[2] += d * d;
            stats[3] += (d - dp) * dp;
            if (dp > stats[4]) stats[4] = dp;
            if (d > stats[5]) stats[5] = d;
            stats[6] += d * (d ? d - 1 : 0) / 2;
        }
    }
    free(crow); free(ccol); free(orow); free(ocol);
    return 0;
}

static int contains(const uint32_t *list, uint64_t len, uint32_t x) {
    return bsearch(&x, list, len, sizeof(uint32_t), cmp_u32) != NULL;
}

/*
 * Per-vertex definition for sampled checks: t(v) = number of edges {x,y}
 * with x,y in N(v), i.e. (1/2) sum_{x in N(v)} |N(v) cap N(x)|.  Input is a
 * clean symmetric CSR with sorted rows.  Each |N(v) cap N(x)| scans the
 * shorter list and looks each element up in the longer one (bsearch).
 */
uint64_t oracle_vertex_triangles(uint64_t n, const uint64_t *rowptr, const uint32_t *col,
                                 uint64_t v) {
    (void)n;
    const uint32_t *Nv = col + rowptr[v];
    uint64_t dv = rowptr[v + 1] - rowptr[v];
    uint64_t twice = 0;
    for (uint64_t i = 0; i < dv; i++) {
        uint32_t x = Nv[i];
        const uint32_t *Nx = col + rowptr[x];
        uint64_t dx = rowptr[x + 1] - rowptr[x];
        const uint32_t *s = dx < dv ? Nx : Nv, *l = dx < dv ? Nv : Nx;
        uint64_t ls = dx < dv ? dx : dv, ll = dx < dv ? dv : dx;
        for (uint64_t k = 0; k < ls; k++) twice += (uint64_t)contains(l, ll, s[k]);
    }
    return twice / 2;
}

/*
 * NEXT-1 ("clustering coefficient and
 * transitivity"), conventions of SURVEY §8(c) reading 9 / DESIGN.md R14, written
 * out by definition on the CLEAN symmetric CSR (d(v) = row length) and the
 * per-vertex counts t(v):
 *   cc[v]   = 2 t(v) / (d(v) (d(v) - 1)), 0 when d(v) < 2;
 *   *wedges = sum_v d(v) (d(v) - 1) / 2 (connected triples);
 *   *sum    = sum_v cc[v], added in vertex order;
 *   *trans  = 3 T / *wedges, 0 when there is no wedge.
 */
void oracle_clustering(uint64_t n, const uint64_t *rowptr, const uint64_t *t, uint64_t T,
                       double *cc, uint64_t *wedges, double *sum, double *trans) {
    uint64_t w = 0;
    double s = 0.0;
    for (uint64_t v = 0; v < n; v++) {
        uint64_t d = rowptr[v + 1] - rowptr[v];
        double c = 0.0;
        if (d >= 2) {
            c = (2.0 * (double)t[v]) / (double)(d * (d - 1));
            w += d * (d - 1) / 2;
        }
        cc[v] = c;
        s += c;
    }
    *wedges = w;
    *sum = s;
    *trans = w ? (3.0 * (double)T) / (double)w : 0.0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * NEXT-2: leaf pruning before orientation.  The paper's
 * filtering stage removes vertices that cannot be in any triangle: "nodes with
 * degree less than two cannot be matched [to] any query vertex, since every node
 * in a triangle has a degree of two", prunes the non-candidate
 * edges and "reconstruct[s] the graph ... update[s] node degree and neighbor list
 * information.  So we can run the above two steps for a few iterations in order
 * to prune out more edges".  One ROUND, written out:
 *   1. d(v) = degree of v in the current graph;
 *   2. delete every edge {u,v} with d(u) < 2 or d(v) < 2.
 * rounds > 0: exactly that many rounds.  rounds = 0: repeat until a round deletes
 * nothing (the result is then the edge set of the 2-core; reading R15).
 * Input: clean symmetric CSR with sorted rows (oracle_clean's output); output in
 * the same format (out_col capacity rowptr[n]).  Returns the number of stored
 * arcs (2m'), *done = rounds executed (in fixed-point mode including the final
 * round that deleted nothing), or -2 on allocation failure.
 */
int64_t oracle_prune(uint64_t n, const uint64_t *rowptr, const uint32_t *col, uint32_t rounds,
                     uint64_t *out_rowptr, uint32_t *out_col, uint32_t *done) {
    uint64_t M = rowptr[n];
    uint64_t *deg = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    uint64_t *tmp_row = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    uint32_t *tmp_col = (uint32_t *)malloc((M ? M : 1) * sizeof(uint32_t));
    if (!deg || !tmp_row || !tmp_col) {
        free(deg); free(tmp_row); free(tmp_col);
        return -2;
    }
    /* current graph := input */
    memcpy(out_rowptr, rowptr, (n + 1) * sizeof(uint64_t));
    if (M) memcpy(out_col, col, M * sizeof(uint32_t));
    uint32_t r = 0;
    for (;;) {
        if (rounds && r == rounds) break;
        /* 1. degrees of the current graph */
        for (uint64_t v = 0; v < n; v++) deg[v] = out_rowptr[v + 1] - out_rowptr[v];
        /* 2. keep arc (u,v) iff d(u) >= 2 and d(v) >= 2 (rows stay sorted) */
        uint64_t k = 0, deleted = 0;
        tmp_row[0] = 0;
        for (uint64_t u = 0; u < n; u++) {
            for (uint64_t e = out_rowptr[u]; e < out_rowptr[u + 1]; e++) {
                uint32_t v = out_col[e];
                if (deg[u] >= 2 && deg[v] >= 2) tmp_col[k++] = v;
                else deleted++;
            }
            tmp_row[u + 1] = k;
        }
        memcpy(out_rowptr, tmp_row, (n + 1) * sizeof(uint64_t));
        if (k) memcpy(out_col, tmp_col, k * sizeof(uint32_t));
        r++;
        if (!rounds && deleted == 0) break;
    }
    if (done) *done = r;
    free(deg); free(tmp_row); free(tmp_col);
    return (int64_t)out_rowptr[n];
}

/*
 * NEXT-3: edge support, the k-truss prerequisite ("enumerating
 * triangles is useful as a subroutine in solving k-truss"; "the three ...
 * algorithms we examine ... will also enumerate triangles").  By
 * definition sup({u,v}) = number of triangles containing the edge {u,v}
 * = |N(u) cap N(v)| in the simple graph.  For every entry e of an oriented CSR
 * (off_plus, col_plus; edge (u, col_plus[e])) this writes sup[e], computed as a
 * two-pointer merge of the FULL sorted rows N(u), N(v) of the clean symmetric
 * CSR (crow, ccol).
 */
void oracle_edge_support(uint64_t n, const uint64_t *crow, const uint32_t *ccol,
                         const uint64_t *off_plus, const uint32_t *col_plus, uint32_t *sup) {
    for (uint64_t u = 0; u < n; u++) {
        for (uint64_t e = off_plus[u]; e < off_plus[u + 1]; e++) {
            uint64_t v = col_plus[e];
            uint64_t i = crow[u], iend = crow[u + 1], j = crow[v], jend = crow[v + 1];
            uint32_t c = 0;
            while (i < iend && j < jend) {
                if (ccol[i] < ccol[j]) i++;
                else if (ccol[i] > ccol[j]) j++;
                else { c++; i++; j++; }
            }
            sup[e] = c;
        }
    }
}

/*
 * NEXT-3: triangle enumeration ("we can get the listings of all the triangles for
 * free").  Every triangle {a,b,c} exactly once as the triple (a,b,c)
 * with a < b < c (input ids), in lexicographic order: for each a, each b in N(a)
 * with b > a, each c in N(a) cap N(b) with c > b.  Input: clean symmetric CSR with
 * sorted rows.  Writes at most `cap` triples (3 uint32 each) to out (nullable
 * when cap = 0) and returns the total number of triangles.
 */
uint64_t oracle_enumerate(uint64_t n, const uint64_t *crow, const uint32_t *ccol, uint32_t *out,
                          uint64_t cap) {
    uint64_t k = 0;
    for (uint64_t a = 0; a < n; a++) {
        for (uint64_t e = crow[a]; e < crow[a + 1]; e++) {
            uint64_t b = ccol[e];
            if (b <= a) continue;
            uint64_t i = crow[a], iend = crow[a + 1], j = crow[b], jend = crow[b + 1];
            while (i < iend && j < jend) {
                if (ccol[i] < ccol[j]) i++;
                else if (ccol[i] > ccol[j]) j++;
                else {
                    uint64_t c = ccol[i];
                    if (c > b) {
                        if (k < cap) {
                            out[3 * k + 0] = (uint32_t)a;
                            out[3 * k + 1] = (uint32_t)b;
                            out[3 * k + 2] = (uint32_t)c;
                        }
                        k++;
                    }
                    i++;
                    j++;
                }
            }
        }
    }
    return k;
}

/*
 * NEXT-4: Alg. 3 "Triangle_Count_Matrix" restricted to
 * A's nonzeros, its future-work "masking", written out step by step on a
 * clean symmetric CSR with sorted rows:
 *   line 1  permute: vertex order pi = increasing number of nonzeros (degree), ties by
 *           id -- or the identity when id_order != 0 (the order of Fig. mm);
 *   line 2  L_ij = A_ij if pi(i) > pi(j), U_ij = A_ij if pi(i) < pi(j), A = L + U;
 *   line 3  B = L U, i.e. B_ij = sum_k L_ik U_kj;
 *   line 4  C = A o B (Hadamard), evaluated at A's nonzeros only;
 *   line 5  n = (1/2) sum_ij C_ij (reading R7: the printed A_ij is C_ij).
 * Output: for every entry e = (i, col_plus[e]) of the upper triangle (off_plus /
 * col_plus as oracle_orient_order writes it, so pi(i) < pi(j)), c_values[e] = C_ij,
 * computed as the sum over k in row i of L (neighbours k of i with pi(k) < pi(i)) of
 * U_kj (A_kj = 1 and pi(k) < pi(j)).  Returns n.
 */
static int order_before(const uint64_t *rowptr, int id_order, uint64_t a, uint64_t b) {
    if (id_order) return a < b;
    return rank_less(rowptr, a, b);
}

/* oracle_orient with either order: N+(u) = { v in N(u) : pi(u) < pi(v) }, rows ascending. */
int64_t oracle_orient_order(uint64_t n, const uint64_t *rowptr, const uint32_t *col, int id_order,
                            uint64_t *off_plus, uint32_t *col_plus) {
    uint64_t k = 0;
    off_plus[0] = 0;
    for (uint64_t u = 0; u < n; u++) {
        for (uint64_t e = rowptr[u]; e < rowptr[u + 1]; e++)
            if (order_before(rowptr, id_order, u, col[e])) col_plus[k++] = col[e];
        off_plus[u + 1] = k;
    }
    return (int64_t)k;
}

uint64_t oracle_masked_spgemm(uint64_t n, const uint64_t *rowptr, const uint32_t *col, int id_order,
                              const uint64_t *off_plus, const uint32_t *col_plus,
                              uint32_t *c_values) {
    uint64_t sum = 0;
    for (uint64_t i = 0; i < n; i++) {
        for (uint64_t e = off_plus[i]; e < off_plus[i + 1]; e++) {
            uint64_t j = col_plus[e];
            uint32_t b = 0;                                   /* B_ij at a nonzero A_ij */
            for (uint64_t p = rowptr[i]; p < rowptr[i + 1]; p++) {
                uint64_t k = col[p];
                if (!order_before(rowptr, id_order, k, i)) continue;       /* L_ik = 0 */
                if (!order_before(rowptr, id_order, k, j)) continue;       /* U_kj = 0 */
                if (contains(col + rowptr[k], rowptr[k + 1] - rowptr[k], (uint32_t)j)) b++;
            }
            c_values[e] = b;                                  /* C_ij = A_ij * B_ij */
            sum += 2 * (uint64_t)b;                           /* C_ij and C_ji */
        }
    }
    return sum / 2;
}
