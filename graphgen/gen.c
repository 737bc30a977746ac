/*
 * graphgen/gen.c -- seeded synthetic input generators (shared by tests, the
 * oracle side and bench.py).  Holds NONE of the triangle-counting method's
 * arithmetic: it only draws arcs.  Cleaning (symmetrize / dedup / self-loop
 * removal) is step a1 of the method and is NOT done here -- outputs are raw
 * arc lists with duplicates, self-loops and one-directional arcs, exactly as
 * the generator draws them.
 *
 * Randomness: a counter-based generator (splitmix64 finaliser of a keyed
 * counter), so every draw is a pure function of (seed, stream, index) and
 * results do not depend on the OpenMP thread count.
 *
 * Shapes follow SURVEY.md §8(d) "Concrete synthetic inputs":
 *   R-MAT (Graph500 A,B,C,D = .57,.19,.19,.05 with integer thresholds),
 *   Chung-Lu (LiveJournal-like power law), road mesh (grid + diagonals),
 *   clique union (co-author-like), Kronecker powers of a small base graph.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t i) {
    uint64_t key = mix64(seed ^ mix64(stream + 0x632BE59BD9B4E019ull));
    return mix64(key + i * 0xD1B54A32D192ED03ull);
}

uint64_t gen_draw(uint64_t seed, uint64_t stream, uint64_t i) { return draw(seed, stream, i); }

/* Bijection on [0, 2^bits): odd multiply, add, xorshift -- each invertible mod 2^bits. */
static inline uint64_t perm_pow2(uint64_t x, uint32_t bits, uint64_t seed) {
    uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    uint64_t k1 = mix64(seed * 3 + 1) | 1, k2 = mix64(seed * 3 + 2) | 1, c = mix64(seed * 3 + 3);
    uint32_t r = bits / 2 + 1;
    for (int round = 0; round < 2; round++) {
        x = (x * k1 + c) & mask;
        x ^= x >> r;
        x = (x * k2) & mask;
        x ^= x >> (r > 1 ? r - 1 : 1);
    }
    return x & mask;
}

/* Bijection on [0, n) by cycle walking over the enclosing power of two. */
static inline uint64_t perm_n(uint64_t x, uint64_t n, uint64_t seed) {
    uint32_t bits = 1;
    while ((1ull << bits) < n) bits++;
    do { x = perm_pow2(x, bits, seed); } while (x >= n);
    return x;
}

uint64_t gen_perm(uint64_t x, uint64_t n, uint64_t seed) { return perm_n(x, n, seed); }

/*
 * R-MAT: npairs = ef * 2^scale arcs.  Per bit level a 32-bit draw r is compared
 * against floor(.57*2^32), floor(.76*2^32), floor(.95*2^32) -> quadrant
 * (0,0),(0,1),(1,0),(1,1).  Labels scrambled by a seeded bijection.
 */
void gen_rmat(uint32_t scale, uint64_t npairs, uint64_t seed, uint32_t *src, uint32_t *dst) {
    const uint32_t tA = 2448131358u, tAB = 3264175144u, tABC = 4080218931u;
    int64_t N = (int64_t)npairs;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < N; ii++) {
        uint64_t i = (uint64_t)ii, u = 0, v = 0;
        for (uint32_t lev = 0; lev < scale; lev++) {
            uint64_t d = draw(seed, 1, i * 32 + lev / 2);
            uint32_t r = (lev & 1) ? (uint32_t)(d >> 32) : (uint32_t)d;
            uint64_t bu = r >= tAB, bv = (r >= tA && r < tAB) || r >= tABC;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        src[i] = (uint32_t)perm_pow2(u, scale, seed);
        dst[i] = (uint32_t)perm_pow2(v, scale, seed);
    }
}

/* Inverse-CDF draw on a 62-bit fixed-point cumulative table cum[0..n) (cum[n-1] = 2^62). */
static inline uint64_t inv_cdf(const uint64_t *cum, uint64_t n, uint64_t r62) {
    uint64_t lo = 0, hi = n - 1;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (cum[mid] > r62) hi = mid; else lo = mid + 1;
    }
    return lo;
}

static void power_cum(uint64_t n, double alpha, double i0, uint64_t *cum) {
    double tot = 0.0;
    for (uint64_t i = 0; i < n; i++) tot += pow((double)i + i0, -alpha);
    double acc = 0.0, scale = 4611686018427387904.0; /* 2^62 */
    for (uint64_t i = 0; i < n; i++) {
        acc += pow((double)i + i0, -alpha);
        double c = acc / tot * scale;
        cum[i] = c >= scale ? (1ull << 62) : (uint64_t)c;
    }
    cum[n - 1] = 1ull << 62;
}

/* Chung-Lu: each endpoint i.i.d. with P(i) proportional to (i+i0)^-alpha; labels scrambled. */
int gen_chung_lu(uint64_t n, uint64_t npairs, double alpha, double i0, uint64_t seed,
                 uint32_t *src, uint32_t *dst) {
    uint64_t *cum = (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!cum) return -2;
    power_cum(n, alpha, i0, cum);
    int64_t N = (int64_t)npairs;
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < N; ii++) {
        uint64_t i = (uint64_t)ii;
        uint64_t a = inv_cdf(cum, n, draw(seed, 2, 2 * i) >> 2);
        uint64_t b = inv_cdf(cum, n, draw(seed, 2, 2 * i + 1) >> 2);
        src[i] = (uint32_t)perm_n(a, n, seed);
        dst[i] = (uint32_t)perm_n(b, n, seed);
    }
    free(cum);
    return 0;
}

/*
 * Road-like mesh on a W x H lattice, row-major ids.  Each lattice edge is kept
 * with probability p; each cell gets one diagonal with probability q ("\" or
 * "/" with probability 1/2).  Returns the number of arcs written (<= cap), or
 * -1 if cap is too small.  p = q = 1 ("all") gives the triangulated grid.
 */
int64_t gen_road_mesh(uint64_t W, uint64_t H, double p, double q, uint64_t seed,
                      uint32_t *src, uint32_t *dst, uint64_t cap) {
    uint64_t tp = p >= 1.0 ? ~0ull : (uint64_t)(p * 18446744073709551616.0);
    uint64_t tq = q >= 1.0 ? ~0ull : (uint64_t)(q * 18446744073709551616.0);
    uint64_t k = 0;
    for (uint64_t y = 0; y < H; y++) {
        for (uint64_t x = 0; x < W; x++) {
            uint64_t id = y * W + x;
            if (x + 1 < W && (p >= 1.0 || draw(seed, 3, 4 * id) < tp)) {
                if (k >= cap) return -1;
                src[k] = (uint32_t)id; dst[k] = (uint32_t)(id + 1); k++;
            }
            if (y + 1 < H && (p >= 1.0 || draw(seed, 3, 4 * id + 1) < tp)) {
                if (k >= cap) return -1;
                src[k] = (uint32_t)id; dst[k] = (uint32_t)(id + W); k++;
            }
            if (x + 1 < W && y + 1 < H && (q >= 1.0 || draw(seed, 3, 4 * id + 2) < tq)) {
                if (k >= cap) return -1;
                if (draw(seed, 3, 4 * id + 3) >> 63) {      /* "\" */
                    src[k] = (uint32_t)id; dst[k] = (uint32_t)(id + W + 1);
                } else {                                     /* "/" */
                    src[k] = (uint32_t)(id + 1); dst[k] = (uint32_t)(id + W);
                }
                k++;
            }
        }
    }
    return (int64_t)k;
}

/*
 * Clique union ("co-author-like"): G groups; group size s in [smin, smax] with
 * P(s) proportional to s^-gamma; members drawn with P(i) proportional to
 * (i+10)^-beta; each group becomes a clique (all s(s-1)/2 pairs; repeated
 * members give self-loops / duplicates, left for cleaning).
 * Two-phase: gen_clique_union_sizes() fills sizes[G] and returns the arc
 * total; gen_clique_union_fill() writes the arcs.
 */
static void size_cum(uint32_t smin, uint32_t smax, double gamma, uint64_t *cum) {
    uint64_t k = smax - smin + 1;
    double tot = 0.0;
    for (uint64_t i = 0; i < k; i++) tot += pow((double)(smin + i), -gamma);
    double acc = 0.0, scale = 4611686018427387904.0;
    for (uint64_t i = 0; i < k; i++) {
        acc += pow((double)(smin + i), -gamma);
        double c = acc / tot * scale;
        cum[i] = c >= scale ? (1ull << 62) : (uint64_t)c;
    }
    cum[k - 1] = 1ull << 62;
}

uint64_t gen_clique_union_sizes(uint64_t G, uint32_t smin, uint32_t smax, double gamma,
                                uint64_t seed, uint32_t *sizes) {
    uint64_t cum[4096];
    if (smax - smin + 1 > 4096) return 0;
    size_cum(smin, smax, gamma, cum);
    uint64_t tot = 0;
    for (uint64_t g = 0; g < G; g++) {
        uint32_t s = smin + (uint32_t)inv_cdf(cum, smax - smin + 1, draw(seed, 5, g) >> 2);
        sizes[g] = s;
        tot += (uint64_t)s * (s - 1) / 2;
    }
    return tot;
}

int gen_clique_union_fill(uint64_t n, uint64_t G, const uint32_t *sizes, double beta,
                          uint64_t seed, uint32_t *src, uint32_t *dst) {
    uint64_t *cum = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint64_t *start = (uint64_t *)malloc((G + 1) * sizeof(uint64_t));
    if (!cum || !start) { free(cum); free(start); return -2; }
    power_cum(n, beta, 10.0, cum);
    start[0] = 0;
    for (uint64_t g = 0; g < G; g++) start[g + 1] = start[g] + (uint64_t)sizes[g] * (sizes[g] - 1) / 2;
    int64_t GG = (int64_t)G;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t gg = 0; gg < GG; gg++) {
        uint64_t g = (uint64_t)gg;
        uint32_t s = sizes[g], mem[4096];
        for (uint32_t j = 0; j < s; j++)
            mem[j] = (uint32_t)perm_n(inv_cdf(cum, n, draw(seed, 6, g * 4096 + j) >> 2), n, seed);
        uint64_t k = start[g];
        for (uint32_t a = 0; a < s; a++)
            for (uint32_t b = a + 1; b < s; b++) { src[k] = mem[a]; dst[k] = mem[b]; k++; }
    }
    free(cum);
    free(start);
    return 0;
}

/*
 * Kronecker product of two arc lists: arc (a1,b1) of A and (a2,b2) of B give
 * arc (a1*nB + a2, b1*nB + b2).  Arc i of the output is (i / mB, i % mB).
 */
void gen_kron(uint64_t nB, uint64_t mA, const uint32_t *srcA, const uint32_t *dstA,
              uint64_t mB, const uint32_t *srcB, const uint32_t *dstB,
              uint32_t *src, uint32_t *dst) {
    int64_t N = (int64_t)(mA * mB);
#pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < N; ii++) {
        uint64_t i = (uint64_t)ii, a = i / mB, b = i % mB;
        src[i] = (uint32_t)(srcA[a] * nB + srcB[b]);
        dst[i] = (uint32_t)(dstA[a] * nB + dstB[b]);
    }
}

/*
 * Package arcs as a CSR grouped by source (counting sort, stable: arcs of a
 * row keep their draw order).  rowptr[n+1], col[npairs].  Returns -1 if an id
 * is >= n.  No dedup, no symmetrisation (that is the method's step a1).
 */
int gen_arcs_to_csr(uint64_t n, uint64_t npairs, const uint32_t *src, const uint32_t *dst,
                    uint64_t *rowptr, uint32_t *col) {
    memset(rowptr, 0, (n + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < npairs; i++) {
        if (src[i] >= n || dst[i] >= n) return -1;
        rowptr[src[i] + 1]++;
    }
    for (uint64_t v = 0; v < n; v++) rowptr[v + 1] += rowptr[v];
    uint64_t *cur = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!cur) return -2;
    memcpy(cur, rowptr, n * sizeof(uint64_t));
    for (uint64_t i = 0; i < npairs; i++) col[cur[src[i]]++] = dst[i];
    free(cur);
    return 0;
}
