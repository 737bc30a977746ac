/*
 * tc.h -- C ABI of libtc_b200.so, the B200 (sm_100a) exact triangle counter.
 *
 * The operation (§3.2, Alg. 2 "TC using edge-based set
 * intersection"; §4.2): for the simple undirected graph G that the
 * input arcs define, return
 *
 *     T(G) = |{ {a,b,c} : {a,b}, {b,c}, {a,c} are edges of G }|
 *
 * computed as in Alg. 2: orient every edge from lower to higher (degree, id)
 * rank and compact (Form_Filtered_Edge_List, filter rule P:520-523,
 * induced subgraph P:523-525), intersect N+(u) and N+(v) for every kept edge
 * (Compute_Intersection; "the number of triangles formed with e is
 * N") and reduce (Count = Reduce(IntersectList)).  Optional
 * per-vertex counts t(v) (number of triangles through v) serve clustering
 * coefficients and transitivity.
 *
 * Every step runs in hand-written sm_100a kernels; there is no CPU fallback.
 * All results are exact integers (uint64): the path has no floating point.
 *
 * INPUT LAYOUT (CSR, "Graph" of SPEC.md S:31-41):
 *   n            number of vertices, ids in [0, n), n < 2^32.
 *   m            number of arcs = row_offsets[n], m < 2^32 (TC_EINVAL otherwise:
 *                edge positions and slots are 32-bit).  Each arc is read as an
 *                undirected edge.
 *   row_offsets  uint64[n+1], row_offsets[0] = 0, non-decreasing,
 *                row_offsets[n] = m.
 *   col_indices  uint32[m]; arc k in row u is u -> col_indices[k].
 *   Unless TC_CLEAN is given, self-loops are dropped, duplicate and
 *   antiparallel arcs collapse to one edge, and one-directional arcs are
 *   symmetrised (Table 1 caption P:604-606).  Isolated vertices are allowed.
 *
 * POINTERS: by default all array pointers are DEVICE pointers on the current
 * CUDA device; with TC_HOST_PTRS they are HOST pointers (pinned memory gives
 * the fastest copies) and the library copies them in and results out.
 * Inputs are borrowed, read-only, and must stay valid for the call.
 *
 * OWNERSHIP: outputs are caller-allocated.  Device workspace comes from
 * tc_options.alloc / .free when the caller supplies them (the Python
 * binding passes torch's caching allocator), called on the call's stream and every
 * block freed before the call returns (stream-ordered: a block is released with the
 * stream that may still use it, exactly like cudaFreeAsync).  Without a hook the
 * workspace comes from a memory pool the LIBRARY creates per device (never the
 * process's default pool); with tc_options.keep_workspace = 1 (the default) that pool
 * keeps freed memory for the next call, tc_trim_workspace() returns it to the driver.
 * tc_count / tc_count_ex / tc_orient are synchronous (they return once results are
 * on their destination); tc_count_shard is stream-ordered (its device result is
 * ready when the stream reaches it).
 *
 * ERRORS: every entry point validates its arguments (null pointers, n >= 2^32,
 * unknown flag bits, bad options) and returns TC_EINVAL before
 * touching the device.  With TC_VALIDATE the graph itself is checked on the
 * device (offsets, ids, and for TC_CLEAN: no self-loops, symmetry, and with
 * TC_SORTED strictly increasing rows) and a violation returns TC_EGRAPH.
 * Without TC_VALIDATE a malformed graph, or a false TC_CLEAN / TC_SORTED
 * claim, is undefined behaviour.  CUDA failures return TC_ECUDA, allocation
 * failures TC_ENOMEM.  tc_last_error() gives a thread-local message.
 *
 * DEVICE: device pointers must belong to the current CUDA device (checked:
 * TC_EINVAL otherwise); all work runs there.
 *
 * THREAD SAFETY: calls on different streams or devices are independent.  Global
 * state: the thread-local error string and pinned read-back scratch, a per-thread
 * side stream per device, the per-device SM count and the per-device library
 * workspace pool (both created once, under a lock).
 */
#ifndef TC_B200_H
#define TC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ERROR UINT64_MAX /* tc_count's failure value (unreachable as a count) */

enum {
    TC_CLEAN = 1u << 0,      /* input is already simple and symmetric: no self-loops, no
                                duplicate arcs, (u,v) present iff (v,u).  Skips step a1.    */
    TC_SORTED = 1u << 1,     /* with TC_CLEAN: every row ascending (checked by TC_VALIDATE)   */
    TC_PER_VERTEX = 1u << 2, /* fill per_vertex[n] with t(v)                                  */
    TC_HOST_PTRS = 1u << 3,  /* all arrays are host pointers                                   */
    TC_VALIDATE = 1u << 4,   /* check the graph on the device; TC_EGRAPH on violation          */
    TC_PRUNE = 1u << 5,      /* NEXT-2 leaf pruning before orientation ("nodes with degree less
                                than two cannot be matched"; repeated "for a few
                                iterations"): each round deletes every edge with an
                                endpoint of degree < 2 in the current graph; rounds =
                                tc_options.prune_rounds, 0 = until a round deletes nothing
                                (the 2-core).  T and t(v) are unchanged (every vertex of a
                                triangle keeps degree >= 2); ranks use the PRUNED degrees, so
                                tc_orient returns the oriented pruned graph.  Not allowed with
                                tc_clustering (c(v) needs the unpruned degrees).             */
    TC_ID_ORDER = 1u << 6,   /* orient by vertex id instead of (degree, id): N+(u) = {v in N(u) :
                                v > u}, the order of the paper's Fig. mm example (Alg. 3 without
                                its row permutation).  Counts are unchanged; slower
                                on skewed graphs (d+ is no longer bounded by sqrt(2m)).         */
    TC_ALL_FLAGS = 0x7fu
};

typedef enum {
    TC_OK = 0,
    TC_EINVAL = 1, /* bad argument                          */
    TC_EGRAPH = 2, /* malformed graph (under TC_VALIDATE)   */
    TC_ENOMEM = 3, /* device allocation failed              */
    TC_ECUDA = 4   /* CUDA launch / runtime failure          */
} tc_status;

/* Intersection variants (§4.2.2 P:527-542 "dynamic grouping"; third kernel P:704-708). */
enum {
    TC_VARIANT_AUTO = -1,
    TC_VARIANT_SHORT = 0,  /* one thread per edge, two-pointer merge ("TwoSmall")      */
    TC_VARIANT_MERGE = 1,  /* one warp per edge, merge-path split ("TwoLarge"/balanced path,
                              P:534-539)                                                      */
    TC_VARIANT_SEARCH = 2, /* short list binary-searched in the long one           */
    TC_VARIANT_HASH = 3    /* the shorter of N+(u), N+(v) probed into a shared-memory hash of
                              the longer; edges grouped by the longer list's vertex (owner):
                              a warp per small owner, a CTA per hub owner (north_star)        */
};

/* Workspace allocator hook.  alloc returns `bytes` of device memory on
 * the current device usable in stream order on `stream` (NULL on failure -> TC_ENOMEM);
 * free releases a block returned by alloc, stream-ordered on `stream` (the block may
 * still be read by work enqueued on `stream` before the call).  `ctx` is alloc_ctx. */
typedef void *(*tc_alloc_fn)(void *ctx, size_t bytes, void *stream);
typedef void (*tc_free_fn)(void *ctx, void *ptr, void *stream);

typedef struct {
    uint32_t short_max;         /* AUTO: edge -> SHORT if max(d+u, d+v) <= short_max           */
    uint32_t skew_ratio;        /* AUTO: edge -> SEARCH if max >= skew_ratio * min (0 = never)  */
    uint32_t hub_min_dplus;     /* HASH owners with d+ >= this get a whole CTA (capped at 129)  */
    int32_t force_variant;      /* TC_VARIANT_AUTO, or route EVERY edge to one variant          */
    void *stream;               /* cudaStream_t to run on; NULL = legacy default stream         */
    uint32_t prune_rounds;      /* TC_PRUNE: rounds to run; 0 = to the fixed point (one 8-byte
                                   device->host read per round)                               */
    uint32_t keep_workspace;    /* no hook: 1 = the library pool keeps freed workspace for the
                                   next call (default), 0 = release it when the call ends     */
    tc_alloc_fn alloc;          /* workspace hook (both or neither); NULL = library pool       */
    tc_free_fn free;
    void *alloc_ctx;            /* passed to alloc / free                                       */
    uint32_t tiny_max_n;        /* tc_count / tc_count_ex / tc_count_shard on graphs with
                                   n <= min(tiny_max_n, 1024) (AUTO, no TC_PRUNE / TC_ID_ORDER):
                                   the whole method in ONE kernel on a shared-memory adjacency
                                   bitmap (small graphs are launch-bound); 0 = off.
                                   Default 1024.  Stats then carry m_undirected and times only */
    uint32_t clean_method;      /* a1 on dirty input (no TC_CLEAN) and tc_clean_shard: the arcs
                                   become 64-bit (min, max) keys, radix-sorted, then unique.
                                   0 (default) = sorted by a hash of the key in its low 24/32
                                   bits only (3-4 passes; duplicates share a run of equal
                                   hash), 1 = sorted in full (min, max) order (6-8 passes).
                                   Same results                                                */
    uint32_t graph_cache;       /* 1 = tc_count / tc_count_ex on device pointers (no stats,
                                   TC_PRUNE, TC_VALIDATE or allocator hook) is captured into a
                                   CUDA graph on first use and REPLAYED by later calls with the
                                   same arguments (sizes, pointers, flags, options; per thread,
                                   up to 4 graphs): one graph launch instead of ~36 kernels and
                                   ~60 workspace allocations -- for launch-bound small and
                                   mid-size graphs.  The graph keeps its workspace reserved
                                   between calls.  0 (default) = off                           */
    uint32_t lowdeg_max;        /* tc_count / tc_count_ex (plain or per-vertex counts, AUTO, no
                                   TC_PRUNE / TC_ID_ORDER / graph_cache, m <= 8n arcs) on graphs
                                   whose every vertex has at most min(lowdeg_max, 32) arc
                                   incidences (road networks, meshes: P:700-702's filter-bound
                                   regime): the bounded-degree path (lowdeg.cu), a thread per
                                   vertex cleans, orients and intersects its lists in local
                                   memory -- 5-6 kernels instead of ~40.  Eligibility is tested
                                   on the device and read back once (one extra synchronisation;
                                   a graph that fails takes the general pipeline).  Stats then
                                   carry m_undirected, work_W, work_probe, max_dplus,
                                   work_stage, skipped_edges, bin_edges[SHORT] (the rest of the
                                   edges) and times.  Default 32; 0 = off                      */
    uint32_t reserved[5];       /* must be zero                                                 */
} tc_options;

typedef struct {
    /* phase times (ms, CUDA events on the call's stream); 0 when the phase did not run */
    double ms_clean;     /* a1: keys, radix sort, unique                                   */
    double ms_orient;    /* a2+a3: degrees, rank filter, compaction into N+ CSR            */
    double ms_sort;      /* a4: reported inside ms_orient (the two-key sort); always 0     */
    double ms_bin;       /* a5: work estimation + binning                                  */
    double ms_intersect; /* a6+a7: intersection kernels and the per-block reduction        */
    double ms_total;     /* whole call, including host<->device copies with TC_HOST_PTRS   */
    uint64_t m_undirected;    /* simple undirected edges = |E+|                             */
    uint64_t work_W;          /* sum over E+ of d+(u) + d+(v)   (merge work)                */
    uint64_t work_probe;      /* sum over E+ of min(|N+(u) after v|, d+v) (HASH probe work)  */
    uint64_t bytes_alg;       /* 4*W + 16*m: algorithmic bytes of the intersection (B_alg)  */
    uint64_t bin_edges[4];    /* edges routed to SHORT, MERGE, SEARCH, HASH                 */
    uint64_t skipped_edges;   /* edges that cannot close a triangle (|N+(u) after v| = 0 or
                                 d+(v) = 0)                                                 */
    uint64_t hub_sources;     /* HASH owners handled by a whole CTA (d+ >= hub_min_dplus)   */
    uint64_t max_dplus;       /* max out-degree after orientation                           */
    uint64_t kernel_launches; /* kernels this call launched                                 */
    uint64_t h2d_bytes;       /* bytes copied host->device (TC_HOST_PTRS)                   */
    uint64_t d2h_bytes;       /* bytes copied device->host                                   */
    uint64_t table_loads;     /* HASH: sum over owner tasks of d+(owner) (table builds)      */
    uint64_t bytes_hash;      /* HASH algorithmic bytes: 4*(probes of the HASH / SHORT edges)
                                 + 8*HASH edges + 4*table_loads (the a6 byte model)       */
    double ms_prune;          /* TC_PRUNE: the pruning rounds (inside ms_orient)             */
    uint64_t pruned_edges;    /* TC_PRUNE: undirected edges deleted                          */
    uint64_t prune_rounds;    /* TC_PRUNE: rounds executed (fixed-point mode: including the
                                 final round that deleted nothing)                         */
    uint64_t work_stage;      /* sum_v d-(v) d+(v): SURVEY 8(d)'s B_stage = 4(m + this) + 16m  */
    uint64_t core_edges;      /* edges counted by the dense-core bitmap path (plain counts)    */
    uint64_t core_words;      /* 32-bit word ANDs they took (work_probe still counts their
                                 HASH-equivalent probes)                                     */
    uint64_t bytes_core;      /* 8 * core_words: the core path's algorithmic bytes           */
} tc_stats;

/* Fill *opt with the defaults (auto variant selection, default stream). */
void tc_default_options(tc_options *opt);

/* Triangle count, or TC_ERROR (reason in tc_last_error()).  Default options. */
uint64_t tc_count(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                  const uint32_t *col_indices, uint32_t flags);

/* Full form.  total: host uint64 (always host).  per_vertex: n entries on the
 * pointer side given by TC_HOST_PTRS, required iff TC_PER_VERTEX.  opt and
 * stats are host structs and may be NULL. */
tc_status tc_count_ex(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                      const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                      uint64_t *total, uint64_t *per_vertex, tc_stats *stats);

/* Multi-GPU shard: every rank passes the SAME graph; the library runs the
 * (replicated) preprocessing and binning, then splits the intersection work: HASH work by
 * OWNER (the vertex whose N+ is staged as the table; owners are cut into `world` contiguous
 * groups of equal estimated work -- probe lengths + 64 per probe entry + the table builds --
 * by a prefix sum, so every table is built on exactly one rank) and the SHORT / MERGE /
 * SEARCH edges by CSR edge range.  No communication is needed for the split; every
 * triangle is counted on exactly one rank.  partial_dev (device, 1
 * entry) is OVERWRITTEN with this rank's partial count; per_vertex_partial
 * (device, n entries, nullable unless TC_PER_VERTEX) is overwritten with this
 * rank's per-vertex contributions.  Summing over ranks (one allreduce) gives
 * exactly tc_count's results.  TC_HOST_PTRS is not allowed here.  Returns
 * once the work is enqueued on opt->stream (stream-ordered). */
tc_status tc_count_shard(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                         const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                         int rank, int world, uint64_t *partial_dev,
                         uint64_t *per_vertex_partial, tc_stats *stats);

/* Sharded a1 for multi-GPU runs (the cleaning step, Table 1 caption P:604-606,
 * split over the ranks instead of repeated on each).  Every rank passes the SAME raw CSR
 * (device pointers; n, m as in tc_count) and cleans only the arcs of ITS undirected edges:
 * those whose smaller endpoint v has v % world == rank (every copy of an edge lands on one
 * rank).  Output: edges[0 .. *m_edges) (device, capacity m) = this rank's unique undirected
 * edges as keys (min << b) | max with b = the bit width of n - 1 (at least 1), in an
 * unspecified order (ascending with tc_options.clean_method = 1);
 * degrees (device, n entries, overwritten) = the degrees those edges give their endpoints;
 * *m_edges (host).  The caller all-reduces (sums) the degrees and concatenates the ranks'
 * edges (any order), then calls tc_count_edges_shard.  No flags.  Synchronous. */
tc_status tc_clean_shard(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                         const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                         int rank, int world, uint64_t *edges, uint32_t *degrees,
                         uint64_t *m_edges);

/* tc_count_shard's work from a cleaned edge list: edges (device, m_edges keys as
 * tc_clean_shard writes them, every rank's, any order, each undirected edge once) and
 * degrees (device, n: the full degrees, e.g. the all-reduced tc_clean_shard outputs);
 * partial_dev / per_vertex_partial as tc_count_shard (summing over ranks gives tc_count's
 * results).  Flags: TC_PER_VERTEX, TC_ID_ORDER.  Stream-ordered like tc_count_shard. */
tc_status tc_count_edges_shard(uint64_t n, uint64_t m_edges, const uint64_t *edges,
                               const uint32_t *degrees, uint32_t flags, const tc_options *opt,
                               int rank, int world, uint64_t *partial_dev,
                               uint64_t *per_vertex_partial, tc_stats *stats);

/* ---- Sharded pipeline (round 2): a2-a5 split over the ranks as well (north_star
 * "the edge range is split by a prefix sum over estimated intersection work, followed by one
 * NCCL allreduce of the 64-bit count").  After tc_clean_shard + the degree all-reduce, each
 * rank runs the six phases below; between them the CALLER runs the collective named in
 * brackets (paper_1804_06926_b200/dist.py: NCCL; shard.py: a one-GPU emulation).  All
 * pointers are device pointers on the current device unless marked host; outputs are
 * caller-owned and overwritten; every phase is synchronous.  world <= 64; n < 2^30 and fewer
 * than 2^31 oriented edges; force_variant must be AUTO.  The buffers passed from one phase to
 * the next are trusted (produced by the previous phase and the collective); sizes named by the
 * caller (m_recv, col_begin, n_entries) must be the ones those produced.  Summing the ranks' partials gives
 * tc_count's total (and, with TC_PER_VERTEX, its t(v)) exactly.
 *
 * tc_shard_orient: newid (n) = the rank relabelling of Alg. 2 (rank = (d, id)) from
 *   the summed degrees; the rank's own unique edges (tc_clean_shard's) oriented low -> high
 *   rank as (src[i], dst[i]) rank ids; dplus (n) = the d+ they contribute.  Flags: TC_ID_ORDER.
 *   [all-reduce dplus] */
tc_status tc_shard_orient(uint64_t n, uint64_t m_local, const uint64_t *edges, const uint32_t *degrees,
                          uint32_t flags, const tc_options *opt, uint32_t *newid, uint32_t *src,
                          uint32_t *dst, uint32_t *dplus);
/* tc_shard_partition: off_plus (n+1) = the exclusive scan of the summed dplus (the oriented
 *   CSR's row offsets, identical on every rank); row range q = rank ids [row_bounds[q],
 *   row_bounds[q+1]) holding about m/world edges, col+ positions [col_bounds[q], col_bounds[q+1])
 *   (host arrays, world+1 entries); pairs_out (m_local, int64 src | dst << 32) = the rank's pairs
 *   grouped by the range of their source, send_counts (host, world) per range.
 *   [all-to-all of the pairs by send_counts] */
tc_status tc_shard_partition(uint64_t n, uint64_t m_local, const uint32_t *src, const uint32_t *dst,
                             const uint32_t *dplus, const tc_options *opt, int rank, int world,
                             uint64_t *off_plus, uint64_t *pairs_out, uint64_t *send_counts,
                             uint64_t *row_bounds, uint64_t *col_bounds);
/* tc_shard_rows: the m_recv received pairs (exactly the rows of this rank's range) sorted by
 *   (source, target) into col_plus[col_begin, col_begin + m_recv): rows ascending (a3 + a4).
 *   [all-gather: each rank's col+ range to every rank] */
tc_status tc_shard_rows(uint64_t n, uint64_t m_recv, const uint64_t *pairs, const tc_options *opt,
                        uint64_t col_begin, uint32_t *col_plus);
/* tc_shard_work: a5 on this rank's rows [row_begin, row_end) = oriented edges [e_begin, e_end)
 *   (only this rank's slice of col_plus is read, so the col+ all-gather may still be in
 *   flight): ent_cnt (n) / ent_len (n, uint64) = per HASH owner the probe entries and probe
 *   lengths these edges give it (bin.cu's rule: owner = target if |N+(u) after x| <= d+(x),
 *   else source); spans (n) = last - first + 1 of N+(x) for its rows, 0 elsewhere.  Flags:
 *   TC_PER_VERTEX (then the dense core is off).  [all-reduce ent_cnt, ent_len, spans] */
tc_status tc_shard_work(uint64_t n, const uint64_t *off_plus, const uint32_t *col_plus, const uint32_t *dplus,
                        uint32_t flags, const tc_options *opt, uint64_t row_begin, uint64_t row_end,
                        uint64_t e_begin, uint64_t e_end, uint32_t *ent_cnt, uint64_t *ent_len,
                        uint32_t *spans);
/* tc_shard_route: owner work w(x) from the summed entries / lengths / spans (the single-GPU
 *   owner split's model), its exclusive prefix, owner x -> rank split_rank(prefix(x));
 *   entries_out = the HASH probe entries of edges [e_begin, e_end) grouped by their owner's rank,
 *   three uint32 each (owner, other endpoint, CSR index | out-part flag << 31), with this rank's
 *   SHORT / SEARCH edges routed to itself (owner field = source | 1 << 31, then the target, the
 *   CSR index | SEARCH flag << 31); send_counts (host, world) entries per rank.  Reads only this
 *   rank's slice of col_plus.  Same flags as tc_shard_work.  [all-to-all of the entries] */
tc_status tc_shard_route(uint64_t n, const uint64_t *off_plus, const uint32_t *col_plus, const uint32_t *dplus,
                         const uint32_t *ent_cnt, const uint64_t *ent_len, const uint32_t *spans, uint32_t flags,
                         const tc_options *opt, int rank, int world, uint64_t e_begin, uint64_t e_end,
                         uint32_t *entries_out, uint64_t *send_counts);
/* tc_shard_count: a6 + a7 of this rank (needs the whole col_plus): its HASH owners' tables
 *   probed with the n_entries received entries, its SHORT / SEARCH edges (received from itself),
 *   the dense-core edges of its interleaved 2048-edge blocks (count mode); n < 2^30.  *partial_dev (uint64) = its share; with
 *   TC_PER_VERTEX (needs newid) per_vertex_partial (n, input ids) = its t(v) shares.  m = the
 *   oriented edge count (off_plus[n]).  ms_a6 (host, nullable): the a6 + a7 kernels' CUDA-event
 *   span (the owner-structure build excluded).  [all-reduce partial_dev (and per_vertex_partial)] */
tc_status tc_shard_count(uint64_t n, uint64_t m, const uint64_t *off_plus, const uint32_t *col_plus,
                         const uint32_t *dplus, const uint32_t *newid, uint64_t n_entries,
                         const uint32_t *entries, uint32_t flags, const tc_options *opt, int rank,
                         int world, uint64_t e_begin, uint64_t e_end, uint64_t *partial_dev,
                         uint64_t *per_vertex_partial, double *ms_a6);

/* Steps a1-a4 only ("Form_Filtered_Edge_List", Alg. 2): writes the
 * oriented, compacted CSR N+ (off_plus: n+1 entries; col_plus: capacity m
 * entries, first m_plus used; each row ascending) and *m_plus (host).
 * Pointer side per TC_HOST_PTRS.  Used by the parity tests of those steps. */
tc_status tc_orient(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                    const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                    uint64_t *off_plus, uint32_t *col_plus, uint64_t *m_plus);

/* NEXT-1: "with little modification ... clustering coefficient
 * and transitivity".  With t(v) the per-vertex triangle count
 * and d(v) the degree of the cleaned graph (reading R14):
 *   local_cc[v]    = 2 t(v) / (d(v) (d(v) - 1)), 0 when d(v) < 2       (double, n entries)
 *   wedges         = sum_v d(v) (d(v) - 1) / 2   (connected triples, exact uint64)
 *   transitivity   = 3 T / wedges, 0 when wedges = 0
 *   avg_clustering = (1/n) sum_v local_cc[v] over all n vertices (isolated ones give 0)
 * Each local_cc[v] and the transitivity are ONE correctly rounded fp64 division of
 * exact integers; avg_clustering is an fp64 sum (deterministic order for a given
 * device, not the oracle's order).  Flags: TC_CLEAN, TC_SORTED, TC_HOST_PTRS,
 * TC_VALIDATE (TC_PER_VERTEX is implied).  local_cc and per_vertex (uint64 t(v))
 * are optional outputs (NULL = not wanted) on the TC_HOST_PTRS side; summary and
 * stats are host structs (nullable).  Synchronous. */
typedef struct {
    uint64_t triangles;     /* T */
    uint64_t wedges;        /* sum_v C(d(v), 2) */
    double transitivity;    /* 3T / wedges */
    double avg_clustering;  /* mean of local_cc over all n vertices */
} tc_clustering_summary;

tc_status tc_clustering(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                        const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                        double *local_cc, uint64_t *per_vertex, tc_clustering_summary *summary,
                        tc_stats *stats);

/* NEXT-3: edge support, the k-truss input ("enumerating triangles is
 * useful as a subroutine in solving k-truss").  sup({u,v}) = number of triangles
 * containing the edge = |N(u) cap N(v)|.  Every triangle found by the a6 kernels credits
 * its three edges (its base edge, and the two edges through the match w, located by
 * their col+ slot / the owner's table position).  Output: the oriented CSR exactly as
 * tc_orient returns it (input ids, each undirected edge once, rows ascending; off_plus
 * n+1 entries, col_plus capacity m entries, *m_plus edges used) and support[e] for each
 * of its entries (capacity m, uint32).  Pointer side per TC_HOST_PTRS (m_plus: host).
 * Flags: TC_CLEAN, TC_SORTED, TC_HOST_PTRS, TC_VALIDATE, TC_PRUNE (pruned edges have
 * support 0 and are not listed).  sum_e support[e] = 3T.  Synchronous. */
tc_status tc_edge_support(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                          const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                          uint64_t *off_plus, uint32_t *col_plus, uint32_t *support,
                          uint64_t *m_plus, tc_stats *stats);

/* NEXT-3: triangle enumeration ("we can get the listings of all the triangles for
 * free").  Writes each triangle {a,b,c} once as three uint32 input ids
 * a < b < c into triangles[3k .. 3k+2], for min(T, capacity) triangles, in an
 * UNSPECIFIED order (slots are reserved by atomic counters; the set is deterministic
 * when capacity >= T), and sets *total (host) = T.  If T > capacity an unspecified
 * subset of `capacity` triangles is written: call again with capacity >= *total.
 * capacity = 0 (triangles may be NULL) only counts.  triangles is on the TC_HOST_PTRS
 * side (host mode stages min(T, capacity) triples in device memory).  Flags: TC_CLEAN,
 * TC_SORTED, TC_HOST_PTRS, TC_VALIDATE, TC_PRUNE.  Synchronous. */
tc_status tc_enumerate(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                       const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                       uint32_t *triangles, uint64_t capacity, uint64_t *total, tc_stats *stats);

/* NEXT-4: the matrix formulation as a front end on the same
 * intersection core (Alg. 3 "Triangle_Count_Matrix", and its future-work
 * "masking" P:723-731: no materialised B, only A's nonzeros, upper triangle only,
 * P:557-561).  With the vertices in rank order (Alg. 3 line 1: rows "ordered by an
 * increasing number of nonzeros", ties by id; or id order under TC_ID_ORDER, the
 * order of Fig. mm), A = L + U and
 *     C = A o (L U),   C_ij = #{ k : k before i and before j, A_ik = A_kj = 1 }
 * for every nonzero A_ij -- the number of triangles whose two LATEST vertices are i, j.
 * Output: the upper triangle (each undirected edge once) in the layout of tc_orient
 * (input ids, rows ascending; off_plus n+1, col_plus capacity m, *nnz_u used) with
 * c_values[e] = C at that entry (C is symmetric), and *total = (1/2) sum_ij C_ij = T
 * (Alg. 3 line 6; R7: the printed "A_ij" there is read as C_ij).  Pointer side per
 * TC_HOST_PTRS (nnz_u, total: host).  Flags: TC_CLEAN, TC_SORTED, TC_HOST_PTRS,
 * TC_VALIDATE, TC_PRUNE, TC_ID_ORDER.  Synchronous. */
tc_status tc_masked_spgemm(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                           const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                           uint64_t *off_plus, uint32_t *col_plus, uint32_t *c_values,
                           uint64_t *nnz_u, uint64_t *total, tc_stats *stats);

/* Thread-local message describing the last failure on this thread ("" if none). */
/* Kernels launched so far by the calls made from this thread (all entry points; a
 * monotone counter for launch accounting, e.g. bench.py's gpu_launches). */
uint64_t tc_launches_issued(void);

const char *tc_last_error(void);

/* Return the library pool's cached workspace on `device` (-1 = current device) to the
 * driver, and drop the calling thread's replay graphs of that device (graph_cache) with the
 * graph memory they reserved (synchronises the device).  Calls in flight keep what they hold. */
tc_status tc_trim_workspace(int device);

/* Library version string. */
const char *tc_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TC_B200_H */
