// tc_api.cu -- the C ABI (include/tc.h): argument checks, workspace, stream,
// host<->device staging, and the phase sequence of Alg. 2:
//   Form_Filtered_Edge_List (a1-a4) -> Partition (a5) -> intersections (a6)
//   -> Reduce (a7, fused).  The whole sequence is stream-ordered: no host
//   synchronisation until the 8-byte count is read back.
#include <cstdio>
#include <cstring>
#include <mutex>

#include "tc_internal.cuh"

namespace tc {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

uint64_t &thread_launches() {
    static thread_local uint64_t n = 0;
    return n;
}

// Per-device state created once under a lock: the SM count and the library's own
// workspace pool (never the process's default pool, which torch / NCCL may rely on).
struct DeviceState {
    int sms = 0;
    cudaMemPool_t pool = nullptr;
};
static std::mutex g_dev_mu;
static DeviceState g_dev[64];

static DeviceState &device_state(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (dev < 0 || dev >= 64) throw Error{TC_EINVAL, "device index out of range"};
    DeviceState &d = g_dev[dev];
    if (!d.sms) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        d.sms = v;
    }
    if (!d.pool) {
        cudaMemPoolProps props;
        memset(&props, 0, sizeof(props));
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        TC_CUDA(cudaMemPoolCreate(&d.pool, &props));
    }
    return d;
}

static void set_pool_keep(cudaMemPool_t pool, bool keep) {
    uint64_t thr = keep ? UINT64_MAX : 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

// 32 uint64 of pinned host memory per thread for asynchronous stat read-back.
static uint64_t *pinned_scratch() {
    static thread_local uint64_t *p = nullptr;
    if (!p) TC_CUDA(cudaMallocHost((void **)&p, 64 * sizeof(uint64_t)));   // [32, 40): lowdeg
    return p;
}

// A false TC_CLEAN claim (more arcs passed the rank filter than a simple symmetric graph
// has edges) is detected on the device; the kernels clamp every write, and the call reports
// TC_EGRAPH once it has synchronised (tc_count_shard: only when stats are requested).
static void check_claim(const uint64_t *pin) {
    if ((uint32_t)pin[26])
        throw Error{TC_EGRAPH, "TC_CLEAN claim is false: more arcs passed the rank filter than "
                               "m/2 (the input is not simple and symmetric)"};
}

enum Mode { kCount, kShard, kOrientOnly, kClustering, kSupport, kEnumerate, kMasked, kCleanShard };

struct Call {
    uint64_t n, M;
    const uint64_t *rowptr;
    const uint32_t *col;
    uint32_t flags;
    tc_options opt;
    int rank = 0, world = 1;
    Mode mode = kCount;
    // outputs
    uint64_t *total_host = nullptr;   // kCount
    uint64_t *partial_dev = nullptr;  // kShard
    uint64_t *per_vertex = nullptr;
    tc_stats *stats = nullptr;
    uint64_t *off_plus = nullptr;     // kOrientOnly
    uint32_t *col_plus = nullptr;
    uint64_t *m_plus = nullptr;
    double *cc = nullptr;             // kClustering (nullable)
    tc_clustering_summary *csum = nullptr;
    uint32_t *support = nullptr;      // kSupport (with off_plus / col_plus / m_plus)
    uint32_t *triangles = nullptr;    // kEnumerate: capacity triples
    uint64_t capacity = 0;
    // kShard from a sharded a1 (tc_count_edges_shard): the unique edges and their degrees
    const uint64_t *edges_in = nullptr;
    const uint32_t *deg_in = nullptr;
    // kCleanShard (tc_clean_shard): this rank's unique edges, degree partials, edge count
    uint64_t *edges_out = nullptr;
    uint32_t *deg_out = nullptr;
    uint64_t *m_edges_out = nullptr;
};

static tc_status check_args(const Call &c) {
    if (c.flags & ~(uint32_t)TC_ALL_FLAGS) return set_error("unknown flag bits"), TC_EINVAL;
    if (c.mode == kCleanShard || c.edges_in) {   // the sharded-a1 pair (tc.h)
        if (c.world < 1 || c.rank < 0 || c.rank >= c.world)
            return set_error("need 0 <= rank < world"), TC_EINVAL;
        if (c.n >= (1ull << 32) || c.M >= (1ull << 32))
            return set_error("n and m must be < 2^32"), TC_EINVAL;
        const uint32_t allowed = c.mode == kCleanShard ? 0u : (uint32_t)(TC_PER_VERTEX | TC_ID_ORDER);
        if (c.flags & ~allowed) return set_error("flag not supported by this entry point"), TC_EINVAL;
        if (c.mode == kCleanShard && (!c.rowptr || (c.M && !c.col) || !c.edges_out || !c.deg_out ||
                                      !c.m_edges_out))
            return set_error("tc_clean_shard: NULL argument"), TC_EINVAL;
        if (c.edges_in && (!c.deg_in || !c.partial_dev || ((c.flags & TC_PER_VERTEX) && !c.per_vertex)))
            return set_error("tc_count_edges_shard: NULL argument"), TC_EINVAL;
        if (c.opt.force_variant < -1 || c.opt.force_variant > 3)
            return set_error("force_variant out of range"), TC_EINVAL;
        if (!c.opt.alloc != !c.opt.free)
            return set_error("tc_options.alloc and .free must be given together"), TC_EINVAL;
        return TC_OK;
    }
    if (c.n >= (1ull << 32)) return set_error("n must be < 2^32"), TC_EINVAL;
    if (c.M >= (1ull << 32))   // edge positions, in-list slots and probe ranges are 32-bit
        return set_error("m (arcs) must be < 2^32"), TC_EINVAL;
    if (!c.rowptr) return set_error("row_offsets is NULL"), TC_EINVAL;
    if (c.M > 0 && !c.col) return set_error("col_indices is NULL with m > 0"), TC_EINVAL;
    if (c.mode == kCount && !c.total_host) return set_error("total is NULL"), TC_EINVAL;
    if (c.mode == kClustering && (c.flags & TC_PER_VERTEX))
        return set_error("tc_clustering: TC_PER_VERTEX is implied (pass per_vertex or NULL)"), TC_EINVAL;
    if (c.mode == kClustering && (c.flags & TC_PRUNE))
        return set_error("tc_clustering: TC_PRUNE would change the degrees d(v) of c(v)"), TC_EINVAL;
    if (c.mode == kShard) {
        if (!c.partial_dev) return set_error("partial_dev is NULL"), TC_EINVAL;
        if (c.world < 1 || c.rank < 0 || c.rank >= c.world)
            return set_error("need 0 <= rank < world"), TC_EINVAL;
        if (c.flags & TC_HOST_PTRS) return set_error("tc_count_shard takes device pointers"), TC_EINVAL;
    }
    const bool csr_out = c.mode == kOrientOnly || c.mode == kSupport || c.mode == kMasked;
    if (csr_out && (!c.off_plus || (!c.col_plus && c.M > 0) || !c.m_plus))
        return set_error("tc_orient / tc_edge_support / tc_masked_spgemm output pointer is NULL"),
               TC_EINVAL;
    if ((c.mode == kSupport || c.mode == kMasked) && !c.support && c.M > 0)
        return set_error("tc_edge_support / tc_masked_spgemm: value output is NULL"), TC_EINVAL;
    if (c.mode == kMasked && !c.total_host)
        return set_error("tc_masked_spgemm: total is NULL"), TC_EINVAL;
    if (c.mode == kEnumerate && (!c.total_host || (c.capacity && !c.triangles)))
        return set_error("tc_enumerate: total is NULL, or triangles is NULL with capacity > 0"),
               TC_EINVAL;
    if ((c.mode == kSupport || c.mode == kEnumerate || c.mode == kMasked) && (c.flags & TC_PER_VERTEX))
        return set_error("TC_PER_VERTEX is not an option of tc_edge_support / tc_enumerate / "
                         "tc_masked_spgemm"),
               TC_EINVAL;
    if ((c.flags & TC_PER_VERTEX) && c.mode != kOrientOnly && !c.per_vertex)
        return set_error("TC_PER_VERTEX needs per_vertex"), TC_EINVAL;
    if ((c.flags & TC_SORTED) && !(c.flags & TC_CLEAN))
        return set_error("TC_SORTED is only meaningful with TC_CLEAN"), TC_EINVAL;
    if (!c.opt.alloc != !c.opt.free)
        return set_error("tc_options.alloc and .free must be given together"), TC_EINVAL;
    if (c.opt.force_variant < -1 || c.opt.force_variant > 3)
        return set_error("force_variant out of range"), TC_EINVAL;
    for (uint32_t r : c.opt.reserved)
        if (r) return set_error("tc_options.reserved must be zero"), TC_EINVAL;
    return TC_OK;
}

// Device pointers must live on the current device (include/tc.h DEVICE).
static void check_device_ptr(const void *p, int dev, const char *what) {
    if (!p) return;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        throw Error{TC_EINVAL, std::string(what) + " is not a CUDA pointer"};
    }
    if (a.type == cudaMemoryTypeDevice && a.device != dev)
        throw Error{TC_EINVAL, std::string(what) + " lives on device " + std::to_string(a.device) +
                                   ", the current device is " + std::to_string(dev)};
    if (a.type == cudaMemoryTypeUnregistered)
        throw Error{TC_EINVAL, std::string(what) + " is a host pointer without TC_HOST_PTRS"};
}

// ------------------------------------------------------------------ CUDA graph replay
// tc_options.graph_cache (round 2): a launch-bound call (small and mid-size graphs: ~36 kernels,
// ~60 stream-ordered allocations, ~300 us of host work at R-MAT s10-s14) is captured once into
// a CUDA graph -- kernels, memsets, graph-owned workspace (memory nodes), the side-stream fork /
// join, the 8-byte read-back -- and replayed by later calls with the same arguments (device,
// sizes, pointers, flags, options): one graph launch.  Count mode on device pointers, without
// stats, TC_PRUNE, TC_VALIDATE or an allocator hook; a capture that fails runs the call the
// normal way.  Per thread: the read-back lands in this thread's pinned scratch.
struct GraphKey {
    int device;
    uint64_t n, M;
    const void *rowptr, *col, *pv;
    uint32_t flags;
    tc_options opt;
    bool operator==(const GraphKey &o) const {
        return device == o.device && n == o.n && M == o.M && rowptr == o.rowptr && col == o.col &&
               pv == o.pv && flags == o.flags && memcmp(&opt, &o.opt, sizeof(opt)) == 0;
    }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    uint64_t launches = 0;
};
static std::vector<GraphEntry> &graph_cache() {
    static thread_local std::vector<GraphEntry> c;
    return c;
}
static cudaStream_t graph_stream(int dev) {   // capture needs a non-legacy stream
    static thread_local cudaStream_t s[64] = {};
    if (!s[dev]) TC_CUDA(cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking));
    return s[dev];
}
static bool graph_eligible(const Call &c) {
    return c.opt.graph_cache && c.mode == kCount && !(c.flags & (TC_HOST_PTRS | TC_PRUNE | TC_VALIDATE)) &&
           !c.stats && !c.opt.alloc;
}
static GraphKey graph_key(const Call &c, int dev) {
    GraphKey k;
    memset(&k, 0, sizeof(k));
    k.device = dev;
    k.n = c.n;
    k.M = c.M;
    k.rowptr = c.rowptr;
    k.col = c.col;
    k.pv = c.per_vertex;
    k.flags = c.flags;
    k.opt = c.opt;
    return k;
}

static void run_impl(Call &c, bool capture);
struct LowDegRetry {};   // thrown by run_impl when the bounded-degree path was not eligible

static void run(Call &c) {
    if (!graph_eligible(c)) {
        try {
            return run_impl(c, false);
        } catch (const LowDegRetry &) {   // more than lowdeg_max incidences somewhere
            Call c2 = c;
            c2.opt.lowdeg_max = 0;
            return run_impl(c2, false);
        }
    }
    int dev = 0;
    TC_CUDA(cudaGetDevice(&dev));
    const GraphKey key = graph_key(c, dev);
    for (GraphEntry &e : graph_cache())
        if (e.key == key) {   // replay: after the caller's earlier work on its stream
            Ctx ctx;
            ctx.device = dev;
            ctx.stream = graph_stream(dev);
            cudaStream_t caller = (cudaStream_t)c.opt.stream;
            cudaEvent_t ev;
            TC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            cudaEventRecord(ev, caller);
            cudaStreamWaitEvent(ctx.stream, ev, 0);
            cudaEventDestroy(ev);
            uint64_t *pin = pinned_scratch();
            pin[26] = 0;
            TC_CUDA(cudaGraphLaunch(e.exec, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            ctx.launches = e.launches;   // the graph's kernels count as launched (tc_launches_issued)
            if (c.n > 0 && c.M > 0) check_claim(pin);
            *c.total_host = pin[20];
            return;
        }
    try {
        run_impl(c, true);
    } catch (const Error &) {   // not capturable here: run it the normal way
        cudaGetLastError();
        Call plain = c;
        plain.opt.graph_cache = 0;
        run_impl(plain, false);
    }
}

// The bounded-degree path (lowdeg.cu): the eligibility passes and the count, enqueued without
// a synchronisation; their flag (some vertex has more than lowdeg_max incidences: nothing was
// counted) is read with the count, and run() then re-runs the call on the general pipeline
// (LowDegRetry).  Fills pin[] as the general path does for the stats it has.
static bool run_lowdeg(Ctx &ctx, const Call &c, const uint64_t *rowptr, const uint32_t *col, Timer *tm,
                       uint64_t *total_dev, uint64_t *pv_dev, uint64_t *pin) {
    const bool clean = c.flags & TC_CLEAN;
    uint64_t *out = ctx.alloc<uint64_t>(8);     // [0..5] lowdeg_count's sums, [6] the flag
    TC_CUDA(cudaMemsetAsync(out, 0, 8 * sizeof(uint64_t), ctx.stream));
    uint32_t *flag = (uint32_t *)(out + 6);
    LowDeg ld;
    phase_begin(tm, kClean);
    lowdeg_prepare(ctx, ld, c.n, c.M, rowptr, col, clean, c.flags & TC_SORTED, c.opt.lowdeg_max, flag);
    lowdeg_count(ctx, ld, c.M, tm, total_dev, pv_dev, out, c.stats != nullptr);
    // pin[32 + i] = out[i] (one copy): the flag, Sum d+ (a false TC_CLEAN claim has more than
    // m/2 arcs passing the rank filter) and the stats sums; pin[39] = Sum d(v) = 2m
    TC_CUDA(cudaMemcpyAsync(pin + 32, out, 7 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
    if (c.stats) {
        if (ld.m2) TC_CUDA(cudaMemcpyAsync(pin + 39, ld.m2, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
        else pin[39] = ld.m2_host;
    }
    return true;
}
// After the final synchronisation: the claim flag and the stats slots of the general path.
static void finish_lowdeg(const Call &c, uint64_t *pin) {
    const uint64_t *o = pin + 32;
    if ((c.flags & TC_CLEAN) && o[5] > c.M / 2) pin[26] = 1;
    if (c.stats) {
        pin[4] = o[0];                    // W
        pin[5] = o[1];                    // probe work
        pin[7] = o[2];                    // max d+
        pin[12] = o[3];                   // Sum d- d+
        pin[6] = o[4];                    // skipped edges
        pin[16] = pin[39] / 2;            // m
        pin[0] = pin[16] - pin[6];        // SHORT-like: every edge that can close a triangle
    }
}

static void run_impl(Call &c, bool capture) {
    Ctx ctx;
    TC_CUDA(cudaGetDevice(&ctx.device));
    ctx.stream = (cudaStream_t)c.opt.stream;
    DeviceState &ds = device_state(ctx.device);
    ctx.num_sms = ds.sms;
    // capture: on the library's graph stream, ordered after the caller's earlier work; the
    // workspace as graph memory nodes (cudaMallocAsync in capture)
    struct CaptureGuard {   // ends an aborted capture on every error path
        cudaStream_t s = nullptr;
        ~CaptureGuard() {
            if (!s) return;
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
        }
    } guard;
    if (capture) {
        cudaStream_t caller = ctx.stream;
        ctx.stream = graph_stream(ctx.device);
        cudaEvent_t ev;
        TC_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        cudaEventRecord(ev, caller);
        cudaStreamWaitEvent(ctx.stream, ev, 0);
        cudaEventDestroy(ev);
        check_device_ptr(c.rowptr, ctx.device, "row_offsets");
        check_device_ptr(c.col, ctx.device, "col_indices");
        check_device_ptr(c.per_vertex, ctx.device, "per_vertex");
        (void)pinned_scratch();
        (void)ctx.side();   // create the per-thread side stream / events outside the capture
        ctx.graph_alloc = true;
        TC_CUDA(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal));
        guard.s = ctx.stream;
    }
    if (c.opt.alloc) {
        ctx.hook_alloc = c.opt.alloc;
        ctx.hook_free = c.opt.free;
        ctx.hook_ctx = c.opt.alloc_ctx;
    } else if (!capture) {
        ctx.pool = ds.pool;
        set_pool_keep(ds.pool, c.opt.keep_workspace != 0);
    }
    if (c.mode == kCleanShard) {
        check_device_ptr(c.rowptr, ctx.device, "row_offsets");
        check_device_ptr(c.col, ctx.device, "col_indices");
        check_device_ptr(c.edges_out, ctx.device, "edges");
        check_device_ptr(c.deg_out, ctx.device, "degrees");
        if (c.n) TC_CUDA(cudaMemsetAsync(c.deg_out, 0, c.n * sizeof(uint32_t), ctx.stream));
        uint64_t *m_dev = ctx.alloc<uint64_t>(1);
        TC_CUDA(cudaMemsetAsync(m_dev, 0, sizeof(uint64_t), ctx.stream));
        if (c.n && c.M) clean_shard(ctx, c.n, c.M, c.rowptr, c.col, c.rank, c.world, c.edges_out,
                                    c.deg_out, m_dev, c.opt.clean_method);
        uint64_t *pin = pinned_scratch();
        TC_CUDA(cudaMemcpyAsync(pin + 27, m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
        ctx.release();
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
        *c.m_edges_out = pin[27];
        return;
    }
    const bool host = c.flags & TC_HOST_PTRS;
    if (!host && !capture) {   // (a capture checked them before it began)
        if (!c.edges_in) {
            check_device_ptr(c.rowptr, ctx.device, "row_offsets");
            check_device_ptr(c.col, ctx.device, "col_indices");
        }
        check_device_ptr(c.edges_in, ctx.device, "edges");
        check_device_ptr(c.deg_in, ctx.device, "degrees");
        check_device_ptr(c.per_vertex, ctx.device, "per_vertex");
        check_device_ptr(c.partial_dev, ctx.device, "partial_dev");
        check_device_ptr(c.off_plus, ctx.device, "off_plus");
        check_device_ptr(c.col_plus, ctx.device, "col_plus");
        check_device_ptr(c.support, ctx.device, "support / c_values");
        check_device_ptr(c.cc, ctx.device, "local_cc");
        check_device_ptr(c.triangles, ctx.device, "triangles");
    }
    const bool pv = ((c.flags & TC_PER_VERTEX) && c.mode != kOrientOnly) || c.mode == kClustering;
    const bool pv_out = pv && c.per_vertex;   // t(v) wanted by the caller
    tc_stats st;
    memset(&st, 0, sizeof(st));
    Timer *tm = nullptr;
    cudaEvent_t t_begin = nullptr, t_end = nullptr;
    if (c.stats) {
        tm = new Timer(ctx.stream);
        cudaEventCreate(&t_begin);
        cudaEventCreate(&t_end);
        cudaEventRecord(t_begin, ctx.stream);
    }
    struct Cleanup {
        Timer *&tm;
        cudaEvent_t &a, &b;
        ~Cleanup() {
            delete tm;
            if (a) cudaEventDestroy(a);
            if (b) cudaEventDestroy(b);
        }
    } cleanup{tm, t_begin, t_end};

    // ---- inputs on the device
    const uint64_t *rowptr = c.rowptr;
    const uint32_t *col = c.col;
    if (host) {
        uint64_t *d_row = ctx.alloc<uint64_t>(c.n + 1);
        TC_CUDA(cudaMemcpyAsync(d_row, c.rowptr, (c.n + 1) * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, ctx.stream));
        st.h2d_bytes += (c.n + 1) * sizeof(uint64_t);
        rowptr = d_row;
        if (c.M) {
            uint32_t *d_col = ctx.alloc<uint32_t>(c.M);
            TC_CUDA(cudaMemcpyAsync(d_col, c.col, c.M * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                    ctx.stream));
            st.h2d_bytes += c.M * sizeof(uint32_t);
            col = d_col;
        }
    }
    if (c.flags & TC_VALIDATE) {
        std::string msg = validate_graph(ctx, c.n, c.M, rowptr, col, c.flags & TC_CLEAN,
                                         c.flags & TC_SORTED);
        if (!msg.empty()) throw Error{TC_EGRAPH, msg};
    }

    uint64_t *pv_dev = nullptr, *pv_new = nullptr;  // output side / rank-id side
    if (pv) {
        pv_new = ctx.alloc<uint64_t>(c.n);
        if (c.n) TC_CUDA(cudaMemsetAsync(pv_new, 0, c.n * sizeof(uint64_t), ctx.stream));
    }
    if (pv_out) {
        pv_dev = host ? ctx.alloc<uint64_t>(c.n) : c.per_vertex;
        if (c.n) TC_CUDA(cudaMemsetAsync(pv_dev, 0, c.n * sizeof(uint64_t), ctx.stream));
    }
    double *cc_dev = nullptr;                       // kClustering: local coefficients
    uint64_t *cc_out = nullptr;                     // {wedges, bits of sum c}
    if (c.mode == kClustering) {
        if (c.cc) {
            cc_dev = host ? ctx.alloc<double>(c.n) : c.cc;
            if (c.n) TC_CUDA(cudaMemsetAsync(cc_dev, 0, c.n * sizeof(double), ctx.stream));
        }
        cc_out = ctx.alloc<uint64_t>(2);
        TC_CUDA(cudaMemsetAsync(cc_out, 0, 2 * sizeof(uint64_t), ctx.stream));
    }
    uint64_t *total_dev = c.mode == kShard ? c.partial_dev : ctx.alloc<uint64_t>(1);
    TC_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(uint64_t), ctx.stream));
    uint64_t *pin = pinned_scratch();
    if (c.stats) memset(pin, 0, 32 * sizeof(uint64_t));
    pin[26] = 0;   // the false-TC_CLEAN flag of THIS call (check_claim)

    // Rows of N+ are always put in ascending order (a4): the merge / search variants need
    // it, and the HASH ranges probe only the part of N+(a) after b.

    PruneInfo prune;
    prune.enabled = c.flags & TC_PRUNE;
    prune.rounds_wanted = c.opt.prune_rounds;
    const bool tiny = (c.mode == kCount || c.mode == kShard) && !c.edges_in && c.n > 0 && c.M > 0 &&
                      c.n <= c.opt.tiny_max_n && c.n <= kTinyMaxN && c.opt.force_variant < 0 &&
                      !(c.flags & (TC_PRUNE | TC_ID_ORDER));
    // the bounded-degree path: few incidences per vertex (m <= 8n arcs as a host-side gate,
    // then a device test); never under capture (its decision is a host read of the data)
    const bool lowdeg = c.mode == kCount && !tiny && !capture && !c.edges_in && c.n > 0 && c.M > 0 &&
                        c.opt.lowdeg_max > 0 && c.M <= 8 * c.n && c.opt.force_variant < 0 &&
                        !(c.flags & (TC_PRUNE | TC_ID_ORDER));
    bool ld_ran = false;
    if (tiny) {   // one kernel (tiny.cu); a shard other than rank 0 contributes nothing
        pin[16] = 0;
        uint64_t *m_dev = ctx.alloc<uint64_t>(1);
        TC_CUDA(cudaMemsetAsync(m_dev, 0, sizeof(uint64_t), ctx.stream));
        phase_begin(tm, kIntersect);
        if (c.mode != kShard || c.rank == 0)
            tiny_count(ctx, c.n, rowptr, col, total_dev, pv_out ? pv_dev : nullptr, m_dev);
        phase_end(tm, kIntersect);
        if (c.stats)
            TC_CUDA(cudaMemcpyAsync(pin + 16, m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
    } else if (lowdeg && (ld_ran = run_lowdeg(ctx, c, rowptr, col, tm, total_dev, pv_out ? pv_dev : nullptr,
                                              pin))) {
        // counted by the bounded-degree path (lowdeg.cu); stats are in pin[]
    } else if (c.n > 0 && c.M > 0) {
        Oriented g;
        if (c.edges_in) {   // after a sharded a1: the unique edges of every rank, all degrees
            uint64_t *m_dev = ctx.alloc<uint64_t>(1);
            TC_CUDA(cudaMemcpyAsync(m_dev, &c.M, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx.stream));
            orient_edges(ctx, c.n, c.M, const_cast<uint64_t *>(c.edges_in), m_dev,
                         const_cast<uint32_t *>(c.deg_in), g, tm, prune, c.flags & TC_ID_ORDER);
        } else if (c.flags & TC_CLEAN)
            orient_clean(ctx, c.n, c.M, rowptr, col, g, tm,
                         prune, c.flags & TC_ID_ORDER);
        else
            orient_dirty(ctx, c.n, c.M, rowptr, col, g, tm,
                         prune, c.flags & TC_ID_ORDER, c.opt.clean_method);
        if (g.claim_err && (c.mode != kShard || c.stats))   // read at the final synchronisation
            TC_CUDA(cudaMemcpyAsync(pin + 26, g.claim_err, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
        if (c.stats && prune.m_before)
            TC_CUDA(cudaMemcpyAsync(pin + 24, prune.m_before, sizeof(uint64_t),
                                    cudaMemcpyDeviceToHost, ctx.stream));
        if (c.stats && prune.enabled)
            TC_CUDA(cudaMemcpyAsync(pin + 25, g.m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));

        if (c.mode == kOrientOnly) {  // N+ in the caller's ids, rows ascending (tc_orient)
            uint64_t *off_o = ctx.alloc<uint64_t>(c.n + 1);
            uint32_t *col_o = ctx.alloc<uint32_t>(g.m_cap);
            to_original(ctx, g, off_o, col_o);
            cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
            uint64_t m = 0;
            TC_CUDA(cudaMemcpyAsync(&m, g.m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            check_claim(pin);
            TC_CUDA(cudaMemcpyAsync(c.off_plus, off_o, (c.n + 1) * sizeof(uint64_t), kind, ctx.stream));
            if (m) TC_CUDA(cudaMemcpyAsync(c.col_plus, col_o, m * sizeof(uint32_t), kind, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            *c.m_plus = m;
            return;
        }

        phase_begin(tm, kBin);
        BinParams bp;
        bp.edge_ids = c.mode == kSupport;
        bp.short_max = c.opt.short_max;
        bp.skew_ratio = c.opt.skew_ratio;
        bp.hub_min = c.opt.hub_min_dplus;
        bp.force = c.opt.force_variant;
        bp.rank = c.rank;
        bp.world = c.world;
        bp.core = (c.mode == kCount || c.mode == kShard) && !pv;   // plain count only
        Bins bins;
        bin_edges(ctx, g, bp, bins);
        phase_end(tm, kBin);

        Credit cr;
        uint32_t *sup = nullptr;
        if (pv) {
            cr.mode = kCmVertex;
            cr.pv = pv_new;
        } else if (c.mode == kSupport || c.mode == kMasked) {
            sup = ctx.alloc<uint32_t>(g.m_cap);
            TC_CUDA(cudaMemsetAsync(sup, 0, g.m_cap * sizeof(uint32_t), ctx.stream));
            cr.mode = c.mode == kSupport ? kCmEdge : kCmTop;
            cr.sup = sup;
        } else if (c.mode == kEnumerate) {
            cr.mode = kCmList;
            cr.cap = c.capacity;
            cr.tri = (host && c.capacity) ? ctx.alloc<uint32_t>(3 * c.capacity) : c.triangles;
            cr.cursor = ctx.alloc<uint64_t>(1);
            cr.order = g.order;
            TC_CUDA(cudaMemsetAsync(cr.cursor, 0, sizeof(uint64_t), ctx.stream));
        }
        phase_begin(tm, kIntersect);
        intersect_all(ctx, g, bins, total_dev, cr);
        phase_end(tm, kIntersect);
        if (c.mode == kSupport || c.mode == kMasked) {   // N+ in the caller's ids + values
            uint64_t *off_o = ctx.alloc<uint64_t>(c.n + 1);
            uint32_t *col_o = ctx.alloc<uint32_t>(g.m_cap), *sup_o = ctx.alloc<uint32_t>(g.m_cap);
            to_original(ctx, g, off_o, col_o, sup, sup_o);
            cudaMemcpyKind kind = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
            uint64_t m = 0;
            TC_CUDA(cudaMemcpyAsync(&m, g.m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            TC_CUDA(cudaMemcpyAsync(c.off_plus, off_o, (c.n + 1) * sizeof(uint64_t), kind, ctx.stream));
            if (m) {
                TC_CUDA(cudaMemcpyAsync(c.col_plus, col_o, m * sizeof(uint32_t), kind, ctx.stream));
                TC_CUDA(cudaMemcpyAsync(c.support, sup_o, m * sizeof(uint32_t), kind, ctx.stream));
            }
            if (host) st.d2h_bytes += (c.n + 1) * sizeof(uint64_t) + 2 * m * sizeof(uint32_t);
            *c.m_plus = m;
        }
        if (c.mode == kEnumerate && host && c.capacity) {  // min(T, capacity) triples back
            uint64_t T = 0;
            TC_CUDA(cudaMemcpyAsync(&T, total_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
            TC_CUDA(cudaStreamSynchronize(ctx.stream));
            uint64_t k = T < c.capacity ? T : c.capacity;
            if (k)
                TC_CUDA(cudaMemcpyAsync(c.triangles, cr.tri, 3 * k * sizeof(uint32_t),
                                        cudaMemcpyDeviceToHost, ctx.stream));
            st.d2h_bytes += 3 * k * sizeof(uint32_t);
        }
        if (pv_out) per_vertex_to_original(ctx, g, pv_new, pv_dev);
        if (c.mode == kClustering) clustering(ctx, g, pv_new, cc_dev, cc_out);
        if (c.stats) {  // async into pinned memory; read after the final sync
            TC_CUDA(cudaMemcpyAsync(pin, bins.count, 16 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
            TC_CUDA(cudaMemcpyAsync(pin + 16, g.m_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
            TC_CUDA(cudaMemcpyAsync(pin + 12, g.stage_work, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
        }
    } else if (c.mode == kOrientOnly || c.mode == kSupport || c.mode == kMasked) {
        cudaMemcpyKind kind = host ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice;
        std::vector<uint64_t> zeros(c.n + 1, 0);
        TC_CUDA(cudaMemcpyAsync(c.off_plus, zeros.data(), (c.n + 1) * sizeof(uint64_t), kind,
                                ctx.stream));
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
        *c.m_plus = 0;
        if (c.mode == kMasked) *c.total_host = 0;
        return;
    }

    if (c.mode == kCount || c.mode == kClustering || c.mode == kEnumerate || c.mode == kSupport ||
        c.mode == kMasked) {
        TC_CUDA(cudaMemcpyAsync(pin + 20, total_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                ctx.stream));
        st.d2h_bytes += sizeof(uint64_t);
        if (cc_out) {
            TC_CUDA(cudaMemcpyAsync(pin + 21, cc_out, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                    ctx.stream));
            st.d2h_bytes += 2 * sizeof(uint64_t);
        }
        if (cc_dev && host && c.n) {
            TC_CUDA(cudaMemcpyAsync(c.cc, cc_dev, c.n * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx.stream));
            st.d2h_bytes += c.n * sizeof(double);
        }
        if (pv_out && host && c.n) {
            TC_CUDA(cudaMemcpyAsync(c.per_vertex, pv_dev, c.n * sizeof(uint64_t),
                                    cudaMemcpyDeviceToHost, ctx.stream));
            st.d2h_bytes += c.n * sizeof(uint64_t);
        }
    }
    if (c.stats) cudaEventRecord(t_end, ctx.stream);
    ctx.release();
    if (capture) {   // the graph of this call: cache it, then run it
        guard.s = nullptr;
        cudaGraph_t graph = nullptr;
        TC_CUDA(cudaStreamEndCapture(ctx.stream, &graph));
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        TC_CUDA(ie);
        auto &cache = graph_cache();
        if (cache.size() >= 4) {   // small per-thread cache: drop the oldest
            cudaGraphExecDestroy(cache.front().exec);
            cache.erase(cache.begin());
        }
        cache.push_back(GraphEntry{graph_key(c, ctx.device), exec, ctx.launches});
        TC_CUDA(cudaGraphLaunch(exec, ctx.stream));
    }
    const bool synced = c.mode != kShard || c.stats;
    if (synced) TC_CUDA(cudaStreamSynchronize(ctx.stream));
    TC_CUDA(cudaGetLastError());
    if (ld_ran && pin[38]) throw LowDegRetry{};   // not eligible: run() re-runs on the pipeline
    if (ld_ran) finish_lowdeg(c, pin);
    if (synced && c.n > 0 && c.M > 0) check_claim(pin);
    if (c.mode == kCount || c.mode == kEnumerate || c.mode == kMasked) *c.total_host = pin[20];
    if (c.mode == kClustering && c.csum) {
        tc_clustering_summary &r = *c.csum;
        r.triangles = pin[20];
        r.wedges = pin[21];
        double sum;
        memcpy(&sum, &pin[22], sizeof(sum));
        // 3T and the wedge count are exact integers below 2^53: one rounded division
        r.transitivity = r.wedges ? (3.0 * (double)r.triangles) / (double)r.wedges : 0.0;
        r.avg_clustering = c.n ? sum / (double)c.n : 0.0;
    }

    if (c.stats) {
        st.ms_clean = tm->ms(kClean);
        st.ms_orient = tm->ms(kOrient);
        st.ms_sort = tm->ms(kSort);
        st.ms_bin = tm->ms(kBin);
        st.ms_intersect = tm->ms(kIntersect);
        float t = 0.f;
        cudaEventElapsedTime(&t, t_begin, t_end);
        st.ms_total = t;
        st.m_undirected = pin[16];
        st.work_W = pin[4];
        st.work_probe = pin[5];
        st.bytes_alg = 4 * st.work_W + 16 * st.m_undirected;
        st.bin_edges[0] = pin[0];
        st.bin_edges[1] = pin[1];
        st.bin_edges[2] = pin[2];
        st.bin_edges[3] = pin[3];
        st.skipped_edges = pin[6];
        st.hub_sources = pin[9] + pin[10];
        st.max_dplus = pin[7];
        st.table_loads = pin[11];
        st.work_stage = pin[12];
        st.core_edges = pin[13];
        st.core_words = pin[14];
        // bytes the HASH method reads in a6: probed elements + one 8-byte range per probe
        // entry (<= 2 per edge, 1 for ~96%) + the owners' lists for the table builds
        // (core edges are binned before HASH; their probes pin[15] are not HASH bytes)
        st.bytes_hash = 4 * (st.work_probe - pin[15]) + 8 * st.bin_edges[3] + 4 * st.table_loads;
        st.bytes_core = 8 * st.core_words;
        st.kernel_launches = ctx.launches;
        if (prune.enabled && c.n > 0 && c.M > 0) {
            st.ms_prune = tm->ms(kPrune);
            uint64_t before = prune.m_before ? pin[24] : prune.m_before_host;
            st.pruned_edges = before - pin[25];
            st.prune_rounds = prune.rounds;
        }
        *c.stats = st;
    }
}

static tc_status guarded(Call &c) {
    tc_status s = check_args(c);
    if (s != TC_OK) return s;
    try {
        run(c);
    } catch (const Error &e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return TC_ENOMEM;
    }
    set_error("");
    return TC_OK;
}

static tc_options resolve(const tc_options *opt) {
    tc_options o;
    tc_default_options(&o);
    if (opt) o = *opt;  // taken as given: 0 disables the SHORT / SEARCH bins
    return o;
}

// The phase entry points of shard.cu: options resolved and checked, workspace (hook or the
// library pool) and stream set up, fn run, every exception mapped to a tc_status.  fn ends
// with whatever synchronisation its outputs need.
tc_status run_phase(const tc_options *opt_in, const std::function<void(Ctx &, const tc_options &)> &fn) {
    const tc_options opt = resolve(opt_in);
    for (uint32_t r : opt.reserved)
        if (r) return set_error("tc_options.reserved must be zero"), TC_EINVAL;
    if (!opt.alloc != !opt.free)
        return set_error("tc_options.alloc and .free must be given together"), TC_EINVAL;
    try {
        Ctx ctx;
        TC_CUDA(cudaGetDevice(&ctx.device));
        ctx.stream = (cudaStream_t)opt.stream;
        DeviceState &ds = device_state(ctx.device);
        ctx.num_sms = ds.sms;
        if (opt.alloc) {
            ctx.hook_alloc = opt.alloc;
            ctx.hook_free = opt.free;
            ctx.hook_ctx = opt.alloc_ctx;
        } else {
            ctx.pool = ds.pool;
            set_pool_keep(ds.pool, opt.keep_workspace != 0);
        }
        fn(ctx, opt);
        ctx.release();
        TC_CUDA(cudaStreamSynchronize(ctx.stream));
    } catch (const Error &e) {
        set_error(e.msg);
        return e.status;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return TC_ENOMEM;
    }
    set_error("");
    return TC_OK;
}

void check_device(const void *p, int dev, const char *what) { check_device_ptr(p, dev, what); }

}  // namespace tc

using namespace tc;

extern "C" {

void tc_default_options(tc_options *opt) {
    if (!opt) return;
    memset(opt, 0, sizeof(*opt));
    // AUTO defaults, measured on R-MAT s21: the HASH
    // variant (cost min(d+u, d+v) per edge) beats SHORT / SEARCH / MERGE on every
    // bin, so those bins are off unless enabled here or forced.
    opt->short_max = 20;
    opt->skew_ratio = 0;
    opt->hub_min_dplus = 80;
    opt->force_variant = TC_VARIANT_AUTO;
    opt->stream = nullptr;
    opt->keep_workspace = 1;
    opt->tiny_max_n = (uint32_t)kTinyMaxN;
    opt->lowdeg_max = kLowDegMax;
}

tc_status tc_trim_workspace(int device) {
    try {
        if (device < 0) TC_CUDA(cudaGetDevice(&device));
        DeviceState &d = device_state(device);
        TC_CUDA(cudaMemPoolTrimTo(d.pool, 0));
        // this thread's replay graphs (graph_cache) of the device, and the graph memory they held
        auto &cache = graph_cache();
        for (size_t i = 0; i < cache.size();)
            if (cache[i].key.device == device) {
                cudaGraphExecDestroy(cache[i].exec);
                cache.erase(cache.begin() + i);
            } else {
                i++;
            }
        TC_CUDA(cudaDeviceSynchronize());
        TC_CUDA(cudaDeviceGraphMemTrim(device));
    } catch (const Error &e) {
        set_error(e.msg);
        return e.status;
    }
    set_error("");
    return TC_OK;
}

tc_status tc_count_ex(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                      const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                      uint64_t *total, uint64_t *per_vertex, tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kCount;
    c.total_host = total;
    c.per_vertex = per_vertex;
    c.stats = stats;
    return guarded(c);
}

uint64_t tc_count(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                  const uint32_t *col_indices, uint32_t flags) {
    uint64_t total = 0;
    if (flags & TC_PER_VERTEX) {
        set_error("tc_count has no per-vertex output; use tc_count_ex");
        return TC_ERROR;
    }
    tc_status s = tc_count_ex(n, m, row_offsets, col_indices, flags, nullptr, &total, nullptr, nullptr);
    return s == TC_OK ? total : TC_ERROR;
}

tc_status tc_count_shard(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                         const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                         int rank, int world, uint64_t *partial_dev,
                         uint64_t *per_vertex_partial, tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kShard;
    c.rank = rank;
    c.world = world;
    c.partial_dev = partial_dev;
    c.per_vertex = per_vertex_partial;
    c.stats = stats;
    return guarded(c);
}

tc_status tc_clean_shard(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                         const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                         int rank, int world, uint64_t *edges, uint32_t *degrees, uint64_t *m_edges) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kCleanShard;
    c.rank = rank;
    c.world = world;
    c.edges_out = edges;
    c.deg_out = degrees;
    c.m_edges_out = m_edges;
    return guarded(c);
}

tc_status tc_count_edges_shard(uint64_t n, uint64_t m_edges, const uint64_t *edges,
                               const uint32_t *degrees, uint32_t flags, const tc_options *opt,
                               int rank, int world, uint64_t *partial_dev,
                               uint64_t *per_vertex_partial, tc_stats *stats) {
    static const uint64_t kNoRows = 0;   // the CSR is not read on this path
    Call c{n, m_edges, &kNoRows, nullptr, flags, resolve(opt)};
    c.mode = kShard;
    c.rank = rank;
    c.world = world;
    c.edges_in = edges;
    c.deg_in = degrees;
    c.partial_dev = partial_dev;
    c.per_vertex = per_vertex_partial;
    c.stats = stats;
    return guarded(c);
}

tc_status tc_orient(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                    const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                    uint64_t *off_plus, uint32_t *col_plus, uint64_t *m_plus) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kOrientOnly;
    c.off_plus = off_plus;
    c.col_plus = col_plus;
    c.m_plus = m_plus;
    return guarded(c);
}

tc_status tc_clustering(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                        const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                        double *local_cc, uint64_t *per_vertex, tc_clustering_summary *summary,
                        tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kClustering;
    c.cc = local_cc;
    c.per_vertex = per_vertex;
    c.csum = summary;
    c.stats = stats;
    return guarded(c);
}

tc_status tc_edge_support(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                          const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                          uint64_t *off_plus, uint32_t *col_plus, uint32_t *support,
                          uint64_t *m_plus, tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kSupport;
    c.off_plus = off_plus;
    c.col_plus = col_plus;
    c.support = support;
    c.m_plus = m_plus;
    c.stats = stats;
    return guarded(c);
}

tc_status tc_enumerate(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                       const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                       uint32_t *triangles, uint64_t capacity, uint64_t *total, tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kEnumerate;
    c.triangles = triangles;
    c.capacity = capacity;
    c.total_host = total;
    c.stats = stats;
    return guarded(c);
}

tc_status tc_masked_spgemm(uint64_t n, uint64_t m, const uint64_t *row_offsets,
                           const uint32_t *col_indices, uint32_t flags, const tc_options *opt,
                           uint64_t *off_plus, uint32_t *col_plus, uint32_t *c_values,
                           uint64_t *nnz_u, uint64_t *total, tc_stats *stats) {
    Call c{n, m, row_offsets, col_indices, flags, resolve(opt)};
    c.mode = kMasked;
    c.off_plus = off_plus;
    c.col_plus = col_plus;
    c.support = c_values;
    c.m_plus = nnz_u;
    c.total_host = total;
    c.stats = stats;
    return guarded(c);
}

const char *tc_last_error(void) { return g_last_error.c_str(); }

uint64_t tc_launches_issued(void) { return thread_launches(); }

const char *tc_version(void) { return "tc_b200 0.1 (sm_100a)"; }

}  // extern "C"
