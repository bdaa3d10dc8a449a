// lcsg_api.cu -- C-ABI (include/lcsgrid_b200.h) and the device-resident level
// scheduler of the Lu-Liu recursion.
//
// The reference builds its tree depth-first and sequentially, one combine at
// a time through a CPU thread pool (solver.py:113-119, parallel.py:50-66).
// Here the whole tree is laid out in ONE HBM arena up front and every
// combine of one height is launched as a single batched grid, in height
// order, on one stream: leaf step -> height 1 .. H -> walk -> assemble.
// The node numbering equals the reference's creation order (post-order), so
// per-node fixtures compare node by node.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lcsgrid_b200.h"
#include "lcsg_internal.cuh"

extern char **environ;

using namespace lcsg;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                            \
    do {                                                                                    \
        cudaError_t e__ = (call);                                                           \
        if (e__ != cudaSuccess)                                                             \
            return fail(e__ == cudaErrorMemoryAllocation ? LCSG_ENOMEM : LCSG_ECUDA,        \
                        std::string(#call) + ": " + cudaGetErrorString(e__));               \
    } while (0)

#define CKL(call)                                                                           \
    do {                                                                                    \
        int e__ = (call);                                                                   \
        if (e__ != 0)                                                                       \
            return fail(LCSG_ECUDA, std::string("kernel launch ") + #call + ": " +          \
                                        cudaGetErrorString((cudaError_t)e__));              \
    } while (0)

int bits_for(int64_t x) {
    if (x <= 0) return 1;
    int b = 0;
    while (x > 0) { ++b; x >>= 1; }
    return b;
}

std::mutex g_pool_mu;
cudaMemPool_t g_pool[64] = {};

// Saves the caller's current device and restores it on scope exit: no entry
// point leaves the calling thread on another device (torch allocations and
// kernels of the caller keep going to the device it had selected).
struct SaveDevice {
    int prev = -1;
    SaveDevice() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~SaveDevice() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// Selects `device` (callers hold a SaveDevice) and makes sure the library's
// own memory pool exists there.  The pool is private to the library (not the
// device's default pool, which PyTorch's cudaMallocAsync backend and other
// libraries share): it keeps freed blocks so repeated solves reuse the same
// HBM without cudaMalloc/cudaFree round trips, and lcsg_trim() returns them.
int prepare_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(LCSG_ENODEV, "no CUDA device visible");
    }
    if (device < 0 || device >= count || device >= 64)
        return fail(LCSG_EINVAL, "device index out of range");
    CK(cudaSetDevice(device));
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (!g_pool[device]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaMemPool_t pool;
        CK(cudaMemPoolCreate(&pool, &props));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        g_pool[device] = pool;
    }
    return LCSG_OK;
}

// stream-ordered allocation from the library pool of `device`
cudaError_t pool_alloc(void **p, size_t bytes, int device, cudaStream_t s) {
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        pool = (device >= 0 && device < 64) ? g_pool[device] : nullptr;
    }
    if (!pool) return cudaMallocAsync(p, bytes, s);
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

int current_device_prepared(int *dev) {
    CK(cudaGetDevice(dev));
    return prepare_device(*dev);
}

// Kernel choice per combine:
//   kind 0: narrow tables (w1 <= LCSG_THREAD_MAX_W1, default 65): staged
//           brute-force first-wins min (lcsg_narrow.cu; LCSG_NARROW=0 selects
//           the thread-per-row exact bisection instead)
//   kind 2: skeleton rows (exact bisection: thread / warp / CTA per row by
//           width) + refinement passes             (wider)
//   kind 1: warp-per-row exact bisection          (fallback: U rows too big for smem)

int env_int(const char *name, int def) {
    const char *v = getenv(name);
    return v && *v ? atoi(v) : def;
}

// 64-bit packed (value, k) keys when the value and split bits do not fit in
// 32; LCSG_FORCE_KEY64=1 selects them everywhere, so the 64-bit
// instantiation of every kernel is parity-tested at small sizes too.
bool need_key64(int value_bits, int shift) {
    return value_bits + shift > 32 || env_int("LCSG_FORCE_KEY64", 0) != 0;
}

// Skeleton stride (rows computed by the exact bisection) and column-refinement
// block size by column count: short strings have few CTAs per level, so a
// denser skeleton and shallower refinement stages (fewer dependent passes)
// win; long strings amortise the refinement (measured with tools/sweep.py on
// cfg1 256^2: 8/4 0.24 ms vs 32/8 0.32; cfg2 2048^2: 8/4 0.96 vs 1.25; cfg3
// 4096^2: 16/4 2.20 vs 2.30; cfg4/cfg5 keep 64/8).
int default_skeleton_stride(int64_t n1) {
    return n1 <= 2049 ? 8 : n1 <= 4097 ? 16 : n1 <= 8193 ? 32 : 64;
}
int default_col_block(int64_t n1) { return n1 <= 4097 ? 4 : 8; }
// Rows per block of the row sweep (= its skeleton stride): a block is a
// sequential chain of row steps, so short strings (few blocks per level)
// need short chains (measured: cfg1 256^2 stride 4 0.20 ms vs 64 0.44; cfg2
// 2048^2 8 0.81 vs 1.89; cfg3 4096^2 16 1.51 vs 2.14; cfg4/cfg5 32..64 equal)
int default_sweep_stride(int64_t n1) {
    return n1 <= 513 ? 4 : n1 <= 2049 ? 8 : n1 <= 4097 ? 16 : n1 <= 8193 ? 32 : 64;
}

struct NodeH {
    int32_t top_row, bottom_row, w1, upper, lower, height, depth, leaf_row;
    int32_t pair = 0;  // batched solves: the pair this node belongs to
    int64_t reach_off = -1, trace_off = -1, kmax_off = -1, ev_off = -1;  // int32 element offsets
    int64_t flag_off = -1;  // kind 2: block flags of the row sweep (index into d_flags)
    int kind = 0;
    bool virt = false;  // virtual height-1 node: no table (TabDev closed form of its leaves)
};

struct LaunchH {
    // 0 thread, 1 warp, 3 skeleton CTA, 4 refine pass, 5/6 skeleton thread/warp,
    // 7 column-refinement stage, 8 finalize, 9 staged thread, 10 narrow
    int kind;
    int32_t desc_off, count;
    int shift;
    bool key64;
    int32_t stride_or_delta = 0;
    int wpr_log2 = 0;
    int32_t ustride = 0;
};

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

struct SolveEntry;  // per-shape graph cache entry (below)

}  // namespace

struct lcsg_tree_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t m_grid = 0, m_slab = 0, n = 0;
    int32_t inf = 0, top_row = 1, bottom_row = 2;
    // batched solves (lcsg_lcs_batch): npairs independent trees of the same
    // shape side by side -- pair p's nodes are ids [p*pair_nodes, (p+1)*pair_nodes),
    // its tables pair_tab ints after pair p-1's; every level is one launch
    int32_t npairs = 1, pair_nodes = 0;
    int64_t pair_tab = 0;
    bool with_trace = true, timing = false;
    std::vector<NodeH> nodes;
    int32_t root = -1;
    std::vector<LaunchH> plan;
    std::vector<std::pair<int32_t, int32_t>> depth_ranges;  // (offset, count) into walk ids
    int walk_shift = 1;
    bool walk_key64 = false;
    // device
    char *arena = nullptr;
    size_t arena_bytes = 0;
    uint8_t *d_rows = nullptr, *d_cols = nullptr, *d_subseq = nullptr;
    int32_t *d_nx = nullptr, *d_sym_wstar = nullptr, *d_node_wstar = nullptr, *d_tables = nullptr;
    CombineDesc *d_descs = nullptr;
    WalkNode *d_walk = nullptr;
    int32_t *d_walk_ids = nullptr, *d_leaf_nodes = nullptr, *d_leaf_rows = nullptr;
    int32_t *d_wi = nullptr, *d_wj = nullptr, *d_path = nullptr, *d_out = nullptr;
    int32_t nleaves = 0;
    std::map<int32_t, int32_t *> leaf_cache;  // materialised leaves / virtual nodes (API only)
    int32_t nvirt = 0;
    int32_t *d_vnodes = nullptr;
    int32_t *d_flags = nullptr;  // row-sweep block flags of every kind-2 node (zeroed per solve)
    size_t flags_bytes = 0;
    int64_t launches = 0, h2d_bytes = 0, d2h_bytes = 0;
    cudaEvent_t ev[5] = {};
    bool ev_ok = false;
    bool owns_events = true;
    SolveEntry *entry = nullptr;  // per-shape graph cache entry this handle runs on

    Ctx ctx() const {
        Ctx c;
        c.rows = d_rows;
        c.nx = d_nx;
        c.nx_stride = (int64_t)256 * (n + 1);
        c.n = (int32_t)n;
        c.inf = inf;
        return c;
    }
    RootBatch root_batch() const {
        RootBatch rb;
        rb.npairs = npairs;
        rb.pair_nodes = pair_nodes;
        rb.pair_rows = (int32_t)m_slab;
        rb.tab_stride = pair_tab;
        return rb;
    }
    TabDev tab(int32_t id) const {
        const NodeH &nd = nodes[id];
        TabDev t;
        t.w1 = nd.w1;
        t.wstar = d_node_wstar + id;
        t.leaf2 = 0;
        t.pair = nd.pair;
        if (nd.upper < 0) {
            t.reach = nullptr;
            t.kmax = nullptr;
            t.leaf_row = nd.leaf_row;
        } else if (nd.virt) {
            t.reach = nullptr;
            t.kmax = nullptr;
            t.leaf_row = nodes[nd.upper].leaf_row;
            t.leaf2 = nodes[nd.lower].leaf_row + 1;
        } else {
            t.reach = d_tables + nd.reach_off;
            t.kmax = d_tables + nd.kmax_off;
            t.leaf_row = -1;
        }
        return t;
    }
};

namespace {

// solver.py:113-119 -- same split, same (post-)order of node creation.
int32_t build_tree(lcsg_tree_s *t, int32_t top, int32_t bottom, int32_t depth) {
    NodeH nd;
    nd.top_row = top;
    nd.bottom_row = bottom;
    nd.depth = depth;
    int64_t w = std::min<int64_t>(bottom - top, t->n);
    nd.w1 = (int32_t)(w + 1);
    if (bottom == top + 1) {
        nd.upper = nd.lower = -1;
        nd.height = 0;
        nd.leaf_row = top - t->top_row;
        t->nodes.push_back(nd);
        return (int32_t)t->nodes.size() - 1;
    }
    int32_t mid = (top + bottom) / 2;
    int32_t up = build_tree(t, top, mid, depth + 1);
    int32_t lo = build_tree(t, mid, bottom, depth + 1);
    nd.upper = up;
    nd.lower = lo;
    nd.leaf_row = -1;
    nd.height = 1 + std::max(t->nodes[up].height, t->nodes[lo].height);
    t->nodes.push_back(nd);
    return (int32_t)t->nodes.size() - 1;
}

thread_local std::vector<NodeH> t_spare_nodes;  // node storage reused across solves

// tree + table layout of the last shape solved on this host thread
struct LayoutCache {
    bool valid = false, with_trace = false;
    int32_t top_row = 0, bottom_row = 0, root = -1, nleaves = 0, ncomb = 0, maxh0 = 0;
    int64_t n = -1, tab_elems = 0, scratch_elems = 0;
    int skel_stride = 0, thread_max_w1 = 0, virt_on = -1;
    int32_t nvirt = 0;
    std::vector<NodeH> nodes;
};
thread_local LayoutCache t_layout;

// Side stream of a build: after a row sweep, the finalize kernel only writes the
// INF-suffix traces of the level (kmax is the sweep's, wstar the skeleton
// kernel's: kmax is nonincreasing in the start column, so row 0 holds the
// maximum) -- nothing later in the build reads them, so it runs beside the next
// levels and joins the handle's stream at the end.  Leased per build call from a
// small per-device pool (a re-recorded event does not disturb waits already
// enqueued, so a lease can be reused as soon as the call returns).
struct SideCtx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_side_mu;
std::vector<SideCtx *> g_side_free;

struct SideLease {
    SideCtx *c = nullptr;
    bool dirty = false;
    void acquire(int device) {
        if (env_int("LCSG_FINALIZE_SIDE", 1) == 0) return;
        {
            std::lock_guard<std::mutex> lk(g_side_mu);
            for (size_t i = 0; i < g_side_free.size(); ++i)
                if (g_side_free[i]->device == device) {
                    c = g_side_free[i];
                    g_side_free.erase(g_side_free.begin() + i);
                    return;
                }
        }
        SideCtx *n = new SideCtx();
        n->device = device;
        if (cudaStreamCreateWithFlags(&n->stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&n->fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&n->join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            delete n;  // no side stream: the finalize kernels stay on the handle's stream
            return;
        }
        c = n;
    }
    // enqueue `fn(stream)` beside the work already on s
    template <typename F>
    int fork(cudaStream_t s, F fn) {
        if (cudaEventRecord(c->fork, s) != cudaSuccess ||
            cudaStreamWaitEvent(c->stream, c->fork, 0) != cudaSuccess)
            return (int)cudaGetLastError();
        dirty = true;
        return fn(c->stream);
    }
    int join(cudaStream_t s) {
        if (!c || !dirty) return 0;
        dirty = false;
        if (cudaEventRecord(c->join, c->stream) != cudaSuccess ||
            cudaStreamWaitEvent(s, c->join, 0) != cudaSuccess)
            return (int)cudaGetLastError();
        return 0;
    }
    ~SideLease() {
        if (!c) return;
        std::lock_guard<std::mutex> lk(g_side_mu);
        g_side_free.push_back(c);
    }
};

// One entry of the level plan on stream s (kernel choice: DESIGN.md 4).
int launch_plan_entry(lcsg_tree_s *t, const LaunchH &L, cudaStream_t s) {
    const Ctx c = t->ctx();
    const int64_t n1 = t->n + 1;
    const CombineDesc *dd = t->d_descs + L.desc_off;
    if (L.kind <= 1) return launch_combine(L.kind, dd, L.count, c, L.shift, L.key64, s);
    if (L.kind == 9) return launch_combine_staged(dd, L.count, c, L.shift, L.key64, s);
    if (L.kind == 10)
        return launch_narrow(dd, L.count, c, L.shift, L.key64, L.stride_or_delta, s,
                             L.wpr_log2 != 0);
    if (L.kind == 11) return launch_narrow_leafpair(dd, L.count, c, L.shift, L.key64, s);
    if (L.kind == 3)
        return launch_skeleton(dd, L.count, c, L.shift, L.key64, L.stride_or_delta, s);
    if (L.kind == 6 && L.stride_or_delta > 1 && t->with_trace &&
        env_int("LCSG_SKEL_WARP_BATCHED", 1))
        return launch_skeleton_warp(dd, L.count, c, L.shift, L.key64, L.stride_or_delta, s);
    if (L.kind == 5 || L.kind == 6)
        return launch_combine(L.kind == 5 ? 0 : 1, dd, L.count, c, L.shift, L.key64, s,
                              L.stride_or_delta);
    if (L.kind == 7)
        return launch_block_refine(dd, L.count, c, L.shift, L.key64, L.stride_or_delta,
                                   L.wpr_log2, L.ustride, s);
    if (L.kind == 8)
        return launch_finalize_rows(dd, L.count, c, L.stride_or_delta, s, L.ustride, L.wpr_log2 != 0);
    if (L.kind == 12) return launch_table_events(dd, L.count, c, s);
    if (L.kind == 13)
        return launch_sweep(dd, L.count, c, L.shift, L.key64, L.stride_or_delta, L.ustride, s);
    if (refine_rows(n1, L.stride_or_delta) > 0)
        return launch_refine(dd, L.count, c, L.shift, L.key64, L.stride_or_delta, s);
    return -1;  // no launch
}

// A plan entry, with the finalize kernels that follow a row sweep forked onto the
// side stream (traced builds) or dropped (low-memory builds keep no traces, and
// kmax / wstar do not come from that kernel).  Returns like launch_plan_entry.
int launch_plan_entry_side(lcsg_tree_s *t, const LaunchH &L, cudaStream_t s, SideLease &side) {
    if (L.kind == 8 && L.wpr_log2 != 0 && side.c) {
        if (!t->with_trace) return -1;
        return side.fork(s, [&](cudaStream_t ss) { return launch_plan_entry(t, L, ss); });
    }
    return launch_plan_entry(t, L, s);
}

// Every kernel of a build after the inputs and the plan metadata are in the
// arena (what build_impl enqueues, minus its host-to-device copies): the
// sequence a per-shape CUDA graph captures.  Returns a CUDA error or 0.
int enqueue_build_kernels(lcsg_tree_s *t, cudaStream_t s, int64_t *launches, bool events = true) {
    const Ctx c = t->ctx();
    const int32_t nn = (int32_t)t->nodes.size();
    cudaError_t e = cudaMemsetAsync(t->d_node_wstar, 0, (size_t)nn * 4, s);
    if (e) return (int)e;
    if (t->flags_bytes && (e = cudaMemsetAsync(t->d_flags, 0, t->flags_bytes, s))) return (int)e;
    int r = launch_nx(t->d_cols, (int32_t)t->n, t->npairs, t->d_nx, t->d_sym_wstar, s);
    if (r) return r;
    r = launch_leaf_wstar(t->d_rows, t->d_leaf_nodes, t->d_leaf_rows, t->nleaves,
                          (int32_t)std::max<int64_t>(t->m_slab, 1), t->d_sym_wstar,
                          t->d_node_wstar, s);
    if (r) return r;
    int64_t nl = 2;
    if (t->nvirt > 0) {
        r = launch_virtual_wstar(c, t->d_vnodes, t->nvirt, t->d_node_wstar, s);
        if (r) return r;
        ++nl;
    }
    if (events && t->timing && t->ev_ok && (e = cudaEventRecord(t->ev[1], s))) return (int)e;
    SideLease side;
    side.acquire(t->device);
    for (const LaunchH &L : t->plan) {
        r = launch_plan_entry_side(t, L, s, side);
        if (r > 0) {
            side.join(s);
            return r;
        }
        if (r == 0) nl += L.kind == 13 ? sweep_launch_count(L.shift, L.key64, L.stride_or_delta, L.ustride) : 1;
    }
    if ((r = side.join(s)) != 0) return r;
    if (events && t->timing && t->ev_ok && (e = cudaEventRecord(t->ev[2], s))) return (int)e;
    if (launches) *launches = nl;
    return 0;
}

// ---- per-shape CUDA graphs ---------------------------------------------------
// A repeated solve of the same shape (rows, columns, pairs, flags, LCSG_*
// knobs) replays the first solve's kernels as two CUDA graphs -- the build
// (every level) and the extraction walk -- on the first solve's arena, whose
// plan metadata (level descriptors, walk nodes with absolute arena pointers)
// is already resident: per solve the host copies the strings in and launches
// two graphs instead of planning ~50 launches.  An entry serves
// one handle at a time (a second concurrent solve of the shape takes the
// normal path); the next user waits on the previous user's stream through
// `released`.  Entries are kept only for arenas up to LCSG_GRAPH_MAX_MB
// (default: a quarter of the device's memory) and at most 8 of them, LRU-evicted; lcsg_trim() drops them.
struct SolveEntry {
    std::string key;
    int device = 0;
    bool in_use = false;  // guarded by g_graph_mu
    uint64_t last_use = 0;
    lcsg_tree_s *tmpl = nullptr;  // layout, plan and arena pointers of the first solve
    char *arena = nullptr;
    size_t arena_bytes = 0;
    cudaGraphExec_t build = nullptr, walk = nullptr;
    bool walk_failed = false;
    cudaStream_t cap = nullptr;     // capture stream (nothing executes on it)
    cudaEvent_t released = nullptr;  // recorded on the last user's stream
    bool released_valid = false;
    cudaEvent_t ev[5] = {};
    bool ev_ok = false;
    int64_t build_launches = 0, walk_launches = 0;
};
std::mutex g_graph_mu;
std::vector<SolveEntry *> g_graph_cache;
uint64_t g_graph_tick = 0;
constexpr size_t GRAPH_MAX_ENTRIES = 8;

std::string knob_signature() {
    std::vector<std::string> kv;
    for (char **e = environ; e && *e; ++e)
        if (std::strncmp(*e, "LCSG_", 5) == 0 && std::strncmp(*e, "LCSG_LIB_PATH", 13) != 0 &&
            std::strncmp(*e, "LCSG_HOST_PROFILE", 17) != 0)
            kv.emplace_back(*e);
    std::sort(kv.begin(), kv.end());
    std::string sig;
    for (auto &x : kv) sig += x + ";";
    return sig;
}

void free_entry(SolveEntry *en) {  // caller: entry not in use
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(en->device);
    if (en->released_valid) cudaEventSynchronize(en->released);
    if (en->build) cudaGraphExecDestroy(en->build);
    if (en->walk) cudaGraphExecDestroy(en->walk);
    if (en->arena) cudaFree(en->arena);  // stream-ordered pool block; all users are done
    if (en->ev_ok)
        for (auto &e : en->ev) cudaEventDestroy(e);
    if (en->released) cudaEventDestroy(en->released);
    if (en->cap) cudaStreamDestroy(en->cap);
    delete en->tmpl;
    delete en;
    cudaGetLastError();
    if (prev >= 0) cudaSetDevice(prev);
}

void release_entry(lcsg_tree_s *t) {
    SolveEntry *en = t->entry;
    if (cudaEventRecord(en->released, t->stream) == cudaSuccess) en->released_valid = true;
    else cudaGetLastError();
    if (t != en->tmpl) t->nodes.swap(en->tmpl->nodes);  // hand the node list back
    std::lock_guard<std::mutex> lk(g_graph_mu);
    en->in_use = false;
}

void destroy(lcsg_tree_s *t) {
    if (!t) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(t->device);
    for (auto &kv : t->leaf_cache) cudaFreeAsync(kv.second, t->stream);
    if (t->entry) {
        release_entry(t);  // the arena and the events stay with the cache entry
    } else {
        if (t->nodes.capacity() > t_spare_nodes.capacity()) t->nodes.swap(t_spare_nodes);
        if (t->arena) cudaFreeAsync(t->arena, t->stream);
    }
    if (t->ev_ok && t->owns_events)
        for (auto &e : t->ev) cudaEventDestroy(e);
    if (t->own_stream) {
        cudaStreamSynchronize(t->stream);
        cudaStreamDestroy(t->stream);
    }
    if (prev >= 0) cudaSetDevice(prev);
    delete t;
}

// Host staging of the plan metadata: pinned buffers reused across solves (no
// page faults on a fresh multi-MB vector -- they cost 1-3 ms per cfg5 solve --
// and a truly asynchronous upload).  Stages live in a small per-device free
// list shared by all host threads (bounded by the number of concurrent
// solves, so short-lived worker threads do not leak pinned memory); `done`
// is recorded after a solve's uploads and waited on before the buffer is
// rewritten by the next solve that takes it (normally long completed).
struct MetaStage {
    char *buf = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
    int device = -1;
};

std::mutex g_meta_mu;
std::vector<MetaStage *> g_meta_free[64];

// RAII lease of one stage: returned to the device's free list on scope exit
// (after recording `done` on the solve stream, so a later user waits for
// this solve's uploads even on an error path).
struct MetaLease {
    MetaStage *ms = nullptr;
    cudaStream_t stream = nullptr;
    MetaLease() = default;
    MetaLease(const MetaLease &) = delete;
    MetaLease &operator=(const MetaLease &) = delete;
    ~MetaLease() { finish(); }
    // record `done` after everything enqueued so far and hand the stage back
    // (call while the stream is still alive)
    void finish() {
        if (!ms) return;
        if (ms->done && stream && cudaEventRecord(ms->done, stream) != cudaSuccess) {
            cudaGetLastError();
            cudaStreamSynchronize(stream);
            cudaGetLastError();
        }
        std::lock_guard<std::mutex> lk(g_meta_mu);
        g_meta_free[ms->device].push_back(ms);
        ms = nullptr;
    }
    // buffer of >= bytes on `device` (current device), or nullptr
    char *acquire(int device, size_t bytes, cudaStream_t s) {
        stream = s;
        {
            std::lock_guard<std::mutex> lk(g_meta_mu);
            auto &fl = g_meta_free[device];
            if (!fl.empty()) {
                ms = fl.back();
                fl.pop_back();
            }
        }
        if (!ms) {
            ms = new MetaStage();
            ms->device = device;
        }
        if (ms->done) cudaEventSynchronize(ms->done);  // previous upload finished
        if (ms->cap < bytes) {
            if (ms->buf) cudaFreeHost(ms->buf);
            ms->cap = std::max(bytes, ms->cap * 2);
            if (cudaMallocHost((void **)&ms->buf, ms->cap) != cudaSuccess) {
                cudaGetLastError();
                ms->buf = nullptr;
                ms->cap = 0;
                return nullptr;
            }
        }
        if (!ms->done && cudaEventCreateWithFlags(&ms->done, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            ms->done = nullptr;
        }
        return ms->buf;
    }
};

std::string graph_key(int device, int64_t m, int32_t top, int32_t bottom, int64_t n, int32_t npairs,
                      uint32_t flags) {
    return std::to_string(device) + "|" + std::to_string(m) + "|" + std::to_string(top) + "|" +
           std::to_string(bottom) + "|" + std::to_string(n) + "|" + std::to_string(npairs) + "|" +
           std::to_string(flags & (LCSG_WITH_TRACE | LCSG_TIMING)) + "|" + knob_signature();
}

// A free entry for `key` (marked in use), or nullptr.
SolveEntry *acquire_entry(const std::string &key) {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (SolveEntry *en : g_graph_cache)
        if (en->key == key && !en->in_use && en->build) {
            en->in_use = true;
            en->last_use = ++g_graph_tick;
            return en;
        }
    return nullptr;
}

// Build through the shape's graph: the template's layout / plan / pointers,
// fresh strings, one graph launch.
int graph_build(lcsg_tree_s *t, SolveEntry *en, const uint8_t *rows, bool rows_dev,
                const uint8_t *cols, bool cols_dev) {
    lcsg_tree_s *tp = en->tmpl;
    std::vector<NodeH> nodes;
    nodes.swap(tp->nodes);  // the node list travels with the handle while it runs
    const cudaStream_t st = t->stream;
    const bool own = t->own_stream;
    *t = *tp;
    t->nodes.swap(nodes);
    t->stream = st;
    t->own_stream = own;
    t->entry = en;
    t->owns_events = false;
    t->ev_ok = en->ev_ok;
    for (int q = 0; q < 5; ++q) t->ev[q] = en->ev[q];
    t->launches = en->build_launches;
    t->d2h_bytes = 0;
    const cudaStream_t s = t->stream;
    const int64_t B = t->npairs;
    t->h2d_bytes = (rows_dev ? 0 : B * t->m_slab) + (cols_dev ? 0 : B * t->n);
    CK(en->released_valid ? cudaStreamWaitEvent(s, en->released, 0) : cudaSuccess);
    if (t->timing && t->ev_ok) CK(cudaEventRecord(t->ev[0], s));
    if (t->m_slab > 0)
        CK(cudaMemcpyAsync(t->d_rows, rows + (t->top_row - 1), (size_t)(B * t->m_slab),
                           rows_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (t->n > 0)
        CK(cudaMemcpyAsync(t->d_cols, cols, (size_t)(B * t->n),
                           cols_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    // combine time of a replayed build: the whole graph (the leaf step's three
    // small kernels included, ~15 us at cfg5 sizes)
    if (t->timing && t->ev_ok) CK(cudaEventRecord(t->ev[1], s));
    CK(cudaGraphLaunch(en->build, s));
    if (t->timing && t->ev_ok) CK(cudaEventRecord(t->ev[2], s));
    return LCSG_OK;
}

// After a normal build: keep its arena and capture its kernels as the
// shape's build graph (best effort: any failure leaves the handle normal).
void try_create_entry(lcsg_tree_s *t, const std::string &key) {
    // cache bounds: a quarter of the device's memory per arena, 35% in total (the
    // library's pool keeps a freed arena mapped anyway until lcsg_trim, so caching
    // it costs no extra HBM in steady state); LCSG_GRAPH_MAX_MB / _TOTAL_MB override
    size_t dev_free = 0, dev_total = 0;
    if (cudaMemGetInfo(&dev_free, &dev_total) != cudaSuccess) {
        cudaGetLastError();
        dev_total = (size_t)32 << 30;
    }
    const int def_max_mb = (int)std::min<size_t>(dev_total / 4 >> 20, 1u << 30);
    const int def_total_mb = (int)std::min<size_t>((dev_total / 20 * 7) >> 20, 1u << 30);
    const size_t max_bytes = (size_t)std::max(0, env_int("LCSG_GRAPH_MAX_MB", def_max_mb)) << 20;
    if (t->arena_bytes > max_bytes) return;
    const size_t max_total = (size_t)std::max(0, env_int("LCSG_GRAPH_TOTAL_MB", def_total_mb)) << 20;
    std::vector<SolveEntry *> evict;
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        size_t total = t->arena_bytes;
        for (SolveEntry *en : g_graph_cache) {
            if (en->key == key) return;  // the shape's entry is busy: no second one
            total += en->arena_bytes;
        }
        while (g_graph_cache.size() >= GRAPH_MAX_ENTRIES || total > max_total) {
            SolveEntry *lru = nullptr;
            for (SolveEntry *en : g_graph_cache)
                if (!en->in_use && (!lru || en->last_use < lru->last_use)) lru = en;
            if (!lru) break;  // all busy
            g_graph_cache.erase(std::find(g_graph_cache.begin(), g_graph_cache.end(), lru));
            total -= lru->arena_bytes;
            evict.push_back(lru);
        }
    }
    for (SolveEntry *en : evict) free_entry(en);
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        if (g_graph_cache.size() >= GRAPH_MAX_ENTRIES) return;
        size_t total = t->arena_bytes;
        for (SolveEntry *en : g_graph_cache) total += en->arena_bytes;
        if (total > max_total) return;
    }
    SolveEntry *en = new SolveEntry();
    en->key = key;
    en->device = t->device;
    bool ok = cudaStreamCreateWithFlags(&en->cap, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&en->released, cudaEventDisableTiming) == cudaSuccess;
    if (ok && t->timing) {
        en->ev_ok = true;
        for (auto &e : en->ev)
            if (cudaEventCreate(&e) != cudaSuccess) en->ev_ok = false;
    }
    if (ok) {
        en->tmpl = new lcsg_tree_s(*t);
        en->tmpl->leaf_cache.clear();
        en->tmpl->entry = nullptr;
        en->tmpl->owns_events = false;
        en->tmpl->ev_ok = en->ev_ok;
        for (int q = 0; q < 5; ++q) en->tmpl->ev[q] = en->ev[q];
        cudaGraph_t g = nullptr;
        ok = cudaStreamBeginCapture(en->cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            // timing events stay outside the graph (recorded around its launch)
            const int r = enqueue_build_kernels(en->tmpl, en->cap, &en->build_launches, false);
            const cudaError_t e = cudaStreamEndCapture(en->cap, &g);
            ok = r == 0 && e == cudaSuccess && g != nullptr;
        }
        if (ok) ok = cudaGraphInstantiate(&en->build, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();
    if (!ok) {
        en->arena = nullptr;  // the handle keeps its arena
        free_entry(en);
        return;
    }
    en->arena = t->arena;
    en->arena_bytes = t->arena_bytes;
    en->in_use = true;  // by t
    en->last_use = ++g_graph_tick;
    t->entry = en;
    std::lock_guard<std::mutex> lk(g_graph_mu);
    g_graph_cache.push_back(en);
}

int build_impl(const uint8_t *rows, bool rows_dev, int64_t m, const uint8_t *cols, bool cols_dev,
               int64_t n, int32_t top_row, int32_t bottom_row, uint32_t flags, int device,
               void *stream, lcsg_handle *out, int32_t npairs = 1) {
    if (!out) return fail(LCSG_EINVAL, "null output handle");
    *out = nullptr;
    if (m < 0 || n < 0) return fail(LCSG_EINVAL, "negative length");
    if (npairs < 1) return fail(LCSG_EINVAL, "npairs < 1");
    if (npairs > 1 && !(top_row == 1 && bottom_row == m + 1))
        return fail(LCSG_EINVAL, "batched builds cover the full grid");
    if (!(1 <= top_row && top_row < bottom_row && (int64_t)bottom_row <= m + 1))
        return fail(LCSG_EINVAL, "1 <= top_row < bottom_row <= m + 1");
    if (n > (int64_t)INT32_MAX - 4) return fail(LCSG_EINVAL, "column string too long for int32 tables");
    SaveDevice keep_caller_device;
    int rc = prepare_device(device);
    if (rc) return rc;

    lcsg_tree_s *t = new lcsg_tree_s();
    t->device = device;
    t->m_grid = m;
    t->m_slab = bottom_row - top_row;
    t->n = n;
    t->inf = (int32_t)(n + 2);
    t->top_row = top_row;
    t->bottom_row = bottom_row;
    t->with_trace = (flags & LCSG_WITH_TRACE) != 0;
    t->timing = (flags & LCSG_TIMING) != 0;
    t->npairs = npairs;
    if (stream) {
        t->stream = (cudaStream_t)stream;
    } else {
        if (cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete t;
            return fail(LCSG_ECUDA, "cudaStreamCreate failed");
        }
        t->own_stream = true;
    }
    if (t->timing) {
        t->ev_ok = true;
        for (auto &e : t->ev)
            if (cudaEventCreate(&e) != cudaSuccess) t->ev_ok = false;
    }

    // a repeated shape replays its CUDA graph (per-shape graph cache above)
    const bool graph_on = env_int("LCSG_GRAPH", 1) != 0;
    std::string gkey;
    if (graph_on) {
        gkey = graph_key(device, m, top_row, bottom_row, n, npairs, flags);
        if (SolveEntry *en = acquire_entry(gkey)) {
            if (t->ev_ok)
                for (auto &e : t->ev) cudaEventDestroy(e);
            t->ev_ok = false;
            const int r = graph_build(t, en, rows, rows_dev, cols, cols_dev);
            if (r) {
                destroy(t);
                return r;
            }
            *out = t;
            return LCSG_OK;
        }
    }
    // LCSG_HOST_PROFILE=1: host-side phase times of this call to stderr
    const bool hprof = env_int("LCSG_HOST_PROFILE", 0) != 0;
    auto hclock = [] { return std::chrono::steady_clock::now(); };
    auto hms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto h0 = hclock();
    // skeleton stride: 32 rows for small column counts (the extra skeleton
    // rows are cheaper than the latency of a coarser refinement stage), 64
    // above (measured on cfg2/cfg3 vs cfg4/cfg5)
    const int skel_stride = std::max(1, env_int("LCSG_SKELETON_STRIDE", default_skeleton_stride(n + 1)));
    const int thread_max_w1 = env_int("LCSG_THREAD_MAX_W1", 65);
    // virtual height-1 nodes (LCSG_VIRTUAL_H1=0 materialises them)
    const int virt_on = (env_int("LCSG_VIRTUAL_H1", 1) != 0 && n >= 2) ? 1 : 0;
    // the tree and the table layout depend only on the shape and the knobs:
    // a repeated shape reuses them (saves ~0.5 ms of host work at cfg5 before
    // the first kernel can be enqueued)
    LayoutCache &lc = t_layout;
    const bool layout_hit = lc.valid && lc.top_row == top_row && lc.bottom_row == bottom_row &&
                            lc.n == n && lc.with_trace == t->with_trace &&
                            lc.skel_stride == skel_stride && lc.thread_max_w1 == thread_max_w1 &&
                            lc.virt_on == virt_on;
    t->nodes.swap(t_spare_nodes);  // keeps the capacity of an earlier solve
    t->nodes.clear();
    if (layout_hit) {
        t->nodes.assign(lc.nodes.begin(), lc.nodes.end());
        t->root = lc.root;
    } else {
        t->nodes.reserve(2 * t->m_slab);
        t->root = build_tree(t, top_row, bottom_row, 0);
    }
    const int32_t nn1 = (int32_t)t->nodes.size();  // nodes of one pair
    const int32_t nn = nn1 * npairs;
    const int64_t B = npairs;
    t->pair_nodes = nn1;
    const int64_t n1 = n + 1;

    // ---- arena layout ----
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off = align_up(off + bytes);
        return o;
    };
    const int64_t kmin = std::min<int64_t>(t->m_slab, n);
    size_t o_rows = take((size_t)(B * t->m_slab));
    size_t o_cols = take((size_t)std::max<int64_t>(B * n, 1));
    size_t o_nx = take((size_t)(B * 256 * n1 * 4));
    size_t o_symw = take((size_t)B * 256 * 4);
    size_t o_nodew = take((size_t)nn * 4);
    size_t o_wi = take((size_t)nn * 4), o_wj = take((size_t)nn * 4);
    size_t o_path = take((size_t)(B * (t->m_slab + 1)) * 4);
    size_t o_out = take((size_t)(B * (1 + 2 * std::max<int64_t>(kmin, 1))) * 4);
    size_t o_sub = take((size_t)(B * std::max<int64_t>(kmin, 1)));
    const int skel_thread_max = env_int("LCSG_SKEL_THREAD_MAX_W1", 65);
    const int skel_warp_max = env_int("LCSG_SKEL_WARP_MAX_W1", 257);
    // refinement mode: tiled (default) or one launch per pass ("LCSG_REFINE_PASSES=1")
    const bool tiled = env_int("LCSG_REFINE_PASSES", 0) == 0;
    const bool narrow_on = env_int("LCSG_NARROW", 1) != 0;
    // wide combines: row sweep below the skeleton rows (LCSG_SWEEP=0: the
    // column-refinement stages)
    const bool sweep_on = env_int("LCSG_SWEEP", 1) != 0;
    int sm_count = 0;
    if (cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) {
        cudaGetLastError();
        sm_count = 0;
    }
    const int sweep_stride = std::max(2, env_int("LCSG_SWEEP_STRIDE", default_sweep_stride(n + 1)));
    // block size (local rows) of each column-refinement stage, power of two
    int col_block = 1;
    while (col_block * 2 <= std::min(16, std::max(2, env_int("LCSG_COL_BLOCK", default_col_block(n1)))))
        col_block *= 2;
    size_t o_tab = off;
    // int32 tables of every combine node
    int64_t tab_elems = 0, scratch_elems = 0;
    int32_t ncomb = 0;
    int32_t maxh0 = 0;
    if (layout_hit) {
        t->nleaves = lc.nleaves;
        t->nvirt = lc.nvirt;
        ncomb = lc.ncomb;
        maxh0 = lc.maxh0;
        tab_elems = lc.tab_elems;
        scratch_elems = lc.scratch_elems;
    } else {
        for (auto &nd : t->nodes) {
            if (nd.upper < 0) { t->nleaves++; continue; }
            ++ncomb;
            maxh0 = std::max(maxh0, nd.height);
            // the refinement kernels read both children as materialised slabs
            const bool kids_are_slabs =
                t->nodes[nd.upper].upper >= 0 && t->nodes[nd.lower].upper >= 0;
            nd.kind = (nd.w1 <= thread_max_w1 || !kids_are_slabs) ? 0 : 2;
            // the refinement kernels use 32-bit element offsets into each table
            if (nd.kind == 2 && n1 * (int64_t)nd.w1 >= ((int64_t)1 << 32)) nd.kind = 1;
            if (skel_stride == 1 && nd.kind == 2) nd.kind = 1;
        }
        // height-1 children of narrow (kind 0) combines are virtual: those
        // kernels read them through TabAcc / stage_rows, which evaluate the
        // closed form from NX (the wide kernels need materialised slabs)
        if (virt_on)
            for (auto &nd : t->nodes) {
                if (nd.upper < 0 || nd.kind != 0) continue;
                for (int32_t ch : {nd.upper, nd.lower}) {
                    NodeH &cn = t->nodes[ch];
                    if (cn.upper >= 0 && cn.height == 1 && !cn.virt) {
                        cn.virt = true;
                        ++t->nvirt;
                    }
                }
            }
        for (auto &nd : t->nodes) {
            if (nd.upper < 0 || nd.virt) continue;
            // every table starts on a 128-byte boundary (vector / async copies)
            tab_elems = (tab_elems + 31) / 32 * 32;
            nd.reach_off = tab_elems;
            tab_elems += n1 * nd.w1;
            if (t->with_trace) {
                tab_elems = (tab_elems + 31) / 32 * 32;
                nd.trace_off = tab_elems;
                tab_elems += n1 * nd.w1;
            }
        }
        // kmax rows of every combine (written by the kernel that finishes each row:
        // narrow / skeleton / finalize -- no initialisation needed)
        for (auto &nd : t->nodes) {
            if (nd.upper < 0 || nd.virt) continue;
            nd.kmax_off = tab_elems;
            tab_elems += (n1 + 63) / 64 * 64;
            nd.ev_off = tab_elems;  // per-row insertion ranks (row-sweep kernels)
            tab_elems += (n1 + 63) / 64 * 64;
        }
        // low-memory mode: the refinement passes still need this level's traces
        // (they bound neighbouring rows); one scratch region reused level by level
        std::vector<int64_t> level_scratch(maxh0 + 1, 0);
        if (!t->with_trace) {
            for (auto &nd : t->nodes)
                if (nd.upper >= 0 && nd.kind == 2) {
                    level_scratch[nd.height] = (level_scratch[nd.height] + 31) / 32 * 32;
                    nd.trace_off = level_scratch[nd.height];  // relative to the scratch base
                    level_scratch[nd.height] += n1 * nd.w1;
                }
            for (int64_t v : level_scratch) scratch_elems = std::max(scratch_elems, v);
        }
        lc.valid = true;
        lc.top_row = top_row;
        lc.bottom_row = bottom_row;
        lc.n = n;
        lc.with_trace = t->with_trace;
        lc.skel_stride = skel_stride;
        lc.thread_max_w1 = thread_max_w1;
        lc.virt_on = virt_on;
        lc.nvirt = t->nvirt;
        lc.nodes.assign(t->nodes.begin(), t->nodes.end());
        lc.root = t->root;
        lc.nleaves = t->nleaves;
        lc.ncomb = ncomb;
        lc.maxh0 = maxh0;
        lc.tab_elems = tab_elems;
        lc.scratch_elems = scratch_elems;
    }
    // pair p's tables occupy [p * pair_tab, (p+1) * pair_tab); the low-memory
    // level scratch of every pair follows all of them
    const int64_t pair_tab = (tab_elems + 31) / 32 * 32;
    t->pair_tab = pair_tab;
    const int64_t scratch_base = B * pair_tab;
    tab_elems = scratch_base + B * scratch_elems;
    if (B > 1) {  // replicate the tree of pair 0 for the other pairs
        t->nodes.resize((size_t)nn);
        for (int32_t p = 1; p < npairs; ++p)
            for (int32_t id = 0; id < nn1; ++id) {
                NodeH nd = t->nodes[id];
                nd.pair = p;
                if (nd.upper >= 0) {
                    nd.upper += p * nn1;
                    nd.lower += p * nn1;
                }
                if (nd.leaf_row >= 0) nd.leaf_row += (int32_t)(p * t->m_slab);
                if (nd.reach_off >= 0) nd.reach_off += p * pair_tab;
                if (nd.kmax_off >= 0) nd.kmax_off += p * pair_tab;
                if (nd.ev_off >= 0) nd.ev_off += p * pair_tab;
                if (nd.trace_off >= 0) nd.trace_off += t->with_trace ? p * pair_tab : p * scratch_elems;
                t->nodes[(size_t)p * nn1 + id] = nd;
            }
        ncomb *= npairs;
        t->nleaves *= npairs;
        t->nvirt *= npairs;
    }
    off = align_up(o_tab + (size_t)tab_elems * 4);
    // row-sweep block flags: one int per block of rows (>= 2 rows) of every kind-2 node
    const int64_t fstride = (n1 / 2 + 64) / 32 * 32;
    int64_t nflag = 0;
    for (auto &nd : t->nodes)
        if (nd.upper >= 0 && nd.kind == 2) nd.flag_off = (nflag++) * fstride;
    t->flags_bytes = (size_t)(nflag * fstride) * 4;
    size_t o_flags = take(std::max<size_t>(t->flags_bytes, 4));
    // metadata region (uploaded with one copy)
    size_t o_meta = off;
    size_t o_desc = take((size_t)std::max(ncomb, 1) * sizeof(CombineDesc));
    size_t o_walk = take((size_t)nn * sizeof(WalkNode));
    size_t o_wids = take((size_t)std::max(ncomb, 1) * 4);
    size_t o_lnodes = take((size_t)std::max(t->nleaves, 1) * 4);
    size_t o_lrows = take((size_t)std::max(t->nleaves, 1) * 4);
    size_t o_vnodes = take((size_t)std::max(t->nvirt, 1) * 16);
    size_t meta_end = off;
    t->arena_bytes = off;

    const auto h1 = hclock();
    cudaError_t ae = pool_alloc((void **)&t->arena, t->arena_bytes, device, t->stream);
    const auto h2 = hclock();
    if (ae != cudaSuccess) {
        t->arena = nullptr;
        destroy(t);
        return fail(LCSG_ENOMEM, std::string("cudaMallocAsync(") + std::to_string(off) +
                                     " B): " + cudaGetErrorString(ae));
    }
    char *A = t->arena;
    t->d_rows = (uint8_t *)(A + o_rows);
    t->d_cols = (uint8_t *)(A + o_cols);
    t->d_nx = (int32_t *)(A + o_nx);
    t->d_sym_wstar = (int32_t *)(A + o_symw);
    t->d_node_wstar = (int32_t *)(A + o_nodew);
    t->d_wi = (int32_t *)(A + o_wi);
    t->d_wj = (int32_t *)(A + o_wj);
    t->d_path = (int32_t *)(A + o_path);
    t->d_out = (int32_t *)(A + o_out);
    t->d_subseq = (uint8_t *)(A + o_sub);
    t->d_tables = (int32_t *)(A + o_tab);
    t->d_descs = (CombineDesc *)(A + o_desc);
    t->d_walk = (WalkNode *)(A + o_walk);
    t->d_walk_ids = (int32_t *)(A + o_wids);
    t->d_leaf_nodes = (int32_t *)(A + o_lnodes);
    t->d_leaf_rows = (int32_t *)(A + o_lrows);
    t->d_vnodes = (int32_t *)(A + o_vnodes);
    t->d_flags = (int32_t *)(A + o_flags);

    // ---- host-side metadata: level plan, descriptors, walk nodes ----
    const size_t meta_bytes = meta_end - o_meta;
    std::vector<char> meta_fallback;
    MetaLease lease;
    char *meta = lease.acquire(device, meta_bytes, t->stream);
    const bool meta_pinned = meta != nullptr;
    if (!meta_pinned) {
        meta_fallback.assign(meta_bytes, 0);
        meta = meta_fallback.data();
    }  // no zero-fill: every descriptor / walk-node field is written below
    CombineDesc *hd = (CombineDesc *)(meta + (o_desc - o_meta));
    WalkNode *hw = (WalkNode *)(meta + (o_walk - o_meta));
    int32_t *hids = (int32_t *)(meta + (o_wids - o_meta));
    int32_t *hln = (int32_t *)(meta + (o_lnodes - o_meta));
    int32_t *hlr = (int32_t *)(meta + (o_lrows - o_meta));
    int32_t *hvn = (int32_t *)(meta + (o_vnodes - o_meta));

    // ---- enqueue: inputs, leaf step; then the levels as they are planned ----
    const cudaStream_t s = t->stream;
#define BCK(call)                            \
    do {                                     \
        int r__ = 0;                         \
        cudaError_t e__ = (call);            \
        if (e__ != cudaSuccess) {            \
            r__ = fail(LCSG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
            lease.finish(); destroy(t);                      \
            return r__;                      \
        }                                    \
    } while (0)
#define BCKL(call)                           \
    do {                                     \
        int e__ = (call);                    \
        if (e__ != 0) {                      \
            int r__ = fail(LCSG_ECUDA, std::string("launch ") + #call + ": " +      \
                                           cudaGetErrorString((cudaError_t)e__));   \
            lease.finish(); destroy(t);                      \
            return r__;                      \
        }                                    \
        ++t->launches;                       \
    } while (0)

    int32_t li = 0, vi = 0;
    for (int32_t id = 0; id < nn; ++id) {
        const NodeH &nd = t->nodes[id];
        if (nd.upper < 0) {
            hln[li] = id;
            hlr[li] = nd.leaf_row;
            ++li;
        } else if (nd.virt) {
            hvn[4 * vi] = id;
            hvn[4 * vi + 1] = t->nodes[nd.upper].leaf_row;
            hvn[4 * vi + 2] = t->nodes[nd.lower].leaf_row;
            hvn[4 * vi + 3] = nd.pair;
            ++vi;
        }
    }

    if (t->timing && t->ev_ok) BCK(cudaEventRecord(t->ev[0], s));
    const uint8_t *rows_slab = rows + (top_row - 1);
    if (t->m_slab > 0)  // batched: full grids, so the pairs' slabs are contiguous
        BCK(cudaMemcpyAsync(t->d_rows, rows_slab, (size_t)(B * t->m_slab),
                            rows_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    if (n > 0)
        BCK(cudaMemcpyAsync(t->d_cols, cols, (size_t)(B * n),
                            cols_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
    // leaf lists now; the level descriptors are uploaded in groups as they
    // are planned (their kernels start while the host plans the next
    // levels), the walk nodes (extraction only) after the last level
    BCK(cudaMemcpyAsync(A + o_lnodes, meta + (o_lnodes - o_meta), meta_end - o_lnodes,
                        cudaMemcpyHostToDevice, s));
    t->h2d_bytes = (int64_t)meta_bytes + (rows_dev ? 0 : B * t->m_slab) + (cols_dev ? 0 : B * n);
    // a pageable fallback copy is staged synchronously, so `meta_fallback` may die
    BCK(cudaMemsetAsync(t->d_node_wstar, 0, (size_t)nn * 4, s));
    if (t->flags_bytes) BCK(cudaMemsetAsync(t->d_flags, 0, t->flags_bytes, s));
    BCKL(launch_nx(t->d_cols, (int32_t)n, npairs, t->d_nx, t->d_sym_wstar, s));
    BCKL(launch_leaf_wstar(t->d_rows, t->d_leaf_nodes, t->d_leaf_rows, t->nleaves,
                           (int32_t)std::max<int64_t>(t->m_slab, 1), t->d_sym_wstar,
                           t->d_node_wstar, s));
    const Ctx c = t->ctx();
    if (t->nvirt > 0) BCKL(launch_virtual_wstar(c, t->d_vnodes, t->nvirt, t->d_node_wstar, s));
    bool ev1_done = false;  // ev[1]: just before the first level's descriptors
    SideLease side;
    side.acquire(device);
    auto launch_entry = [&](const LaunchH &L) -> int { return launch_plan_entry_side(t, L, s, side); };
    int32_t maxh = 0;
    for (auto &nd : t->nodes) maxh = std::max(maxh, nd.height);
    const int vbits = bits_for(t->inf);
    int32_t di = 0;
    // node ids bucketed by height (ascending id order kept): O(nodes) planning
    std::vector<std::vector<int32_t>> by_height(maxh + 1);
    for (int32_t id = 0; id < nn; ++id)
        if (t->nodes[id].upper >= 0 && !t->nodes[id].virt)
            by_height[t->nodes[id].height].push_back(id);
    // levels are flushed (descriptors copied, kernels launched) in three
    // groups -- the first level, the next two, the rest -- so the GPU starts
    // early and runs while the host plans, with only three extra copies in
    // the stream (one copy per level cost ~0.1 ms of gaps between kernels)
    int32_t level_di = 0, nplanned = 0;
    size_t level_plan = 0;
    for (int32_t h = 1; h <= maxh; ++h) {
        const int32_t h_di = di;
        for (int kind = 0; kind < 3; ++kind) {
            int32_t start = di;
            int32_t maxk = 0, maxw1 = 0, maxkl = 0, minw1 = INT32_MAX;
            bool ev_make_any = false;
            for (const int32_t id : by_height[h]) {
                const NodeH &nd = t->nodes[id];
                if (nd.kind != kind) continue;
                CombineDesc &d = hd[di++];
                d.U = t->tab(nd.upper);
                d.L = t->tab(nd.lower);
                d.out_reach = t->d_tables + nd.reach_off;
                d.out_trace = t->with_trace ? t->d_tables + nd.trace_off
                              : (kind == 2 ? t->d_tables + scratch_base + nd.trace_off : nullptr);
                d.out_kmax = t->d_tables + nd.kmax_off;
                d.out_wstar = t->d_node_wstar + id;
                d.w1 = nd.w1;
                d.node = id;
                {
                    const NodeH &un = t->nodes[nd.upper];
                    d.U_ev = un.ev_off >= 0 ? t->d_tables + un.ev_off : nullptr;
                    d.out_ev = t->d_tables + nd.ev_off;
                    // a kind-2 child's events are a by-product of its own sweep
                    d.U_ev_make = (kind == 2 && sweep_on && un.kind != 2) ? 1 : 0;
                    d.pad_ = 0;
                    d.blk_flags = nd.flag_off >= 0 ? t->d_flags + nd.flag_off : nullptr;
                    if (d.U_ev_make) ev_make_any = true;
                }
                maxk = std::max(maxk, t->nodes[nd.upper].w1 - 1);
                maxkl = std::max(maxkl, t->nodes[nd.lower].w1 - 1);
                maxw1 = std::max(maxw1, nd.w1);
                minw1 = std::min(minw1, nd.w1);
            }
            if (di == start) continue;
            LaunchH L;
            L.desc_off = start;
            L.count = di - start;
            L.shift = bits_for(maxk);
            L.key64 = need_key64(vbits, L.shift);
            if (kind < 2) {
                // narrow thread-per-row tables: shared-memory staged row writes
                L.kind = (kind == 0 && maxw1 <= 33 && env_int("LCSG_STAGED_ROWS", 0)) ? 9 : kind;
                const int P = narrow_bucket(std::max(maxk, maxkl));
                if (kind == 0 && P > 0 && narrow_on) {
                    L.kind = 10;
                    L.stride_or_delta = P;
                    L.wpr_log2 = (minw1 == maxw1 && maxw1 == 2 * P + 1 &&
                                  env_int("LCSG_NARROW_FW", 1)) ? 1 : 0;  // full width
                    // height 1: both children are leaves
                    if (h == 1 && env_int("LCSG_LEAFPAIR", 1)) L.kind = 11;
                }
                t->plan.push_back(L);
                continue;
            }
            // skeleton + refinement passes
            // per-height overrides (tuning knobs): LCSG_SKEL_STRIDE_H<h>, LCSG_COL_BLOCK_H<h>
            const std::string hs = std::to_string(h);
            // many narrow-ish wide tables (w1 <= 513, >= 32 combines) of long
            // strings: skeleton rows every 512 (row steps 64, 8, 1) -- cheaper
            // than the skeleton bisection every 64 rows (measured: cfg5 levels
            // s = 128..512 gain 0.4 ms; cfg4's 2..8-combine levels lose 0.2)
            // (re-measured after the fine-kernel changes: the root's stride 32
            // now loses 0.14 ms against 64, so only the 512 rule remains)
            const bool dflt = getenv("LCSG_SKELETON_STRIDE") == nullptr && n1 > 8193;
            const int stride_def = sweep_on ? sweep_stride
                                   : (dflt && maxw1 <= 513 && L.count >= 32) ? 512 : skel_stride;
            const int stride_h =
                std::max(2, env_int(("LCSG_SKEL_STRIDE_H" + hs).c_str(), stride_def));
            int32_t S = 1;
            while (S * 2 <= stride_h) S *= 2;
            if (sweep_on) {  // the sweep takes any block size
                S = std::min(stride_h, 1024);
                if (getenv(("LCSG_SKEL_STRIDE_H" + hs).c_str()) == nullptr &&
                    getenv("LCSG_SWEEP_STRIDE") == nullptr)
                    S = sweep_pick_block(S, maxw1, L.count, (int32_t)n, L.shift, L.key64, sm_count);
            }
            int32_t cb = col_block;
            const int cb_env = env_int(("LCSG_COL_BLOCK_H" + hs).c_str(), 0);
            if (cb_env > 0) {
                cb = 1;
                while (cb * 2 <= std::min(16, std::max(2, cb_env))) cb *= 2;
            }
            // skeleton rows: thread-per-row DFS for narrow tables, warp-per-row
            // DFS for medium, CTA-per-row (cooperative top rounds) for wide
            L.kind = maxw1 <= skel_thread_max ? 5 : (maxw1 <= skel_warp_max ? 6 : 3);
            L.stride_or_delta = S;
            t->plan.push_back(L);
            if (sweep_on) {  // row sweep below every skeleton row + finalize (lcsg_sweep.cu)
                if (ev_make_any) {
                    LaunchH E = L;
                    E.kind = 12;
                    t->plan.push_back(E);
                }
                LaunchH W = L;
                W.kind = 13;
                W.stride_or_delta = S;
                W.ustride = maxw1;
                t->plan.push_back(W);
                LaunchH F = L;
                F.kind = 8;
                F.stride_or_delta = S;
                F.ustride = maxw1;
                F.wpr_log2 = 1;  // kmax is the sweep's
                t->plan.push_back(F);
                continue;
            }
            if (tiled) {  // column-refinement stages (row step S/B, S/B^2, .., 1) + finalize
                int32_t rem = S;
                while (rem > 1) {
                    const int32_t B = std::min<int32_t>(cb, rem);
                    LaunchH P = L;
                    P.kind = 7;
                    P.stride_or_delta = B;
                    P.wpr_log2 = rem / B;  // row step of this stage
                    P.ustride = maxw1;
                    t->plan.push_back(P);
                    rem /= B;
                }
                LaunchH F = L;
                F.kind = 8;
                F.stride_or_delta = S;
                F.ustride = maxw1;
                t->plan.push_back(F);
                continue;
            }
            for (int32_t dl = S / 2; dl >= 1; dl /= 2) {
                LaunchH P = L;
                P.kind = 4;
                P.stride_or_delta = dl;
                t->plan.push_back(P);
            }
        }
        if (di > h_di) ++nplanned;
        if (!(h == maxh || (di > h_di && (nplanned == 1 || nplanned == 3)))) continue;
        if (!ev1_done && di > level_di) {
            if (t->timing && t->ev_ok) BCK(cudaEventRecord(t->ev[1], s));
            ev1_done = true;
        }
        if (di > level_di)  // the group's descriptors, then its kernels
            BCK(cudaMemcpyAsync(t->d_descs + level_di, hd + level_di,
                                (size_t)(di - level_di) * sizeof(CombineDesc),
                                cudaMemcpyHostToDevice, s));
        for (size_t pi = level_plan; pi < t->plan.size(); ++pi) {
            const int e = launch_entry(t->plan[pi]);
            if (e > 0) {
                const int r = fail(LCSG_ECUDA, std::string("launch: ") +
                                                   cudaGetErrorString((cudaError_t)e));
                side.join(s);
                lease.finish(); destroy(t);
                return r;
            }
            if (e == 0) {
                const LaunchH &PL = t->plan[pi];
                t->launches += PL.kind == 13 ? sweep_launch_count(PL.shift, PL.key64, PL.stride_or_delta, PL.ustride) : 1;
            }
        }
        level_di = di;
        level_plan = t->plan.size();
    }
    BCKL(side.join(s));
    --t->launches;  // the join is not a kernel
    const auto h3 = hclock();
    if (!ev1_done && t->timing && t->ev_ok) BCK(cudaEventRecord(t->ev[1], s));  // no combines
    if (t->timing && t->ev_ok) BCK(cudaEventRecord(t->ev[2], s));
    // walk nodes + depth lists of internal nodes
    int32_t maxd = 0, maxku = 0;
    for (int32_t id = 0; id < nn; ++id) {
        const NodeH &nd = t->nodes[id];
        WalkNode &w = hw[id];
        // relative: path index = top_row - 1 (pair p's path after the others')
        w.top_row = nd.top_row - t->top_row + 1 + (int32_t)(nd.pair * (t->m_slab + 1));
        w.bottom_row = nd.bottom_row;
        w.upper = nd.upper;
        w.lower = nd.lower;
        w.w1 = nd.w1;
        w.is_leaf = nd.upper < 0;
        w.trace = (nd.upper >= 0 && !nd.virt && t->with_trace) ? t->d_tables + nd.trace_off
                                                                : nullptr;
        if (nd.upper >= 0) {
            w.U = t->tab(nd.upper);
            w.L = t->tab(nd.lower);
            maxku = std::max(maxku, t->nodes[nd.upper].w1 - 1);
        } else {
            w.U = TabDev{};
            w.L = TabDev{};
        }
        maxd = std::max(maxd, nd.depth);
    }
    t->walk_shift = bits_for(maxku);
    t->walk_key64 = need_key64(vbits, t->walk_shift);
    int32_t wpos = 0;
    std::vector<std::vector<int32_t>> by_depth(maxd + 1);
    for (int32_t id = 0; id < nn; ++id)
        if (t->nodes[id].upper >= 0) by_depth[t->nodes[id].depth].push_back(id);
    for (int32_t dd = 0; dd <= maxd; ++dd) {
        int32_t start = wpos;
        for (const int32_t id : by_depth[dd]) hids[wpos++] = id;
        if (wpos > start) t->depth_ranges.push_back({start, wpos - start});
    }
    BCK(cudaMemcpyAsync(A + o_walk, meta + (o_walk - o_meta), o_lnodes - o_walk,
                        cudaMemcpyHostToDevice, s));
    if (hprof) {
        const auto h4 = hclock();
        fprintf(stderr, "lcsg_build host ms: tree+layout %.3f  arena %.3f  metadata %.3f  enqueue %.3f\n",
                hms(h0, h1), hms(h1, h2), hms(h2, h3), hms(h3, h4));
    }
#undef BCK
#undef BCKL
    lease.finish();
    if (graph_on) try_create_entry(t, gkey);
    *out = t;
    return LCSG_OK;
}

bool full_grid(const lcsg_tree_s *t) { return t->top_row == 1 && t->bottom_row == t->m_grid + 1; }

// recovery walk for weight j from start column i_start (j < 0: the largest
// weight from i_start, read on the device)
int enqueue_walk(lcsg_tree_s *t, cudaStream_t s, int32_t j, int32_t i_start, int64_t *launches) {
    const Ctx c = t->ctx();
    const TabDev rt = t->tab(t->root);
    int r = launch_walk_root(t->d_walk, t->root, c, rt, j, i_start, t->d_wi, t->d_wj, t->d_path,
                             t->root_batch(), s);
    if (r) return r;
    int64_t nl = 1;
    const bool retrace = !t->with_trace;
    for (auto &dr : t->depth_ranges) {
        r = launch_walk_level(t->d_walk, t->d_walk_ids + dr.first, dr.second, c, t->d_wi, t->d_wj,
                              t->d_path, retrace, t->walk_shift, t->walk_key64, s);
        if (r) return r;
        ++nl;
    }
    r = launch_walk_final(c, rt, i_start, (int32_t)t->m_slab, t->root, t->d_wj, t->d_path,
                          t->root_batch(), s);
    if (r) return r;
    if (launches) *launches = nl + 1;
    return 0;
}

// recovery walk for weight j from start column i_start (j < 0: the largest
// weight from i_start, read on the device); a handle on a graph-cache entry
// replays the shape's walk graph for the LCS walk (j < 0 from column 1)
int run_walk(lcsg_tree_s *t, int32_t j, int32_t i_start = 1) {
    SolveEntry *en = t->entry;
    if (en && j < 0 && i_start == 1 && !en->walk_failed) {
        if (!en->walk) {  // capture once (the entry is in use by this handle only)
            cudaGraph_t g = nullptr;
            bool ok = cudaStreamBeginCapture(en->cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
            if (ok) {
                const int r = enqueue_walk(t, en->cap, -1, 1, &en->walk_launches);
                ok = cudaStreamEndCapture(en->cap, &g) == cudaSuccess && r == 0 && g;
            }
            if (ok) ok = cudaGraphInstantiate(&en->walk, g, 0) == cudaSuccess;
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            if (!ok) {
                en->walk = nullptr;
                en->walk_failed = true;
            }
        }
        if (en->walk) {
            CK(cudaGraphLaunch(en->walk, t->stream));
            t->launches += en->walk_launches;
            return LCSG_OK;
        }
    }
    int64_t nl = 0;
    CKL(enqueue_walk(t, t->stream, j, i_start, &nl));
    t->launches += nl;
    return LCSG_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// lcs() (solver.py:237-273) of `npairs` pairs of equal shape: a / b hold the
// pairs back to back (la / lb bytes each); pair p's outputs land at
// length[p], subseq / pos_a / pos_b + p * min(la, lb).  One build of all the
// pairs' trees (one launch per height), one walk, one assembly.
int lcs_impl(const uint8_t *a, int64_t la, const uint8_t *b, int64_t lb, bool dev, uint32_t flags,
             int device, void *stream, int32_t *length, uint8_t *subseq, int32_t *pos_a,
             int32_t *pos_b, int32_t npairs = 1) {
    if (!length) return fail(LCSG_EINVAL, "null length pointer");
    if (npairs < 1) return fail(LCSG_EINVAL, "npairs < 1");
    for (int32_t p = 0; p < npairs; ++p) length[p] = 0;
    if (la == 0 || lb == 0) return LCSG_OK;  // solver.py:255-256
    const bool swapped = la > lb;             // solver.py:257-258
    const uint8_t *rows = swapped ? b : a, *cols = swapped ? a : b;
    const int64_t m = swapped ? lb : la, n = swapped ? la : lb;
    lcsg_handle h = nullptr;
    int rc = build_impl(rows, dev, m, cols, dev, n, 1, (int32_t)(m + 1), flags, device, stream, &h,
                        npairs);
    if (rc) return rc;
    DeviceGuard g(h->device);
    const int64_t k = std::min(m, n), ostride = 1 + 2 * k;
    rc = run_walk(h, -1);
    if (rc == 0) {
        int r2 = launch_assemble(h->d_rows, (int32_t)m, h->d_cols, (int32_t)n, h->d_path, h->d_out,
                                 h->d_out + 1, h->d_out + 1 + k, h->d_subseq, h->stream, npairs,
                                 ostride, k);
        if (r2) rc = fail(LCSG_ECUDA, std::string("assemble: ") + cudaGetErrorString((cudaError_t)r2));
        ++h->launches;
    }
    if (rc == 0) {
        std::vector<int32_t> hb((size_t)(npairs * ostride));
        std::vector<uint8_t> hs((size_t)(npairs * k));
        cudaError_t e = cudaMemcpyAsync(hb.data(), h->d_out, hb.size() * 4, cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hs.data(), h->d_subseq, hs.size(), cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess && h->timing && h->ev_ok) e = cudaEventRecord(h->ev[3], h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            rc = fail(LCSG_ECUDA, std::string("lcs result copy: ") + cudaGetErrorString(e));
        } else {
            h->d2h_bytes += (int64_t)(hb.size() * 4 + hs.size());
            for (int32_t p = 0; p < npairs; ++p) {
                const int32_t *ob = hb.data() + p * ostride;
                const int32_t len = ob[0];
                length[p] = len;
                int32_t *rp = swapped ? pos_b : pos_a, *cp = swapped ? pos_a : pos_b;
                if (subseq) std::memcpy(subseq + p * k, hs.data() + p * k, (size_t)len);
                if (rp) std::memcpy(rp + p * k, ob + 1, (size_t)len * 4);
                if (cp) std::memcpy(cp + p * k, ob + 1 + k, (size_t)len * 4);
            }
        }
    }
    destroy(h);
    return rc;
}

}  // namespace

extern "C" {

const char *lcsg_last_error(void) { return g_err.c_str(); }
int lcsg_abi_version(void) { return 100; }

int lcsg_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

int lcsg_build(const uint8_t *rows, int64_t m, const uint8_t *cols, int64_t n, int32_t top_row,
               int32_t bottom_row, uint32_t flags, int device, void *stream, lcsg_handle *out) {
    return build_impl(rows, false, m, cols, false, n, top_row, bottom_row, flags, device, stream, out);
}

int lcsg_build_device(const uint8_t *rows_dev, int64_t m, const uint8_t *cols_dev, int64_t n,
                      int32_t top_row, int32_t bottom_row, uint32_t flags, int device,
                      void *stream, lcsg_handle *out) {
    return build_impl(rows_dev, true, m, cols_dev, true, n, top_row, bottom_row, flags, device,
                      stream, out);
}

int lcsg_free(lcsg_handle h) {
    destroy(h);
    return LCSG_OK;
}

int lcsg_reserve(int device, int64_t bytes) {
    if (bytes < 0) return fail(LCSG_EINVAL, "negative size");
    SaveDevice keep_caller_device;
    int rc = prepare_device(device);
    if (rc) return rc;
    if (bytes == 0) return LCSG_OK;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        pool = g_pool[device];
    }
    // grow the pool once (physical backing mapped now, not inside the first
    // solve) and hand the block back: it stays in the pool (no release threshold)
    void *p = nullptr;
    CK(cudaMallocFromPoolAsync(&p, (size_t)bytes, pool, 0));
    CK(cudaFreeAsync(p, 0));
    CK(cudaStreamSynchronize(0));
    return LCSG_OK;
}

int lcsg_trim(int device) {
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (device < 0 || device >= 64) return fail(LCSG_EINVAL, "device index out of range");
        pool = g_pool[device];
    }
    std::vector<SolveEntry *> drop;
    {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        for (auto it = g_graph_cache.begin(); it != g_graph_cache.end();) {
            if ((*it)->device == device && !(*it)->in_use) {
                drop.push_back(*it);
                it = g_graph_cache.erase(it);
            } else {
                ++it;
            }
        }
    }
    for (SolveEntry *en : drop) free_entry(en);
    if (!pool) return LCSG_OK;  // nothing allocated on that device yet
    CK(cudaMemPoolTrimTo(pool, 0));
    return LCSG_OK;
}

int lcsg_sync(lcsg_handle h) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    DeviceGuard g(h->device);
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

int32_t lcsg_num_nodes(lcsg_handle h) { return h ? (int32_t)h->nodes.size() : -1; }
int32_t lcsg_root(lcsg_handle h) { return h ? h->root : -1; }

int lcsg_node_info(lcsg_handle h, int32_t node, int32_t *info) {
    if (!h || node < 0 || node >= (int32_t)h->nodes.size()) return fail(LCSG_EINVAL, "bad node");
    const NodeH &nd = h->nodes[node];
    info[0] = nd.top_row;
    info[1] = nd.bottom_row;
    info[2] = nd.w1;
    info[3] = nd.upper;
    info[4] = nd.lower;
    info[5] = (nd.upper >= 0 && h->with_trace) ? 1 : 0;
    info[6] = (int32_t)h->n;
    info[7] = h->inf;
    return LCSG_OK;
}

int lcsg_node_wstar(lcsg_handle h, int32_t node, int32_t *wstar) {
    if (!h || node < 0 || node >= (int32_t)h->nodes.size()) return fail(LCSG_EINVAL, "bad node");
    DeviceGuard g(h->device);
    CK(cudaMemcpyAsync(wstar, h->d_node_wstar + node, 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

// Leaves and virtual height-1 nodes have no table in the arena; the API
// materialises one on first access (reach [+ trace] + kmax, cached per node):
// leaves by leaf_table_kernel, virtual nodes by the leaf-pair combine kernel
// (the same kernel that computes a stored height-1 node, INF-cell traces
// included).
static int leaf_device(lcsg_handle h, int32_t node, int32_t **reach) {
    auto it = h->leaf_cache.find(node);
    if (it != h->leaf_cache.end()) {
        *reach = it->second;
        return LCSG_OK;
    }
    const NodeH &nd = h->nodes[node];
    const int64_t n1 = h->n + 1;
    int32_t *buf = nullptr;
    if (nd.virt) {
        // reach | trace | kmax | wstar, then the combine descriptor
        const size_t tab = (size_t)(n1 * nd.w1);
        const size_t desc_off = align_up((2 * tab + n1 + 1) * 4);
        CK(pool_alloc((void **)&buf, desc_off + sizeof(CombineDesc), h->device, h->stream));
        h->leaf_cache[node] = buf;
        CombineDesc d;
        std::memset(&d, 0, sizeof(d));
        d.U = h->tab(nd.upper);
        d.L = h->tab(nd.lower);
        d.out_reach = buf;
        d.out_trace = buf + tab;
        d.out_kmax = buf + 2 * tab;
        d.out_wstar = buf + 2 * tab + n1;
        d.w1 = nd.w1;
        d.node = node;
        CombineDesc *dd = (CombineDesc *)((char *)buf + desc_off);
        CK(cudaMemcpyAsync(dd, &d, sizeof(d), cudaMemcpyHostToDevice, h->stream));
        const int shift = bits_for(std::max(h->nodes[nd.upper].w1 - 1, 1));
        CKL(launch_narrow_leafpair(dd, 1, h->ctx(), shift, need_key64(bits_for(h->inf), shift),
                                   h->stream));
    } else {
        CK(pool_alloc((void **)&buf, (size_t)(n1 * nd.w1 + n1) * 4, h->device, h->stream));
        h->leaf_cache[node] = buf;
        CKL(launch_leaf_table(h->ctx(), nd.leaf_row, nd.w1, buf, buf + n1 * nd.w1, h->stream));
    }
    ++h->launches;
    *reach = buf;
    return LCSG_OK;
}

static bool materialised_on_demand(const NodeH &nd) { return nd.upper < 0 || nd.virt; }

int lcsg_node_reach_device(lcsg_handle h, int32_t node, void **dev_ptr) {
    if (!h || node < 0 || node >= (int32_t)h->nodes.size()) return fail(LCSG_EINVAL, "bad node");
    DeviceGuard g(h->device);
    const NodeH &nd = h->nodes[node];
    if (materialised_on_demand(nd)) {
        int32_t *p = nullptr;
        int rc = leaf_device(h, node, &p);
        if (rc) return rc;
        *dev_ptr = p;
    } else {
        *dev_ptr = h->d_tables + nd.reach_off;
    }
    return LCSG_OK;
}

static int copy_node(lcsg_handle h, int32_t node, int which, int32_t *host_out) {
    if (!h || node < 0 || node >= (int32_t)h->nodes.size()) return fail(LCSG_EINVAL, "bad node");
    DeviceGuard g(h->device);
    const NodeH &nd = h->nodes[node];
    const int64_t n1 = h->n + 1;
    const int32_t *src = nullptr;
    size_t elems = 0;
    if (nd.upper < 0) {
        if (which == 1) return fail(LCSG_EINVAL, "leaf tables carry no trace");
        int32_t *p = nullptr;
        int rc = leaf_device(h, node, &p);
        if (rc) return rc;
        src = which == 0 ? p : p + n1 * nd.w1;
        elems = which == 0 ? (size_t)(n1 * nd.w1) : (size_t)n1;
    } else if (nd.virt) {
        if (which == 1 && !h->with_trace) return fail(LCSG_EINVAL, "table was built without traces");
        int32_t *p = nullptr;
        int rc = leaf_device(h, node, &p);
        if (rc) return rc;
        const size_t tab = (size_t)(n1 * nd.w1);
        src = p + which * tab;  // reach | trace | kmax
        elems = which == 2 ? (size_t)n1 : tab;
    } else if (which == 0) {
        src = h->d_tables + nd.reach_off;
        elems = (size_t)(n1 * nd.w1);
    } else if (which == 1) {
        if (!h->with_trace) return fail(LCSG_EINVAL, "table was built without traces");
        src = h->d_tables + nd.trace_off;
        elems = (size_t)(n1 * nd.w1);
    } else {
        src = h->d_tables + nd.kmax_off;
        elems = (size_t)n1;
    }
    CK(cudaMemcpyAsync(host_out, src, elems * 4, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

int lcsg_node_reach(lcsg_handle h, int32_t node, int32_t *o) { return copy_node(h, node, 0, o); }
int lcsg_node_trace(lcsg_handle h, int32_t node, int32_t *o) { return copy_node(h, node, 1, o); }
int lcsg_node_kmax(lcsg_handle h, int32_t node, int32_t *o) { return copy_node(h, node, 2, o); }

int lcsg_length(lcsg_handle h, int32_t *length) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    DeviceGuard g(h->device);
    const NodeH &r = h->nodes[h->root];
    if (r.upper < 0) {
        int32_t *p = nullptr;
        int rc = leaf_device(h, h->root, &p);
        if (rc) return rc;
        CK(cudaMemcpyAsync(length, p + (h->n + 1) * r.w1, 4, cudaMemcpyDeviceToHost, h->stream));
    } else {
        CK(cudaMemcpyAsync(length, h->d_tables + r.kmax_off, 4, cudaMemcpyDeviceToHost, h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

int lcsg_recover(lcsg_handle h, int32_t j, int32_t *cols_out) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    if (!full_grid(h)) return fail(LCSG_EINVAL, "recovery needs the full-grid table");
    int32_t len = 0;
    int rc = lcsg_length(h, &len);
    if (rc) return rc;
    if (j > len) return fail(LCSG_ERANGE, "no path of weight " + std::to_string(j) +
                                              " exists (max " + std::to_string(len) + ")");
    if (j < 0) return fail(LCSG_EINVAL, "negative weight");
    DeviceGuard g(h->device);
    rc = run_walk(h, j);
    if (rc) return rc;
    CK(cudaMemcpyAsync(cols_out, h->d_path, (size_t)(h->m_slab + 1) * 4, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

int lcsg_extract(lcsg_handle h, int32_t j, int32_t *length, uint8_t *subseq, int32_t *row_pos,
                 int32_t *col_pos) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    if (!full_grid(h)) return fail(LCSG_EINVAL, "recovery needs the full-grid table");
    DeviceGuard g(h->device);
    if (j >= 0) {
        int32_t len = 0;
        int rc = lcsg_length(h, &len);
        if (rc) return rc;
        if (j > len) return fail(LCSG_ERANGE, "no path of weight " + std::to_string(j) +
                                                  " exists (max " + std::to_string(len) + ")");
    }
    int rc = run_walk(h, j);
    if (rc) return rc;
    const int64_t m = h->m_slab, n = h->n, k = std::min(m, n);
    CKL(launch_assemble(h->d_rows, (int32_t)m, h->d_cols, (int32_t)n, h->d_path, h->d_out,
                        h->d_out + 1, h->d_out + 1 + std::max<int64_t>(k, 1), h->d_subseq, h->stream));
    ++h->launches;
    std::vector<int32_t> hb((size_t)(1 + 2 * std::max<int64_t>(k, 1)));
    CK(cudaMemcpyAsync(hb.data(), h->d_out, hb.size() * 4, cudaMemcpyDeviceToHost, h->stream));
    std::vector<uint8_t> hs((size_t)std::max<int64_t>(k, 1));
    CK(cudaMemcpyAsync(hs.data(), h->d_subseq, hs.size(), cudaMemcpyDeviceToHost, h->stream));
    if (h->timing && h->ev_ok) CK(cudaEventRecord(h->ev[3], h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->d2h_bytes += (int64_t)(hb.size() * 4 + hs.size());
    const int32_t len = hb[0];
    *length = len;
    if (subseq) std::memcpy(subseq, hs.data(), (size_t)len);
    if (row_pos) std::memcpy(row_pos, hb.data() + 1, (size_t)len * 4);
    if (col_pos) std::memcpy(col_pos, hb.data() + 1 + std::max<int64_t>(k, 1), (size_t)len * 4);
    return LCSG_OK;
}

int lcsg_assemble(const uint8_t *rows, int64_t m, const uint8_t *cols, int64_t n,
                  const int32_t *path, int device, int32_t *length, uint8_t *subseq,
                  int32_t *row_pos, int32_t *col_pos) {
    if (!length) return fail(LCSG_EINVAL, "null length pointer");
    *length = 0;
    if (m == 0 || n == 0) return LCSG_OK;  // solver.py:219-220
    SaveDevice keep_caller_device;
    int rc = prepare_device(device);
    if (rc) return rc;
    const int64_t k = std::min(m, n);
    size_t bytes = align_up(m) + align_up(n) + align_up((m + 1) * 4) + align_up((1 + 2 * k) * 4) + align_up(k);
    char *buf = nullptr;
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaError_t e = pool_alloc((void **)&buf, bytes, device, s);
    if (e != cudaSuccess) {
        cudaStreamDestroy(s);
        return fail(LCSG_ENOMEM, cudaGetErrorString(e));
    }
    uint8_t *d_rows = (uint8_t *)buf;
    uint8_t *d_cols = (uint8_t *)(buf + align_up(m));
    int32_t *d_path = (int32_t *)(buf + align_up(m) + align_up(n));
    int32_t *d_out = (int32_t *)((char *)d_path + align_up((m + 1) * 4));
    uint8_t *d_sub = (uint8_t *)((char *)d_out + align_up((1 + 2 * k) * 4));
    std::vector<int32_t> hb((size_t)(1 + 2 * k));
    e = cudaMemcpyAsync(d_rows, rows, m, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_cols, cols, n, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_path, path, (m + 1) * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        int r = launch_assemble(d_rows, (int32_t)m, d_cols, (int32_t)n, d_path, d_out, d_out + 1,
                                d_out + 1 + k, d_sub, s);
        if (r) e = (cudaError_t)r;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(hb.data(), d_out, hb.size() * 4, cudaMemcpyDeviceToHost, s);
    std::vector<uint8_t> hs((size_t)k);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data(), d_sub, (size_t)k, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(buf, s);
    cudaError_t e2 = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    if (e == cudaSuccess) e = e2;
    if (e != cudaSuccess) return fail(LCSG_ECUDA, std::string("assemble: ") + cudaGetErrorString(e));
    *length = hb[0];
    if (subseq) std::memcpy(subseq, hs.data(), (size_t)hb[0]);
    if (row_pos) std::memcpy(row_pos, hb.data() + 1, (size_t)hb[0] * 4);
    if (col_pos) std::memcpy(col_pos, hb.data() + 1 + k, (size_t)hb[0] * 4);
    return LCSG_OK;
}

int lcsg_lcs(const uint8_t *a, int64_t la, const uint8_t *b, int64_t lb, uint32_t flags,
             int device, void *stream, int32_t *length, uint8_t *subseq, int32_t *pos_a,
             int32_t *pos_b) {
    return lcs_impl(a, la, b, lb, false, flags, device, stream, length, subseq, pos_a, pos_b);
}

int lcsg_lcs_device(const uint8_t *a_dev, int64_t la, const uint8_t *b_dev, int64_t lb,
                    uint32_t flags, int device, void *stream, int32_t *length, uint8_t *subseq,
                    int32_t *pos_a, int32_t *pos_b) {
    return lcs_impl(a_dev, la, b_dev, lb, true, flags, device, stream, length, subseq, pos_a, pos_b);
}

int lcsg_lcs_batch(const uint8_t *a, int64_t la, const uint8_t *b, int64_t lb, int32_t npairs,
                   uint32_t flags, int device, void *stream, int32_t *lengths, uint8_t *subseq,
                   int32_t *pos_a, int32_t *pos_b) {
    return lcs_impl(a, la, b, lb, false, flags, device, stream, lengths, subseq, pos_a, pos_b,
                    npairs);
}

int lcsg_lcs_batch_device(const uint8_t *a_dev, int64_t la, const uint8_t *b_dev, int64_t lb,
                          int32_t npairs, uint32_t flags, int device, void *stream,
                          int32_t *lengths, uint8_t *subseq, int32_t *pos_a, int32_t *pos_b) {
    return lcs_impl(a_dev, la, b_dev, lb, true, flags, device, stream, lengths, subseq, pos_a,
                    pos_b, npairs);
}

int lcsg_combine_level(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                       const int32_t *lower_reach, int32_t wl1, int32_t lower_wstar,
                       int32_t *out_reach, int32_t *out_trace, int32_t w1, int with_trace,
                       int32_t inf, int64_t n1, int64_t i_lo, int64_t i_hi, void *stream) {
    if (i_lo < 0 || i_hi > n1 || i_lo > i_hi) return fail(LCSG_EINVAL, "bad row range");
    if (i_hi == i_lo) return LCSG_OK;
    int dev = 0;
    int rc = current_device_prepared(&dev);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t rows = i_hi - i_lo;
    struct Scratch {
        CombineDesc d;
        int32_t wstar_l, wstar_out;
    };
    char *buf = nullptr;
    CK(pool_alloc((void **)&buf, sizeof(Scratch) + 256 + (size_t)rows * 4, dev, s));
    Scratch *sc = (Scratch *)buf;
    int32_t *kmax_scratch = (int32_t *)(buf + align_up(sizeof(Scratch)));
    Scratch hs;
    std::memset(&hs, 0, sizeof(hs));
    hs.d.U = TabDev{upper_reach + i_lo * wu1, upper_kmax + i_lo, nullptr, wu1, -1};
    hs.d.L = TabDev{lower_reach, nullptr, &sc->wstar_l, wl1, -1};
    hs.d.out_reach = out_reach + i_lo * w1;
    hs.d.out_trace = with_trace ? out_trace + i_lo * w1 : nullptr;
    hs.d.out_kmax = kmax_scratch;
    hs.d.out_wstar = &sc->wstar_out;
    hs.d.w1 = w1;
    hs.wstar_l = lower_wstar;
    CK(cudaMemcpyAsync(sc, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    Ctx c;
    c.rows = nullptr;
    c.nx = nullptr;
    c.n = (int32_t)(rows - 1);
    c.inf = inf;
    const int shift = bits_for(wu1 - 1);
    const bool key64 = need_key64(bits_for(inf), shift);
    CKL(launch_combine(w1 <= 65 ? 0 : 1, &sc->d, 1, c, shift, key64, s));
    CK(cudaFreeAsync(buf, s));
    CK(cudaStreamSynchronize(s));
    return LCSG_OK;
}

int lcsg_base_case_row(const uint8_t *cols_dev, int64_t n, uint8_t sym, int32_t *out_dev,
                       void *stream) {
    if (n <= 0) return LCSG_OK;
    CKL(launch_base_case_row(cols_dev, (int32_t)n, sym, out_dev, (cudaStream_t)stream));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    return LCSG_OK;
}

int lcsg_stats(lcsg_handle h, int64_t *launches, double *combine_ms, double *leaf_ms,
               double *total_ms, int64_t *h2d_bytes, int64_t *d2h_bytes) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    DeviceGuard g(h->device);
    if (launches) *launches = h->launches;
    float a = 0, b = 0, c = 0;
    if (h->timing && h->ev_ok) {
        CK(cudaStreamSynchronize(h->stream));
        cudaEventElapsedTime(&a, h->ev[1], h->ev[2]);
        cudaEventElapsedTime(&b, h->ev[0], h->ev[1]);
        if (cudaEventQuery(h->ev[3]) == cudaSuccess) cudaEventElapsedTime(&c, h->ev[0], h->ev[3]);
        cudaGetLastError();
    }
    if (combine_ms) *combine_ms = a;
    if (leaf_ms) *leaf_ms = b;
    if (total_ms) *total_ms = c;
    if (h2d_bytes) *h2d_bytes = h->h2d_bytes;
    if (d2h_bytes) *d2h_bytes = h->d2h_bytes;
    return LCSG_OK;
}

int lcsg_recover_from(lcsg_handle h, int32_t i_start, int32_t j, int32_t *cols_out) {
    if (!h) return fail(LCSG_EINVAL, "null handle");
    if (i_start < 1 || (int64_t)i_start > h->n + 1) return fail(LCSG_EINVAL, "start column out of range");
    if (j < 0) return fail(LCSG_EINVAL, "negative weight");
    DeviceGuard g(h->device);
    const NodeH &r = h->nodes[h->root];
    const int64_t n1 = h->n + 1;
    int32_t km = 0;
    if (r.upper < 0) {
        int32_t *p = nullptr;
        int rc = leaf_device(h, h->root, &p);
        if (rc) return rc;
        CK(cudaMemcpyAsync(&km, p + n1 * r.w1 + (i_start - 1), 4, cudaMemcpyDeviceToHost, h->stream));
    } else {
        CK(cudaMemcpyAsync(&km, h->d_tables + r.kmax_off + (i_start - 1), 4, cudaMemcpyDeviceToHost,
                           h->stream));
    }
    CK(cudaStreamSynchronize(h->stream));
    if (j > km)
        return fail(LCSG_ERANGE, "no path of weight " + std::to_string(j) + " from column " +
                                     std::to_string(i_start) + " (max " + std::to_string(km) + ")");
    int rc = run_walk(h, j, i_start);
    if (rc) return rc;
    CK(cudaMemcpyAsync(cols_out, h->d_path, (size_t)(h->m_slab + 1) * 4, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return LCSG_OK;
}

int lcsg_combine_rows(const int32_t *upper_reach, int32_t wu1, const int32_t *upper_kmax,
                      const int32_t *lower_reach, int32_t wl1, const int32_t *lower_kmax,
                      int32_t lower_wstar, int32_t *out_reach, int32_t *out_trace,
                      int32_t *out_kmax, int32_t *out_wstar, int32_t w1, int32_t inf, int64_t n1,
                      int64_t i_lo, int64_t i_hi, void *stream) {
    if (i_lo < 0 || i_hi > n1 || i_lo > i_hi) return fail(LCSG_EINVAL, "bad row range");
    if (!out_trace || !out_kmax || !out_wstar) return fail(LCSG_EINVAL, "null output buffer");
    const int64_t rows = i_hi - i_lo;
    if (rows == 0) return LCSG_OK;
    int dev = 0;
    int rc = current_device_prepared(&dev);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    struct Scratch {
        CombineDesc d;
        int32_t wstar_l;
    };
    // scratch after the descriptor: per-row events of the U window and of the
    // output, block flags (row sweep)
    const size_t ev_elems = (size_t)(rows + 63) / 64 * 64;
    const size_t flag_elems = (size_t)(rows / 2 + 64) / 32 * 32;
    const size_t sc_head = align_up(sizeof(Scratch));
    char *scbuf = nullptr;
    CK(pool_alloc((void **)&scbuf, sc_head + (2 * ev_elems + flag_elems) * 4, dev, s));
    Scratch *sc = (Scratch *)scbuf;
    int32_t *sc_ints = (int32_t *)(scbuf + sc_head);
    Scratch hs;
    std::memset(&hs, 0, sizeof(hs));
    // the row window [i_lo, i_hi) is addressed as a table of `rows` rows; L
    // keeps absolute rows (x = U[i,k] indexes it directly)
    hs.d.U = TabDev{upper_reach + i_lo * wu1, upper_kmax + i_lo, nullptr, wu1, -1};
    hs.d.L = TabDev{lower_reach, lower_kmax, &sc->wstar_l, wl1, -1};
    hs.d.out_reach = out_reach + i_lo * w1;
    hs.d.out_trace = out_trace + i_lo * w1;
    hs.d.out_kmax = out_kmax + i_lo;
    hs.d.out_wstar = out_wstar;
    hs.d.w1 = w1;
    hs.d.U_ev = sc_ints;
    hs.d.out_ev = sc_ints + ev_elems;
    hs.d.blk_flags = sc_ints + 2 * ev_elems;
    hs.d.U_ev_make = 1;
    hs.wstar_l = lower_wstar;
    CK(cudaMemcpyAsync(sc, &hs, sizeof(hs), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(sc_ints + 2 * ev_elems, 0, flag_elems * 4, s));
    Ctx c;
    c.rows = nullptr;
    c.nx = nullptr;
    c.n = (int32_t)(rows - 1);
    c.inf = inf;
    const int shift = bits_for(wu1 - 1);
    const bool key64 = need_key64(bits_for(inf), shift);
    const int thread_max_w1 = env_int("LCSG_THREAD_MAX_W1", 65);
    const bool sweep_on = env_int("LCSG_SWEEP", 1) != 0;
    int S = 1;
    while (S * 2 <= std::max(1, sweep_on ? env_int("LCSG_SWEEP_STRIDE", default_sweep_stride(n1))
                                         : env_int("LCSG_SKELETON_STRIDE", default_skeleton_stride(n1))))
        S *= 2;
    int col_block = 1;
    while (col_block * 2 <= std::min(16, std::max(2, env_int("LCSG_COL_BLOCK", default_col_block(n1)))))
        col_block *= 2;
    const int P = narrow_bucket(std::max(wu1, wl1) - 1);
    if (w1 <= thread_max_w1 && P > 0 && env_int("LCSG_NARROW", 1) != 0) {
        CKL(launch_narrow(&sc->d, 1, c, shift, key64, P, s));
    } else if (w1 <= thread_max_w1 || S == 1 || rows < 3 ||
               n1 * (int64_t)w1 >= ((int64_t)1 << 32)) {  // refinement: 32-bit offsets
        CKL(launch_combine(w1 <= 65 ? 0 : 1, &sc->d, 1, c, shift, key64, s));
    } else {
        if (w1 <= env_int("LCSG_SKEL_THREAD_MAX_W1", 65))
            CKL(launch_combine(0, &sc->d, 1, c, shift, key64, s, S));
        else if (w1 <= env_int("LCSG_SKEL_WARP_MAX_W1", 257))
            CKL(launch_combine(1, &sc->d, 1, c, shift, key64, s, S));
        else
            CKL(launch_skeleton(&sc->d, 1, c, shift, key64, S, s));
        if (sweep_on) {  // row sweep below the skeleton rows (lcsg_sweep.cu)
            CKL(launch_table_events(&sc->d, 1, c, s));
            CKL(launch_sweep(&sc->d, 1, c, shift, key64, S, w1, s));
        } else {
            for (int32_t rem = S; rem > 1;) {
                const int32_t B = std::min<int32_t>(col_block, rem);
                CKL(launch_block_refine(&sc->d, 1, c, shift, key64, B, rem / B, w1, s));
                rem /= B;
            }
        }
        CKL(launch_finalize_rows(&sc->d, 1, c, S, s, w1, sweep_on));
    }
    CK(cudaFreeAsync(scbuf, s));
    return LCSG_OK;
}

}  // extern "C"
