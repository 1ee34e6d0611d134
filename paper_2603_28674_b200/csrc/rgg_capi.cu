// rgg_capi.cu — host side of the C-ABI in include/rgg_gpu.h.
//
// Owns the device-resident store (cell-sorted SoA in HBM, resident across
// updates), the per-batch scratch, and the stream every kernel is launched on.
// No CPU fallback: creation fails with RGG_ECUDA unless an sm_100 device is
// present, and every compute entry launches the kernels of rgg_kernels.cu.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <atomic>
#include <cstring>
#include <chrono>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/rgg_gpu.h"
#include "rgg_kernels.cuh"

using rggk::Batch;
using rggk::Event;
using rggk::Store;

struct rgg_gpu {
    std::string err;
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    Store s{};
    // device allocations
    double2* d_aabb = nullptr;
    double* d_sat = nullptr;
    rggd::Box32* d_sat32 = nullptr;
    int32_t* d_row = nullptr;
    double* d_seg = nullptr;
    float4* d_seg32 = nullptr;
    double* d_spline = nullptr;
    int32_t* d_orig = nullptr;
    int32_t* d_rank = nullptr;
    double* d_cell_aabb = nullptr;
    double* d_slice_aabb = nullptr;
    rggk::CellGrid grid{};   // the binning's uniform grid over the cell boxes
    uint32_t* d_cmask = nullptr;  // Batch::cmask (ncells x cmask_words)
    int32_t cmask_words = 0;
    double* d_evbox = nullptr;
    double* d_evt = nullptr;
    float4* d_evs = nullptr;
    int4* d_units = nullptr;
    int32_t* d_unit_ready = nullptr;  // Batch::unit_ready: units_cap generation stamps
    int32_t units_cap = 0;
    double* d_ohe = nullptr;
    double* d_osl = nullptr;
    double* d_osr = nullptr;
    int32_t* d_osn = nullptr;
    uint8_t* d_state = nullptr;
    uint8_t* d_state_c = nullptr;  // cell-order copy of the owned labels (Store::state_c)
    uint32_t* d_cnt = nullptr;
    unsigned long long* d_over = nullptr;
    unsigned long long* d_under = nullptr;
    Event* d_cur = nullptr;
    double* d_cur_union = nullptr;
    int32_t* d_ctr = nullptr;
    unsigned long long* d_census = nullptr;
    int32_t* d_gray = nullptr;
    int32_t* d_tiles = nullptr;
    int32_t* d_hits = nullptr;
    uint8_t* d_hits_prev = nullptr;
    // exact resolve (rgg_resolve.cu): per-configuration body poses, obstacle polytopes
    bool res_ready = false;
    int32_t res_B = 0;
    double* d_res_he = nullptr;
    long long* d_res_off = nullptr;
    double* d_res_pose = nullptr;
    rggk::ObsPoly* d_opoly = nullptr;
    double* d_res_spose = nullptr;  // M*12 scene poses of pre-active obstacles
    uint8_t* d_res_sact = nullptr;  // M
    int32_t* d_res_ids = nullptr;  // N: scratch id list (rgg_gpu_exact_check)
    int32_t* d_res_cnt = nullptr;
    uint8_t* d_res_out = nullptr;  // N
    // eager batches: staged moves and per-move report slots (8 ints each)
    int32_t eager_cap = 0;
    int32_t* d_eg_ids = nullptr;
    double* d_eg_rt = nullptr;
    int32_t* d_eg_rep = nullptr;
    int32_t* h_eg_rep = nullptr;
    int32_t* d_cell_count = nullptr;
    int32_t* d_cell_list = nullptr;
    int32_t* d_cell_ovf = nullptr;
    int4* d_crec = nullptr;
    long long* d_mtop = nullptr;
    // batch buffers (grown on demand)
    int32_t cap_moves = 0;
    int32_t* d_ids = nullptr;
    double* d_rt = nullptr;
    size_t in_off = 0;
    uint8_t* d_last = nullptr;
    int32_t* d_unknown = nullptr;
    cudaEvent_t done_ev = nullptr;        // stream_wait
    int32_t* d_evready = nullptr;         // Batch::evready[8] (split pipeline)
    unsigned long long* d_tl = nullptr;  // RGG_DEBUG_TIMELINE: 16 x 8 words (rgg_kernels.cu tl_stop)
    Event* d_ev = nullptr;
    int32_t* d_mv = nullptr;
    int32_t* d_pool = nullptr;
    int64_t pool_cap = 0;
    uint32_t* d_mpool = nullptr;
    int64_t mpool_cap = 0;
    int4* d_items_over = nullptr;
    int4* d_items_under = nullptr;
    int32_t items_cap = 0;
    int4* d_items_recheck = nullptr;  // Batch::items_recheck (rggk::kRecheckCap entries)
    int32_t recheck_cap = 0;
    int32_t recheck_min_moves = 0;  // batches of at least this many moves queue the undecided SAT pairs
    // pinned staging
    int32_t cap_pin = 0;
    int32_t* h_ids = nullptr;
    double* h_rt = nullptr;
    size_t pin_off = 0;
    int32_t* h_mv = nullptr;   // mapped pinned (device view dh_mv)
    int32_t* h_ctr = nullptr;  // mapped pinned (device view dh_ctr)
    int32_t* dh_mv = nullptr;
    int32_t* dh_ids = nullptr;  // device view of the mapped move staging (h_ids, then h_rt at pin_off)
    int32_t* dh_ctr = nullptr;
    // host mirrors
    std::vector<int32_t> orig;  // sorted -> id (owned)
    int32_t words = 1;
    int32_t last_n = 0;
    int32_t last_flags = 0;
    bool last_single = false;  // the last update took the single-move path (no cell lists)
    bool last_hits_valid = false;
    int32_t unknown = 0;
    bool unknown_stale = false;
    cudaEvent_t ev[6] = {};
    // CUDA graphs of the update pipeline, keyed by (moves, kernel flags, buffer generation)
    struct GraphEntry {
        int32_t n, kf, gen;
        cudaGraphExec_t exec;
    };
    std::vector<GraphEntry> graphs;
    int32_t gen = 0;
    bool phase_timing = false;  // per-kernel phase events (rgg_gpu_set_phase_timing)
    bool gray_fresh = true;    // d_gray holds the ids of the current labels
    bool timed = false;
    int grid_classify = 1;
    int64_t total_segs_owned = 0;
    bool poisoned = false;  // a failed eager batch left a partial state (rgg_gpu_update fails from then on)
    int32_t* h_gray = nullptr;  // pinned host copy of the gray list (rgg_gpu_gray_view)
    int32_t gray_pin_cap = 0;
    // mapped pinned gray list (capacity N) that a synchronous host update with RGG_GRAY_LIST
    // writes inside the update; gray_host_fresh: it holds the current labels' list
    int32_t* h_gray_map = nullptr;
    int32_t* dh_gray_map = nullptr;
    bool gray_host_fresh = false;
};

namespace {

int fail(rgg_gpu* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

// Entry points first drop any stale non-sticky error left by an earlier runtime
// call, so a launcher's cudaGetLastError() reports its own launch only.
inline void clear_stale_error() { (void)cudaGetLastError(); }

#define CK(expr)                                                                                 \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess) return fail(h, RGG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Wait for the handle's stream by polling an event: cudaStreamSynchronize costs about
// 11 us of wake-up per call on the B200 boxes, a poll about 1 us.
cudaError_t stream_wait(rgg_gpu* h) {
    if (!h->done_ev) {
        const cudaError_t e = cudaEventCreateWithFlags(&h->done_ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaEventRecord(h->done_ev, h->stream);
    if (e != cudaSuccess) return e;
    while ((e = cudaEventQuery(h->done_ev)) == cudaErrorNotReady) {
    }
    return e;
}

template <class T>
cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(1, n) * sizeof(T));
}

int grow_batch(rgg_gpu* h, int32_t n) {
    if (n <= h->cap_moves && static_cast<int64_t>(h->s.ncells) * n <= h->pool_cap) return RGG_OK;
    const int32_t cap = std::max(n, std::max(64, h->cap_moves * 2));
    cudaFree(h->d_ids);  // ids and poses share one allocation (d_rt points into it)
    cudaFree(h->d_last);
    cudaFree(h->d_ev);
    cudaFree(h->d_evbox);
    cudaFree(h->d_evt);
    cudaFree(h->d_evs);
    cudaFree(h->d_units);
    cudaFree(h->d_unit_ready);
    cudaFree(h->d_mv);
    cudaFree(h->d_pool);
    cudaFree(h->d_mpool);
    cudaFree(h->d_cmask);
    // moves: ids then poses in one block, so the host path needs a single H2D copy
    h->in_off = ((static_cast<size_t>(cap) * 4 + 15) / 16) * 16;
    CK(dalloc(reinterpret_cast<char**>(&h->d_ids), h->in_off + static_cast<size_t>(cap) * 96));
    h->d_rt = reinterpret_cast<double*>(reinterpret_cast<char*>(h->d_ids) + h->in_off);
    CK(dalloc(&h->d_last, cap));
    CK(dalloc(&h->d_ev, cap));
    CK(dalloc(&h->d_evbox, static_cast<size_t>(cap) * 12));
    CK(dalloc(&h->d_evt, static_cast<size_t>(cap) * 24));
    CK(dalloc(&h->d_evs, static_cast<size_t>(cap) * rggk::kEvS));
    // touch work units: at most ceil(cap / 32) chunks per cell
    const int64_t units = std::max<int64_t>(1, static_cast<int64_t>(h->s.ncells) * ((cap + 31) / 32));
    if (units > INT32_MAX) return fail(h, RGG_ENOMEM, "batch too large for the touch work list; split it");
    h->units_cap = static_cast<int32_t>(units);
    CK(dalloc(&h->d_units, static_cast<size_t>(units)));
    CK(dalloc(&h->d_unit_ready, static_cast<size_t>(units)));
    CK(cudaMemsetAsync(h->d_unit_ready, 0, static_cast<size_t>(units) * sizeof(int32_t), h->stream));
    CK(dalloc(&h->d_mv, static_cast<size_t>(cap) * 4));
    // every (cell, event) pair fits: the overflow pool can never run out
    h->pool_cap = std::max<int64_t>(1, static_cast<int64_t>(h->s.ncells) * cap);
    CK(dalloc(&h->d_pool, static_cast<size_t>(h->pool_cap)));
    // mask words of the touch / narrow / apply kernels: 3 * ceil(L/32) per component of a listed cell
    h->mpool_cap = std::max<int64_t>(1, 3ll * h->s.ncells * h->s.cell * ((cap + 31) / 32));
    if (h->mpool_cap > INT32_MAX) return fail(h, RGG_ENOMEM, "batch too large for the mask pool; split it");
    CK(dalloc(&h->d_mpool, static_cast<size_t>(h->mpool_cap)));
    // event bitmask per cell (binning); zero between updates
    h->cmask_words = (cap + 31) / 32;
    const size_t cm = std::max<size_t>(1, static_cast<size_t>(h->s.ncells) * h->cmask_words);
    CK(dalloc(&h->d_cmask, cm));
    CK(cudaMemsetAsync(h->d_cmask, 0, cm * sizeof(uint32_t), h->stream));
    h->cap_moves = cap;
    ++h->gen;  // buffers moved: captured graphs are stale
    return RGG_OK;
}

int grow_items(rgg_gpu* h, int64_t need) {
    const int64_t cap = std::min<int64_t>(INT32_MAX / 2, std::max<int64_t>(2 * need, h->items_cap));
    if (cap <= h->items_cap) return fail(h, RGG_ENOMEM, "narrow item queue cannot grow further; split the batch");
    cudaFree(h->d_items_over);
    cudaFree(h->d_items_under);
    h->d_items_over = nullptr;
    h->d_items_under = nullptr;
    CK(dalloc(&h->d_items_over, static_cast<size_t>(cap)));
    CK(dalloc(&h->d_items_under, static_cast<size_t>(cap)));
    h->items_cap = static_cast<int32_t>(cap);
    ++h->gen;  // captured graphs hold the old queue pointers
    return RGG_OK;
}

int grow_pinned(rgg_gpu* h, int32_t n) {
    if (n <= h->cap_pin) return RGG_OK;
    const int32_t cap = std::max(n, std::max(64, h->cap_pin * 2));
    cudaFreeHost(h->h_ids);
    cudaFreeHost(h->h_mv);
    h->pin_off = ((static_cast<size_t>(cap) * 4 + 15) / 16) * 16;
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_ids), h->pin_off + static_cast<size_t>(cap) * 96,
                     cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_ids), h->h_ids, 0));
    h->h_rt = reinterpret_cast<double*>(reinterpret_cast<char*>(h->h_ids) + h->pin_off);
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_mv), cap * 4 * sizeof(int32_t), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_mv), h->h_mv, 0));
    h->cap_pin = cap;
    ++h->gen;  // graphs with host copies hold the old staging pointers
    return RGG_OK;
}

Batch batch_of(rgg_gpu* h, int32_t n) {
    Batch b{};
    b.n = n;
    b.ids = h->d_ids;
    b.rt = h->d_rt;
    b.last = h->d_last;
    b.ev = h->d_ev;
    b.evbox = h->d_evbox;
    b.evt = h->d_evt;
    b.evs = h->d_evs;
    b.units = h->d_units;
    b.units_cap = h->units_cap;
    b.cell_count = h->d_cell_count;
    b.cell_list = h->d_cell_list;
    b.cell_ovf = h->d_cell_ovf;
    b.pool = h->d_pool;
    b.pool_cap = static_cast<int32_t>(std::min<int64_t>(h->pool_cap, INT32_MAX));
    b.ctr = h->d_ctr;
    b.mv = h->d_mv;
    b.hits = h->d_hits;
    b.hits_prev = h->d_hits_prev;
    b.census = h->d_census;
    b.unknown = h->d_unknown;
    b.mpool = h->d_mpool;
    b.mtop = h->d_mtop;
    b.mpool_cap = h->mpool_cap;
    b.crec = h->d_crec;
    b.items_over = h->d_items_over;
    b.items_under = h->d_items_under;
    b.items_cap = h->items_cap;
    b.items_recheck = h->d_items_recheck;
    b.recheck_cap = h->recheck_cap;
    b.recheck_queue = n >= h->recheck_min_moves;
    static const bool timeline = std::getenv("RGG_DEBUG_TIMELINE") != nullptr;
    if (timeline && !h->d_tl) cudaMalloc(reinterpret_cast<void**>(&h->d_tl), 128 * 8);
    b.tl = h->d_tl;
    if (!h->d_evready) {
        cudaMalloc(reinterpret_cast<void**>(&h->d_evready), 8 * sizeof(int32_t));
        cudaMemsetAsync(h->d_evready, 0, 8 * sizeof(int32_t), h->stream);
    }
    static const bool no_early_bin = std::getenv("RGG_NO_EARLY_BIN") != nullptr;  // tests: the plain PDL waits
    b.evready = no_early_bin ? nullptr : h->d_evready;
    // touch on published units (RGG_EARLY_TOUCH_MIN moves and more; off by default): its
    // warps take slice-units with a same-address atomic and poll the units' stamps, which
    // costs more than the overlap saves once the binning is short
    static const int early_touch_min = [] {
        const char* e = std::getenv("RGG_EARLY_TOUCH_MIN");
        return e ? std::atoi(e) : 1 << 30;
    }();
    b.unit_ready = b.evready && n >= early_touch_min ? h->d_unit_ready : nullptr;
    b.bin_warps = h->s.ncells;  // one counted warp per cell, whichever bin kernel runs
    b.cmask = h->d_cmask;
    b.cmask_words = h->cmask_words;
    return b;
}

// RGG_DEBUG_TIMELINE: one stderr line per update, microseconds from the first
// pose warp: per kernel first start / last start / first end / last end / mean
// warp duration, then each PDL kernel's earliest arrival before its wait.
void dump_timeline(rgg_gpu* h) {
    if (!h->d_tl) return;
    unsigned long long t[128];
    if (cudaMemcpy(t, h->d_tl, sizeof(t), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    const double z = static_cast<double>(~t[0]);
    const auto us = [&](unsigned long long v) { return (static_cast<double>(v) - z) * 1e-3; };
    static const char* name[10] = {"pose", "bin", "touch", "narrow", "apply", "", "", "", "", "scatter"};
    std::fprintf(stderr, "[tl]");
    for (int k = 0; k < 10; ++k) {
        if (k >= 5 && k < 9) continue;
        const unsigned long long* p = t + 8 * k;
        if (!p[5]) continue;
        std::fprintf(stderr, " %s %.1f %.1f %.1f %.1f %.2f |", name[k], us(~p[0]), us(p[1]), us(~p[2]), us(p[3]),
                     p[4] * 1e-3 / p[5]);
    }
    std::fprintf(stderr, " arrive");
    for (int k : {5, 10, 6, 7, 8})
        if (t[8 * k + 5]) std::fprintf(stderr, " %.1f", us(~t[8 * k]));
    std::fprintf(stderr, "\n");
}

// Narrow items pack the event index with a 5-bit position (rgg_kernels.cu).
constexpr int32_t kMaxBatch = 1 << 26;
// internal enqueue flag: host copies inside the update's graph
constexpr int32_t kHostIO = 1 << 20;
// host updates of at most this many moves read them from mapped memory in the pose kernel
constexpr int32_t kMappedMovesMax = 128;

bool graphs_enabled(const rgg_gpu* h) {
    static const bool off = std::getenv("RGG_DEBUG_PHASES") || std::getenv("RGG_NO_GRAPH");
    return !off;
}

rggk::Resolver resolver_of(rgg_gpu* h) {
    rggk::Resolver r{};
    r.B = h->res_B;
    r.he = h->d_res_he;
    r.off = h->d_res_off;
    r.pose = h->d_res_pose;
    r.opoly = h->d_opoly;
    r.spose = h->d_res_spose;
    r.sact = h->d_res_sact;
    return r;
}

// grid bound of the eager resolve (a move's gray over-hits; the kernel strides)
constexpr int kEagerResolveGrid = 592;  // 4 x 148 SMs: one CTA per gray over-hit, strided beyond

// Enqueue the whole pipeline for n moves already in d_ids/d_rt.
int enqueue(rgg_gpu* h, int32_t n, int32_t flags) {
    Batch b = batch_of(h, n);
    b.census_on = (flags & RGG_CENSUS) ? 1 : 0;
    int kf = 0;
    if (flags & RGG_PER_MOVE) kf |= rggk::kPerMove;
    if (n == 1) kf |= rggk::kHits;
    // single moves (update_obstacle, eager): dirty cells straight from the move's boxes and
    // one fused touch + narrow + transition kernel (rggk::launch_single); the census keeps
    // the batched path, whose cell lists and item queues it counts
    static const bool no_single = std::getenv("RGG_NO_SINGLE") != nullptr;
    const bool single = n == 1 && !b.census_on && !no_single;
    if (single) {  // no bin kernel waits on the pose warps' published boxes
        b.evready = nullptr;
        b.unit_ready = nullptr;
    }
    const auto classify = [&]() {
        return single ? rggk::launch_single(h->s, b, kf, h->stream)
                      : rggk::launch_classify(h->s, b, kf, h->grid_classify, h->stream);
    };
    static const bool debug = std::getenv("RGG_DEBUG_PHASES") != nullptr;
    auto phase = [&](const char* name) -> int {
        if (!debug) return RGG_OK;
        CK(stream_wait(h));
        std::fprintf(stderr, "[rgg] %s done\n", name);
        return RGG_OK;
    };
    static const bool no_graph = std::getenv("RGG_NO_GRAPH") != nullptr;
    const bool use_graph = !debug && !no_graph;
    const bool phases = h->phase_timing;
    // the gray id list is compacted in the update only on request; otherwise lazily
    // by rgg_gpu_gray_ids (labels, reports and the gray count never need it)
    const bool gray_list = (flags & RGG_GRAY_LIST) != 0;
    const bool eager = (flags & RGG_EAGER) != 0;  // n == 1: resolve the move's gray over-hits
    // kHostIO (rgg_gpu_update): the moves' H2D copy and the counters' D2H copies are
    // nodes of the graph, so a synchronous update is one graph launch and one wait
    const bool hostio = use_graph && (flags & kHostIO) != 0;
    // synchronous host updates end with one small kernel that stores the counters into
    // mapped host memory and raises the flag the host polls: after apply, or after the
    // gray-list compaction when the update compacts it (eager updates copy them instead)
    const bool out_in_kernel = hostio && !eager;
    if (out_in_kernel) {
        b.out_mv = h->dh_mv;
        b.out_ctr = h->dh_ctr;
    }
    // small batches: the pose kernel reads the moves straight from the mapped staging
    // buffer (no copy node); large ones (a 1024-move batch is 100 KB, read by every pose
    // warp over PCIe) get one H2D copy node into HBM before the pose kernel
    const bool mapped_moves = hostio && n <= kMappedMovesMax;
    // the gray list of a synchronous host update goes straight to mapped host memory
    const bool gray_host = hostio && gray_list && h->s.N > 0;
    if (gray_host && !h->h_gray_map) {
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_gray_map), static_cast<size_t>(h->s.N) * sizeof(int32_t),
                         cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_gray_map), h->h_gray_map, 0));
    }
    if (mapped_moves) {
        b.src_ids = h->dh_ids;
        b.src_rt = reinterpret_cast<const double*>(reinterpret_cast<const char*>(h->dh_ids) + h->pin_off);
    }
    const int32_t key = kf | (b.census_on ? 64 : 0) | (phases ? 128 : 0) | (gray_list ? 256 : 0) | (eager ? 512 : 0) |
                        (hostio ? 1024 : 0) | ((flags & RGG_PER_MOVE) && hostio ? 2048 : 0);
    const auto resolve_hits = [&]() {
        return rggk::launch_resolve(h->s, resolver_of(h), b, h->d_hits, h->d_ctr + 5, kEagerResolveGrid, rggk::kEager,
                                    nullptr, h->stream);
    };
    if (use_graph) {
        cudaGraphExec_t exec = nullptr;
        for (const auto& g : h->graphs)
            if (g.n == n && g.kf == key && g.gen == h->gen) exec = g.exec;
        if (!exec) {
            // capture the launch sequence once (pose, bin, classify, compaction + phase events)
            // phase events become event-record nodes (cudaEventRecordExternal), so they time the replay
            // inner phase events break the programmatic (PDL) edges between kernels, so they are
            // recorded only when phase timing is on; ev[0] / ev[4] always bracket the update
            const auto rec = [&](cudaEvent_t ev) {
                if (!phases && ev != h->ev[0] && ev != h->ev[4]) return cudaSuccess;
                return cudaEventRecordWithFlags(ev, h->stream, cudaEventRecordExternal);
            };
            CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
            cudaError_t e = rec(h->ev[0]);
            if (e == cudaSuccess && hostio && !mapped_moves)
                e = cudaMemcpyAsync(h->d_ids, h->h_ids, h->in_off + static_cast<size_t>(n) * 96, cudaMemcpyHostToDevice,
                                    h->stream);
            if (e == cudaSuccess) e = rggk::launch_pose(h->s, b, h->stream);
            if (e == cudaSuccess) e = rec(h->ev[1]);
            if (e == cudaSuccess && !single) e = rggk::launch_bin(h->s, b, h->stream);
            if (e == cudaSuccess) e = rec(h->ev[2]);
            if (e == cudaSuccess) e = classify();
            if (e == cudaSuccess && out_in_kernel && !gray_list) e = rggk::launch_host_out(b, h->stream);
            if (e == cudaSuccess && eager) e = resolve_hits();
            if (e == cudaSuccess) e = rec(h->ev[3]);
            if (e == cudaSuccess && gray_list)
                e = rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream,
                                         gray_host ? h->dh_gray_map : nullptr);
            if (e == cudaSuccess && out_in_kernel && gray_list) e = rggk::launch_host_out(b, h->stream);
            if (e == cudaSuccess) e = rec(h->ev[4]);
            if (e == cudaSuccess && hostio && !out_in_kernel && (flags & RGG_PER_MOVE))
                e = cudaMemcpyAsync(h->h_mv, h->d_mv, static_cast<size_t>(n) * 4 * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, h->stream);
            if (e == cudaSuccess && hostio && !out_in_kernel)
                e = cudaMemcpyAsync(h->h_ctr, h->d_ctr, 24 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream);
            cudaGraph_t graph = nullptr;
            const cudaError_t e2 = cudaStreamEndCapture(h->stream, &graph);
            CK(e);
            CK(e2);
            CK(cudaGraphInstantiate(&exec, graph, 0));
            cudaGraphDestroy(graph);
            h->graphs.push_back({n, key, h->gen, exec});
        }
        if (h->d_tl) CK(cudaMemsetAsync(h->d_tl, 0, 128 * 8, h->stream));
        CK(cudaGraphLaunch(exec, h->stream));
        h->gray_fresh = gray_list;
        h->gray_host_fresh = gray_host;
        h->last_n = n;
        h->last_flags = flags;
        h->last_single = single;
        h->last_hits_valid = n == 1 && !eager;
        h->timed = true;
        h->unknown_stale = true;
        return RGG_OK;
    }
    CK(cudaEventRecord(h->ev[0], h->stream));
    CK(rggk::launch_pose(h->s, b, h->stream));
    if (phase("pose")) return RGG_ECUDA;
    CK(cudaEventRecord(h->ev[1], h->stream));
    if (!single) CK(rggk::launch_bin(h->s, b, h->stream));
    if (phase("bin")) return RGG_ECUDA;
    CK(cudaEventRecord(h->ev[2], h->stream));
    CK(classify());
    if (phase("classify")) return RGG_ECUDA;
    if (eager) CK(resolve_hits());
    CK(cudaEventRecord(h->ev[3], h->stream));
    if (gray_list) CK(rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream));
    CK(cudaEventRecord(h->ev[4], h->stream));
    h->gray_fresh = gray_list;
    h->gray_host_fresh = false;
    h->last_n = n;
    h->last_flags = flags;
    h->last_single = single;
    h->last_hits_valid = n == 1 && !eager;
    h->timed = true;
    h->unknown_stale = true;
    return RGG_OK;
}

int refresh_unknown(rgg_gpu* h) {
    if (!h->unknown_stale) return RGG_OK;
    int32_t v = 0;
    CK(cudaMemcpyAsync(&v, h->d_unknown, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    h->unknown = v;
    h->unknown_stale = false;
    return RGG_OK;
}

}  // namespace

extern "C" {

const char* rgg_gpu_last_error(const rgg_gpu* h) { return h ? h->err.c_str() : "null handle"; }

}  // extern "C"

namespace {
// Device-resident inputs of rgg_gpu_create_from_components (sat_prep / seg_prep done on
// the device); null: the view's host arrays are uploaded.
struct DeviceInputs {
    const double* comp_aabb = nullptr;
    const double* edge_sat = nullptr;
    const double* segs = nullptr;
    const int32_t* row_off = nullptr;
};
int create_impl(rgg_gpu* h, const rgg_layout_view* v, const rgg_gpu_options* opts, const DeviceInputs* dev);
}  // namespace

extern "C" int rgg_gpu_create(const rgg_layout_view* v, const rgg_gpu_options* opts, rgg_gpu** out) {
    if (!out) return RGG_EINVAL;
    *out = nullptr;
    rgg_gpu* h = new rgg_gpu();
    *out = h;
    if (!v) return fail(h, RGG_EINVAL, "null layout view");
    return create_impl(h, v, opts, nullptr);
}

extern "C" int rgg_gpu_create_from_components(const rgg_component_view* cv, const rgg_gpu_options* opts,
                                              rgg_gpu** out) {
    if (!out) return RGG_EINVAL;
    *out = nullptr;
    rgg_gpu* h = new rgg_gpu();
    *out = h;
    if (!cv) return fail(h, RGG_EINVAL, "null component view");
    const int32_t N = cv->n_components, B = cv->n_bodies, S = cv->n_slots;
    if (N < 0 || B < 1 || S < 1) return fail(h, RGG_EINVAL, "malformed component view");
    if (!cv->row_off || !cv->spline_radius || (N > 0 && !cv->obb_corners) ||
        (cv->n_obstacles > 0 && (!cv->obst_he || !cv->obst_sph_r || !cv->obst_sph_n)))
        return fail(h, RGG_EINVAL, "null array in the component view");
    const int64_t nrows = static_cast<int64_t>(N) * B * S;
    if (cv->row_off[0] != 0) return fail(h, RGG_ELOGIC, "row_off must start at 0");
    for (int64_t r = 0; r < nrows; ++r)
        if (cv->row_off[r + 1] < cv->row_off[r]) return fail(h, RGG_ELOGIC, "row_off must be non-decreasing");
    const int64_t T = cv->row_off[nrows];
    if (T > INT32_MAX) return fail(h, RGG_ELOGIC, "too many segments");
    if (T > 0 && !cv->seg_points) return fail(h, RGG_EINVAL, "null array in the component view");
    rgg_gpu_options o{};
    if (opts) o = *opts;
    clear_stale_error();
    CK(cudaSetDevice(o.device));
    // upload the raw geometry, then sat_prep / AABBs / seg_prep on the device
    struct Bufs {
        std::vector<void*> p;
        ~Bufs() {
            for (void* q : p) cudaFree(q);
        }
    } bufs;
    const auto take = [&](auto** q, size_t n) {
        const cudaError_t e = dalloc(q, n);
        if (e == cudaSuccess) bufs.p.push_back(*q);
        return e;
    };
    double *d_corners, *d_pts, *d_aabb, *d_sat, *d_segs;
    int32_t* d_row;
    CK(take(&d_corners, static_cast<size_t>(N) * B * 24));
    CK(take(&d_pts, static_cast<size_t>(T) * 6));
    CK(take(&d_aabb, static_cast<size_t>(N) * 6));
    CK(take(&d_sat, static_cast<size_t>(N) * B * 21));
    CK(take(&d_segs, static_cast<size_t>(T) * 7));
    CK(take(&d_row, static_cast<size_t>(nrows) + 1));
    CK(cudaMemcpy(d_corners, cv->obb_corners, static_cast<size_t>(N) * B * 24 * 8, cudaMemcpyHostToDevice));
    if (T) CK(cudaMemcpy(d_pts, cv->seg_points, static_cast<size_t>(T) * 6 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_row, cv->row_off, (static_cast<size_t>(nrows) + 1) * 4, cudaMemcpyHostToDevice));
    CK(rggk::prep_components(d_corners, N, B, d_pts, static_cast<int>(T), d_sat, d_aabb, d_segs, nullptr));
    CK(cudaDeviceSynchronize());
    rgg_layout_view v{N, B, S, cv->n_obstacles, cv->max_spheres, nullptr, nullptr, cv->row_off, nullptr,
                      cv->spline_radius, cv->obst_he, cv->obst_sph_local, cv->obst_sph_r, cv->obst_sph_n};
    const DeviceInputs dev{d_aabb, d_sat, d_segs, d_row};
    return create_impl(h, &v, opts, &dev);
}

namespace {
int create_impl(rgg_gpu* h, const rgg_layout_view* v, const rgg_gpu_options* opts, const DeviceInputs* dev) {
    rgg_gpu_options o{};
    if (opts) o = *opts;
    const int32_t N = v->n_components, B = v->n_bodies, S = v->n_slots, M = v->n_obstacles, C = v->max_spheres;
    if (N < 0 || B < 1 || S < 1 || M < 0 || C < 0) return fail(h, RGG_EINVAL, "malformed layout view");
    if (!v->row_off || !v->spline_radius || (!dev && N > 0 && (!v->edge_sat || !v->comp_aabb)) ||
        (M > 0 && (!v->obst_he || !v->obst_sph_r || !v->obst_sph_n || (C > 0 && !v->obst_sph_local))))
        return fail(h, RGG_EINVAL, "null array in the layout view");
    if (M > 64 && !o.allow_wide) return fail(h, RGG_EINVAL, "obstacle bitsets support at most 64 obstacles");
    if (C > rggk::kMaxSpheres) return fail(h, RGG_EINVAL, "too many spheres per obstacle (max 16)");
    if (M > 0xfffe) return fail(h, RGG_EINVAL, "too many obstacles");
    static const int cell_default = [] {  // RGG_CELL_SIZE: experiments only
        const char* e = std::getenv("RGG_CELL_SIZE");
        return e ? std::atoi(e) : 128;
    }();
    const int cell = o.cell_size > 0 ? o.cell_size : cell_default;
    if (cell % 32 != 0 || cell > rggk::kMaxCell) return fail(h, RGG_EINVAL, "cell_size must be a multiple of 32, <= 128");
    const int cap = o.cell_capacity > 0 ? o.cell_capacity : 64;
    const int shards = o.shard_count > 1 ? o.shard_count : 1;
    const int rank = shards > 1 ? o.shard_rank : 0;
    if (rank < 0 || rank >= shards) return fail(h, RGG_EINVAL, "shard_rank out of range");
    for (int32_t i = 0; i < M; ++i)
        if (v->obst_sph_n[i] < 0 || v->obst_sph_n[i] > C) return fail(h, RGG_EINVAL, "bad obstacle sphere count");
    const int64_t nrows = static_cast<int64_t>(N) * B * S;
    if (v->row_off[0] != 0) return fail(h, RGG_ELOGIC, "row_off must start at 0");
    for (int64_t r = 0; r < nrows; ++r)
        if (v->row_off[r + 1] < v->row_off[r]) return fail(h, RGG_ELOGIC, "row_off must be non-decreasing");

    h->device = o.device;
    static const bool dbg_create = std::getenv("RGG_DEBUG_CREATE") != nullptr;
    auto t_create = std::chrono::steady_clock::now();
    const auto mark = [&](const char* what) {
        if (!dbg_create) return;
        cudaDeviceSynchronize();
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[rgg create] %-12s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(t - t_create).count());
        t_create = t;
    };
    clear_stale_error();
    CK(cudaSetDevice(h->device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, h->device));
    if (prop.major != 10) return fail(h, RGG_ECUDA, std::string("needs an sm_100 (B200) device, found ") + prop.name);
    h->sms = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
    mark("context");

    // ---- the cell-sorted store, built on the device (rgg_store.cu): Morton order of
    // the AABB centres, shard = interleaved cells of that order, SoA gathers
    const int64_t gcells = (static_cast<int64_t>(N) + cell - 1) / cell;
    int64_t np64 = 0;
    for (int64_t g = rank; g < gcells; g += shards) np64 += std::min<int64_t>(cell, N - g * cell);
    const int32_t Np = static_cast<int32_t>(np64);
    const int32_t ncells = (Np + cell - 1) / cell;
    h->words = M <= 64 ? 1 : (M + 63) / 64;
    const int64_t T = v->row_off[nrows];
    if (T > INT32_MAX) return fail(h, RGG_ELOGIC, "too many segments");
    if (!dev && T > 0 && !v->segs) return fail(h, RGG_EINVAL, "null array in the layout view");
    CK(dalloc(&h->d_aabb, static_cast<size_t>(Np) * 3));
    CK(dalloc(&h->d_sat, static_cast<size_t>(Np) * B * 22));
    CK(dalloc(&h->d_sat32, static_cast<size_t>(Np) * B));
    CK(dalloc(&h->d_row, static_cast<size_t>(Np) * B * S + 1));
    CK(dalloc(&h->d_spline, static_cast<size_t>(B) * S));
    CK(dalloc(&h->d_orig, Np));
    CK(dalloc(&h->d_rank, N));
    CK(dalloc(&h->d_cell_aabb, static_cast<size_t>(std::max(ncells, 1)) * 6));
    CK(dalloc(&h->d_slice_aabb, static_cast<size_t>(std::max((Np + 31) / 32, 1)) * 6));
    {
        rggk::StoreIn in{N, B, S, static_cast<int32_t>(T), Np, cell, shards, rank,
                         v->comp_aabb, v->edge_sat, v->row_off, v->segs, v->spline_radius};
        if (dev) {
            in.comp_aabb = dev->comp_aabb, in.edge_sat = dev->edge_sat, in.segs = dev->segs;
            in.device = true;
            in.row_off_dev = dev->row_off;
        }
        rggk::StoreOut so{};
        so.aabb = h->d_aabb, so.sat = h->d_sat, so.sat32 = h->d_sat32, so.row = h->d_row, so.spline = h->d_spline;
        so.orig = h->d_orig, so.rank = h->d_rank, so.cell_aabb = h->d_cell_aabb, so.slice_aabb = h->d_slice_aabb;
        mark("allocs");
        CK(rggk::build_store(in, so, h->stream));
        mark("build_store");
        h->d_seg = so.seg;
        h->d_seg32 = so.seg32;
        h->total_segs_owned = so.total_segs;
        CK(rggk::build_cell_grid(h->d_cell_aabb, ncells, h->grid, h->stream));
        mark("cell grid");
        h->orig.resize(Np);
        if (Np) CK(cudaMemcpy(h->orig.data(), h->d_orig, static_cast<size_t>(Np) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
    CK(dalloc(&h->d_ohe, static_cast<size_t>(M) * 3));
    CK(dalloc(&h->d_osl, static_cast<size_t>(M) * std::max(C, 1) * 3));
    CK(dalloc(&h->d_osr, M));
    CK(dalloc(&h->d_osn, M));
    CK(dalloc(&h->d_state, static_cast<size_t>(N) + 16));
    CK(dalloc(&h->d_state_c, static_cast<size_t>(Np) + 16));
    CK(dalloc(&h->d_cnt, Np));
    CK(dalloc(&h->d_over, static_cast<size_t>(h->words) * Np));
    CK(dalloc(&h->d_under, static_cast<size_t>(h->words) * Np));
    CK(dalloc(&h->d_cur, M));
    CK(dalloc(&h->d_cur_union, static_cast<size_t>(M) * 6));
    CK(dalloc(&h->d_ctr, 32));  // [0..15] per batch (zeroed by pose), [16] running gray count
    CK(dalloc(&h->d_mtop, 1));
    h->d_unknown = h->d_ctr + 16;
    CK(dalloc(&h->d_census, 16));
    CK(dalloc(&h->d_crec, ncells));
    h->items_cap = static_cast<int32_t>(std::min<int64_t>(INT32_MAX / 2, std::max<int64_t>(1 << 16, 8ll * Np)));
    if (const char* e = std::getenv("RGG_ITEMS_CAP"))  // tests: start tiny to exercise the grow-and-replay path
        h->items_cap = std::max(16, std::atoi(e));
    CK(dalloc(&h->d_items_over, h->items_cap));
    CK(dalloc(&h->d_items_under, h->items_cap));
    CK(dalloc(&h->d_items_recheck, rggk::kRecheckCap));
    h->recheck_cap = rggk::kRecheckCap;
    if (const char* e = std::getenv("RGG_RECHECK_CAP"))  // tests: a tiny queue takes the re-run-every-item path
        h->recheck_cap = std::min(rggk::kRecheckCap, std::max(0, std::atoi(e)));
    // small batches decide the undecided SAT pairs inline: their narrow phase is short, so the
    // queued pairs' fp64 chain after the over grid costs more than the occupancy saves
    h->recheck_min_moves = 128;
    if (const char* e = std::getenv("RGG_RECHECK_MIN_MOVES"))  // tests: the queue for every batch size
        h->recheck_min_moves = std::max(0, std::atoi(e));
    CK(dalloc(&h->d_gray, N));
    CK(dalloc(&h->d_tiles, N / 4096 + 2));
    CK(dalloc(&h->d_hits, N));
    CK(dalloc(&h->d_hits_prev, static_cast<size_t>(N) + 16));
    CK(dalloc(&h->d_cell_count, ncells));
    CK(dalloc(&h->d_cell_list, static_cast<size_t>(ncells) * cap));
    CK(dalloc(&h->d_cell_ovf, ncells));
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_ctr), 32 * sizeof(int32_t), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->dh_ctr), h->h_ctr, 0));
    auto up = [&](void* dst, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream) : cudaSuccess;
    };
    CK(up(h->d_ohe, v->obst_he, static_cast<size_t>(M) * 3 * sizeof(double)));
    CK(up(h->d_osl, v->obst_sph_local, static_cast<size_t>(M) * C * 3 * sizeof(double)));
    CK(up(h->d_osr, v->obst_sph_r, static_cast<size_t>(M) * sizeof(double)));
    CK(up(h->d_osn, v->obst_sph_n, static_cast<size_t>(M) * sizeof(int32_t)));
    // labels: GREEN for owned components, 0xFF for components of other shards
    CK(cudaMemsetAsync(h->d_state, shards > 1 ? 0xFF : 0, static_cast<size_t>(N) + 16, h->stream));
    if (shards > 1) {
        std::vector<uint8_t> st(static_cast<size_t>(N), 0xFF);
        for (int32_t c : h->orig) st[c] = 0;
        CK(cudaMemcpyAsync(h->d_state, st.data(), st.size(), cudaMemcpyHostToDevice, h->stream));
        CK(stream_wait(h));
    }
    CK(cudaMemsetAsync(h->d_state_c, 0, static_cast<size_t>(Np) + 16, h->stream));
    CK(cudaMemsetAsync(h->d_cnt, 0, static_cast<size_t>(Np) * sizeof(uint32_t), h->stream));
    CK(cudaMemsetAsync(h->d_over, 0, static_cast<size_t>(h->words) * Np * 8, h->stream));
    CK(cudaMemsetAsync(h->d_under, 0, static_cast<size_t>(h->words) * Np * 8, h->stream));
    CK(cudaMemsetAsync(h->d_ctr, 0, 32 * sizeof(int32_t), h->stream));

    Store& s = h->s;
    s.N = N;
    s.Np = Np;
    s.B = B;
    s.S = S;
    s.M = M;
    s.C = C;
    s.W = h->words;
    s.cell = cell;
    s.ncells = ncells;
    s.cap = cap;
    s.use_under = o.use_under ? 1 : 0;
    {
        // narrow operands of the whole roadmap: Box32 lines and segment records
        const double bytes = 128.0 * Np * B + 32.0 * static_cast<double>(h->total_segs_owned);
        int l2 = 0;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device);
        s.prefetch = bytes <= 0.5 * l2 ? 1 : 0;
    }
    s.aabb = h->d_aabb;
    s.sat = h->d_sat;
    s.sat32 = h->d_sat32;
    s.row = h->d_row;
    s.seg = h->d_seg;
    s.seg32 = h->d_seg32;
    s.spline_r = h->d_spline;
    s.orig = h->d_orig;
    s.cell_aabb = h->d_cell_aabb;
    s.slice_aabb = h->d_slice_aabb;
    for (int k = 0; k < 3; ++k) s.gorg[k] = h->grid.org[k], s.ginv[k] = h->grid.inv[k], s.gdim[k] = h->grid.dim[k];
    s.gcell_off = h->grid.off;
    s.gcell = h->grid.cells;
    s.ohe = h->d_ohe;
    s.osl = h->d_osl;
    s.osr = h->d_osr;
    s.osn = h->d_osn;
    s.state = h->d_state;
    s.state_c = h->d_state_c;
    s.rank = h->d_rank;
    s.cnt = h->d_cnt;
    s.over = h->d_over;
    s.under = h->d_under;
    s.cur = h->d_cur;
    s.cur_union = h->d_cur_union;
    mark("rest");
    CK(rggk::launch_init_obstacles(s, nullptr, h->stream));
    h->grid_classify = std::max(1, std::min(ncells, h->sms * rggk::classify_occupancy(cell, rggk::kPerMove)));
    const int rc = grow_batch(h, 64);
    if (rc) return rc;
    CK(stream_wait(h));
    mark("batch");
    h->unknown = 0;
    h->unknown_stale = false;
    return RGG_OK;
}

}  // namespace

extern "C" {

void rgg_gpu_destroy(rgg_gpu* h) {
    if (!h) return;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->done_ev) cudaEventDestroy(h->done_ev);
    void* dev[] = {h->d_aabb, h->d_sat, h->d_sat32, h->grid.off, h->grid.cells, h->d_cmask, h->d_evbox, h->d_evt, h->d_evs, h->d_units, h->d_unit_ready, h->d_row, h->d_seg, h->d_seg32, h->d_spline, h->d_orig, h->d_rank, h->d_cell_aabb, h->d_slice_aabb,
                   h->d_ohe, h->d_osl, h->d_osr, h->d_osn, h->d_state, h->d_state_c, h->d_cnt, h->d_over, h->d_under, h->d_cur,
                   h->d_cur_union, h->d_ctr, h->d_census, h->d_gray, h->d_tiles, h->d_hits, h->d_cell_count,
                   h->d_cell_list, h->d_cell_ovf, h->d_ids, h->d_last, h->d_mtop, h->d_crec, h->d_items_over, h->d_items_under, h->d_items_recheck, h->d_mpool, h->d_ev,
                   h->d_mv, h->d_pool, h->d_tl, h->d_hits_prev, h->d_evready,
                   h->d_res_he, h->d_res_off, h->d_res_pose, h->d_opoly, h->d_res_spose, h->d_res_sact, h->d_res_ids, h->d_res_cnt, h->d_res_out,
                   h->d_eg_ids, h->d_eg_rt, h->d_eg_rep};
    for (void* p : dev)
        if (p) cudaFree(p);
    void* pin[] = {h->h_ids, h->h_mv, h->h_ctr, h->h_eg_rep, h->h_gray, h->h_gray_map};
    for (void* p : pin)
        if (p) cudaFreeHost(p);
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
}

static int update_core(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                       rgg_update_report* reports);
static int update_eager(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                        rgg_update_report* reports);

int rgg_gpu_update(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                   rgg_update_report* reports) {
    if (!h) return RGG_EINVAL;
    clear_stale_error();
    if (h->poisoned) return fail(h, RGG_ELOGIC, "engine state lost after a failed eager update");
    if (n < 0 || (n > 0 && (!ids || !rt12))) return fail(h, RGG_EINVAL, "bad move list");
    if (n >= kMaxBatch) return fail(h, RGG_EINVAL, "at most 2^26 - 1 moves per batch (split it)");
    if (!(flags & (RGG_LAZY | RGG_EAGER)))
        return fail(h, RGG_EINVAL, "pass RGG_LAZY or RGG_EAGER");
    if ((flags & RGG_ASYNC) && (reports || (flags & RGG_EAGER)))
        return fail(h, RGG_EINVAL, "reports and eager updates need a synchronous update");
    if (!(flags & RGG_EAGER)) return update_core(h, ids, rt12, n, flags, reports);
    // eager: one move at a time, each resolving its gray over-hits before the next
    // (BatchEngine::batch_update(moves, false) = update_obstacle per move)
    if (!h->res_ready) return fail(h, RGG_EINVAL, "eager updates need rgg_gpu_set_resolver");
    return update_eager(h, ids, rt12, n, flags, reports);
}

// Eager batch, chained on the device: per move one single-move graph (pose ..
// apply + exact resolve of the move's gray over-hits) and one staging kernel;
// one H2D of all moves before and one D2H of all report slots after.  A single
// move lists at most one event per cell, so its item queues (sized below) and
// pools cannot overflow: no per-move host check is needed.
static int update_eager(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                        rgg_update_report* reports) {
    CK(cudaSetDevice(h->device));
    int32_t k = 0;
    while (k < n && ids[k] >= 0 && ids[k] < h->s.M) ++k;
    if (k > 0) {
        int rc = refresh_unknown(h);
        if (rc) return rc;
        rc = grow_batch(h, 1);
        if (rc) return rc;
        rc = grow_pinned(h, k);
        if (rc) return rc;
        // a single move queues at most one over item per component and one under item per
        // segment: queues this large cannot fill during an eager batch
        const int64_t need = std::max<int64_t>(h->s.Np, h->total_segs_owned);
        if (h->items_cap < need) {
            rc = grow_items(h, need);
            if (rc) return rc;
        }
        if (k > h->eager_cap) {
            const int32_t cap = std::max(k, std::max(64, 2 * h->eager_cap));
            cudaFree(h->d_eg_ids), cudaFree(h->d_eg_rt), cudaFree(h->d_eg_rep), cudaFreeHost(h->h_eg_rep);
            h->d_eg_ids = nullptr, h->d_eg_rt = nullptr, h->d_eg_rep = nullptr, h->h_eg_rep = nullptr;
            CK(dalloc(&h->d_eg_ids, cap));
            CK(dalloc(&h->d_eg_rt, static_cast<size_t>(cap) * 12));
            CK(dalloc(&h->d_eg_rep, static_cast<size_t>(cap) * 8));
            CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_eg_rep), static_cast<size_t>(cap) * 8 * sizeof(int32_t), 0));
            h->eager_cap = cap;
        }
        if (ids != h->h_ids) std::memcpy(h->h_ids, ids, k * sizeof(int32_t));  // moves staged by the caller stay
        if (rt12 != h->h_rt) std::memcpy(h->h_rt, rt12, static_cast<size_t>(k) * 96);
        CK(cudaMemsetAsync(h->d_ctr + 18, 0, sizeof(int32_t), h->stream));  // the batch's sticky status
        CK(cudaMemcpyAsync(h->d_eg_ids, h->h_ids, k * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemcpyAsync(h->d_eg_rt, h->h_rt, static_cast<size_t>(k) * 96, cudaMemcpyHostToDevice, h->stream));
        const Batch b = batch_of(h, 1);
        const int32_t ef = RGG_EAGER | RGG_PER_MOVE | (flags & RGG_GRAY_LIST);
        for (int32_t i = 0; i <= k; ++i) {
            CK(rggk::launch_eager_step(b, h->d_ids, h->d_rt, h->d_eg_ids, h->d_eg_rt, h->d_eg_rep, i, k, h->stream));
            if (i < k) {
                rc = enqueue(h, 1, ef);
                if (rc) return rc;
            }
        }
        CK(cudaMemcpyAsync(h->h_eg_rep, h->d_eg_rep, static_cast<size_t>(k) * 8 * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, h->stream));
        CK(cudaMemcpyAsync(h->h_ctr, h->d_ctr, 24 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
        CK(stream_wait(h));
        if (h->h_ctr[6] | h->h_ctr[18]) {
            // some move failed on the device and the moves after it were applied: the
            // engine's state is no longer the reference's, so every later call fails
            h->poisoned = true;
            return fail(h, RGG_ELOGIC, "eager update failed on the device (engine state lost)");
        }
        int32_t u = h->unknown;
        for (int32_t i = 0; i < k; ++i) {
            const int32_t* q = h->h_eg_rep + 8 * i;  // mv[4], hits, resolve deltas [3]
            const int32_t after = u + q[2] - q[3];
            u = after - q[4];
            if (!reports) continue;
            rgg_update_report& r = reports[i];
            std::memset(&r, 0, sizeof(r));
            r.obstacle = ids[i];
            r.new_green = q[0] + q[5];
            r.new_red = q[1] + q[6];
            r.new_gray = q[2] + q[7];
            r.unknown_after_heuristic = after;
            r.residual_unknown = u;
            r.resolve_checks = q[4];
        }
        if (u != h->h_ctr[16]) return fail(h, RGG_ELOGIC, "eager update: gray count out of step");
        h->unknown = u;
        h->unknown_stale = false;
    }
    if (k < n) return fail(h, RGG_EINVAL, "unknown obstacle id");
    return RGG_OK;
}

static int update_core(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                       rgg_update_report* reports) {
    CK(cudaSetDevice(h->device));
    // the reference applies moves in order and throws at the first bad id
    int32_t k = 0;
    while (k < n && ids[k] >= 0 && ids[k] < h->s.M) ++k;
    const bool bad = k < n;
    if (k > 0) {
        if (reports && (flags & RGG_PER_MOVE)) {
            const int rc = refresh_unknown(h);
            if (rc) return rc;
        }
        const int32_t u0 = h->unknown;
        int rc = grow_batch(h, k);
        if (rc) return rc;
        rc = grow_pinned(h, k);
        if (rc) return rc;
        // moves the caller wrote into the staging buffers (rgg_gpu_stage) are already in place
        if (ids != h->h_ids) std::memcpy(h->h_ids, ids, k * sizeof(int32_t));
        if (rt12 != h->h_rt) std::memcpy(h->h_rt, rt12, static_cast<size_t>(k) * 12 * sizeof(double));
        // synchronous update with matching staging layouts: the copies are graph nodes
        const bool hostio = !(flags & RGG_ASYNC) && !bad && h->pin_off == h->in_off && graphs_enabled(h);
        if (hostio) {
            reinterpret_cast<volatile int32_t*>(h->h_ctr)[31] = 0;
            rc = enqueue(h, k, flags | kHostIO);
            if (rc) return rc;
        } else if (h->pin_off == h->in_off) {  // same layout on both sides: one copy
            CK(cudaMemcpyAsync(h->d_ids, h->h_ids, h->in_off + static_cast<size_t>(k) * 96, cudaMemcpyHostToDevice,
                               h->stream));
        } else {
            CK(cudaMemcpyAsync(h->d_ids, h->h_ids, k * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
            CK(cudaMemcpyAsync(h->d_rt, h->h_rt, static_cast<size_t>(k) * 96, cudaMemcpyHostToDevice, h->stream));
        }
        if (!hostio) {
            rc = enqueue(h, k, flags);
            if (rc) return rc;
        }
        if (!(flags & RGG_ASYNC) || bad) {
            if (!hostio) {
                if (reports) CK(cudaMemcpyAsync(h->h_mv, h->d_mv, static_cast<size_t>(k) * 4 * sizeof(int32_t),
                                                cudaMemcpyDeviceToHost, h->stream));
                CK(cudaMemcpyAsync(h->h_ctr, h->d_ctr, 24 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
            }
            if (hostio) {
                // poll the flag the last kernel stores into mapped memory (lower wake-up latency
                // than a stream sync); the stream is queried now and then so that a failed
                // launch cannot hang the caller
                volatile int32_t* flag = reinterpret_cast<volatile int32_t*>(h->h_ctr) + 31;
                for (unsigned spins = 1; *flag == 0; ++spins) {
                    if ((spins & 1023) == 0) {
                        const cudaError_t q = cudaStreamQuery(h->stream);
                        if (q == cudaSuccess) break;  // stream idle: the flag must be visible now
                        if (q != cudaErrorNotReady) CK(q);
                    }
                }
                std::atomic_thread_fence(std::memory_order_acquire);
            } else {
                CK(stream_wait(h));
            }
            dump_timeline(h);
            for (int attempt = 0; h->h_ctr[6] == 3 && attempt < 4; ++attempt) {
                // the update was not applied (apply kernel skipped): grow the queue and replay it
                rc = grow_items(h, std::max<int64_t>(h->h_ctr[8], h->h_ctr[9]));
                if (rc) return rc;
                rc = enqueue(h, k, flags);
                if (rc) return rc;
                if (reports) CK(cudaMemcpyAsync(h->h_mv, h->d_mv, static_cast<size_t>(k) * 4 * sizeof(int32_t),
                                                cudaMemcpyDeviceToHost, h->stream));
                CK(cudaMemcpyAsync(h->h_ctr, h->d_ctr, 24 * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
                CK(stream_wait(h));
            }
            if (h->h_ctr[6])
                return fail(h, RGG_ELOGIC, h->h_ctr[6] == 1   ? "overflow pool exhausted"
                                           : h->h_ctr[6] == 2 ? "mask pool exhausted"
                                           : h->h_ctr[6] == 4 ? "device handoff timed out"
                                                              : "narrow item queue full (split the batch)");
            h->unknown = h->h_ctr[16];
            h->unknown_stale = false;
            if (reports) {
                float t[4] = {0, 0, 0, 0};
                if (h->phase_timing)
                    for (int p = 0; p < 4; ++p) cudaEventElapsedTime(&t[p], h->ev[p], h->ev[p + 1]);
                int32_t u = u0;
                for (int32_t i = 0; i < k; ++i) {
                    rgg_update_report& r = reports[i];
                    std::memset(&r, 0, sizeof(r));
                    r.obstacle = ids[i];
                    if (flags & RGG_PER_MOVE) {
                        r.new_green = h->h_mv[4 * i];
                        r.new_red = h->h_mv[4 * i + 1];
                        r.new_gray = h->h_mv[4 * i + 2];
                        u += r.new_gray - h->h_mv[4 * i + 3];
                        r.unknown_after_heuristic = u;
                        r.residual_unknown = u;
                    } else {
                        r.unknown_after_heuristic = r.residual_unknown = h->unknown;
                    }
                    if (flags & RGG_EAGER) {  // n == 1: the resolve's finish_counts terms
                        const int32_t checks = h->h_ctr[5];
                        r.new_green += h->h_ctr[20];
                        r.new_red += h->h_ctr[21];
                        r.new_gray += h->h_ctr[22];
                        r.resolve_checks = checks;
                        r.residual_unknown = r.unknown_after_heuristic - checks;
                    }
                }
                rgg_update_report& last = reports[k - 1];
                last.reval_us = static_cast<int64_t>(t[0] * 1000.0f);
                last.over_us = static_cast<int64_t>(t[1] * 1000.0f);
                last.under_us = static_cast<int64_t>(t[2] * 1000.0f);
                last.resolve_us = static_cast<int64_t>(t[3] * 1000.0f);
            }
        }
    }
    if (bad) return fail(h, RGG_EINVAL, "unknown obstacle id");
    return RGG_OK;
}

int rgg_gpu_update_device(rgg_gpu* h, const int32_t* d_ids, const double* d_rt12, int32_t n, int32_t flags) {
    if (!h) return RGG_EINVAL;
    clear_stale_error();
    if (n <= 0) return RGG_OK;
    if (!(flags & RGG_LAZY)) return fail(h, RGG_EINVAL, "only lazy updates run on device");
    if (n >= kMaxBatch) return fail(h, RGG_EINVAL, "at most 2^26 - 1 moves per batch (split it)");
    CK(cudaSetDevice(h->device));
    const int rc = grow_batch(h, n);
    if (rc) return rc;
    // no host round trip: ids are trusted; prev/last links are computed by the pose kernel
    CK(cudaMemcpyAsync(h->d_ids, d_ids, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_rt, d_rt12, static_cast<size_t>(n) * 12 * sizeof(double), cudaMemcpyDeviceToDevice,
                       h->stream));
    return enqueue(h, n, flags | RGG_ASYNC);
}

int rgg_gpu_sync(rgg_gpu* h) {
    if (!h) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    int32_t err = 0;
    CK(cudaMemcpyAsync(&err, h->d_ctr + 6, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    dump_timeline(h);
    if (err == 3) {
        int32_t need[2] = {0, 0};
        CK(cudaMemcpy(need, h->d_ctr + 8, sizeof(need), cudaMemcpyDeviceToHost));
        const int rc = grow_items(h, std::max(need[0], need[1]));
        if (rc) return rc;
        return fail(h, RGG_ELOGIC, "narrow item queue was full: the last asynchronous update was not applied "
                                   "(queue grown; resubmit it)");
    }
    return RGG_OK;
}

void* rgg_gpu_stream(rgg_gpu* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

int rgg_gpu_count(const rgg_gpu* h, int32_t* n_components, int32_t* n_obstacles, int32_t* words_per_comp) {
    if (!h) return RGG_EINVAL;
    if (n_components) *n_components = h->s.N;
    if (n_obstacles) *n_obstacles = h->s.M;
    if (words_per_comp) *words_per_comp = h->words;
    return RGG_OK;
}

int rgg_gpu_read_states(rgg_gpu* h, uint8_t* out) {
    if (!h || !out) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(out, h->d_state, h->s.N, cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    return RGG_OK;
}

int rgg_gpu_read_bits(rgg_gpu* h, uint64_t* out, int32_t words_per_comp) {
    if (!h || !out) return RGG_EINVAL;
    if (words_per_comp < h->words) return fail(h, RGG_EINVAL, "words_per_comp too small");
    CK(cudaSetDevice(h->device));
    const int32_t Np = h->s.Np;
    std::vector<uint64_t> w(static_cast<size_t>(h->words) * Np);
    if (!w.empty()) {
        CK(cudaMemcpyAsync(w.data(), h->d_over, w.size() * 8, cudaMemcpyDeviceToHost, h->stream));
        CK(stream_wait(h));
    }
    std::memset(out, 0, static_cast<size_t>(h->s.N) * words_per_comp * 8);
    for (int32_t i = 0; i < Np; ++i)
        for (int32_t k = 0; k < h->words; ++k)
            out[static_cast<size_t>(h->orig[i]) * words_per_comp + k] = w[static_cast<size_t>(k) * Np + i];
    return RGG_OK;
}

int rgg_gpu_unknown_count(rgg_gpu* h, int32_t* out) {
    if (!h || !out) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    const int rc = refresh_unknown(h);
    if (rc) return rc;
    *out = h->unknown;
    return RGG_OK;
}

int rgg_gpu_gray_ids(rgg_gpu* h, int32_t* out, int32_t cap, int32_t* n) {
    if (!h || !n) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    if (!h->gray_fresh) {  // ordered ballot/prefix compaction of the current labels
        CK(rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream));
        h->gray_fresh = true;
    }
    const int rc = refresh_unknown(h);
    if (rc) return rc;
    *n = h->unknown;
    if (out && cap > 0 && h->unknown > 0) {
        CK(cudaMemcpyAsync(out, h->d_gray, std::min(cap, h->unknown) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                           h->stream));
        CK(stream_wait(h));
    }
    return RGG_OK;
}

int rgg_gpu_gray_device(rgg_gpu* h, int32_t* d_count, int32_t* d_ids, int32_t cap) {
    if (!h) return RGG_EINVAL;
    if (cap < 0 || (cap > 0 && !d_ids)) return fail(h, RGG_EINVAL, "bad gray id buffer");
    CK(cudaSetDevice(h->device));
    if (!h->gray_fresh) {
        CK(rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream));
        h->gray_fresh = true;
    }
    if (d_count) CK(cudaMemcpyAsync(d_count, h->d_ctr + 4, sizeof(int32_t), cudaMemcpyDeviceToDevice, h->stream));
    const int32_t n = std::min(cap, h->s.N);
    if (n > 0) CK(cudaMemcpyAsync(d_ids, h->d_gray, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                                  h->stream));
    return RGG_OK;
}

int rgg_gpu_stage(rgg_gpu* h, int32_t n, int32_t** ids, double** rt12) {
    if (!h || n < 0 || !ids || !rt12) return RGG_EINVAL;
    if (n >= kMaxBatch) return fail(h, RGG_EINVAL, "at most 2^26 - 1 moves per batch (split it)");
    CK(cudaSetDevice(h->device));
    int rc = grow_batch(h, std::max(n, 1));  // device and staging capacities grow together
    if (rc) return rc;
    rc = grow_pinned(h, std::max(n, 1));
    if (rc) return rc;
    *ids = h->h_ids;
    *rt12 = h->h_rt;
    return RGG_OK;
}

int rgg_gpu_gray_view(rgg_gpu* h, const int32_t** ids, int32_t* n) {
    if (!h || !ids || !n) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    if (h->gray_host_fresh) {  // written by the last update itself (synchronous, RGG_GRAY_LIST);
        *ids = h->h_gray_map;    // its count came back with the update's counters (ctr[4])
        *n = h->h_ctr[4];
        return RGG_OK;
    }
    if (!h->gray_fresh) {
        CK(rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream));
        h->gray_fresh = true;
    }
    const int rc = refresh_unknown(h);
    if (rc) return rc;
    const int32_t cnt = h->unknown;
    if (cnt > h->gray_pin_cap) {
        cudaFreeHost(h->h_gray);
        h->h_gray = nullptr;
        h->gray_pin_cap = 0;
        CK(cudaHostAlloc(reinterpret_cast<void**>(&h->h_gray), static_cast<size_t>(std::max(cnt, 1)) * sizeof(int32_t),
                         cudaHostAllocDefault));
        h->gray_pin_cap = std::max(cnt, 1);
    }
    if (cnt > 0) {
        CK(cudaMemcpyAsync(h->h_gray, h->d_gray, static_cast<size_t>(cnt) * sizeof(int32_t), cudaMemcpyDeviceToHost,
                           h->stream));
        CK(stream_wait(h));
    }
    *ids = h->h_gray;
    *n = cnt;
    return RGG_OK;
}

int rgg_gpu_last_hits(rgg_gpu* h, int32_t* out, int32_t cap, int32_t* n) {
    if (!h || !n) return RGG_EINVAL;
    if (!h->last_hits_valid) return fail(h, RGG_EINVAL, "last hits are kept for single-move updates only");
    CK(cudaSetDevice(h->device));
    int32_t cnt = 0;
    CK(cudaMemcpyAsync(&cnt, h->d_ctr + 5, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    *n = cnt;
    if (out && cap > 0 && cnt > 0) {
        CK(cudaMemcpyAsync(out, h->d_hits, std::min(cap, cnt) * sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
        CK(stream_wait(h));
        std::sort(out, out + std::min(cap, cnt));
    }
    return RGG_OK;
}

int rgg_gpu_write_states(rgg_gpu* h, const int32_t* ids, const uint8_t* st, int32_t n) {
    if (!h) return RGG_EINVAL;
    if (n <= 0) return RGG_OK;
    for (int32_t i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= h->s.N) return fail(h, RGG_EINVAL, "unknown component id");
        if (st[i] > 2) return fail(h, RGG_EINVAL, "bad validity state");
    }
    CK(cudaSetDevice(h->device));
    int32_t* d_ids = nullptr;
    uint8_t* d_st = nullptr;
    CK(dalloc(&d_ids, n));
    CK(dalloc(&d_st, n));
    CK(cudaMemcpyAsync(d_ids, ids, n * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(d_st, st, n, cudaMemcpyHostToDevice, h->stream));
    CK(rggk::launch_write_states(h->s, d_ids, d_st, n, h->stream));
    CK(rggk::launch_compact(h->s, h->d_gray, h->d_tiles, h->d_ctr + 4, h->stream));
    CK(cudaMemcpyAsync(h->d_unknown, h->d_ctr + 4, sizeof(int32_t), cudaMemcpyDeviceToDevice, h->stream));
    CK(stream_wait(h));
    h->gray_fresh = true;
    h->gray_host_fresh = false;
    cudaFree(d_ids);
    cudaFree(d_st);
    h->unknown_stale = true;
    h->last_hits_valid = false;
    return RGG_OK;
}

int rgg_gpu_filter_stats(rgg_gpu* h, int64_t* sat_rechecks, int64_t* seg_rechecks, int32_t reset) {
    if (!h) return RGG_EINVAL;
    CK(cudaSetDevice(h->device));
    CK(stream_wait(h));
    unsigned long long fs[4] = {0, 0, 0, 0};
    rggk::filter_stats(fs, reset != 0);
    if (sat_rechecks) *sat_rechecks = static_cast<int64_t>(fs[1]);
    if (seg_rechecks) *seg_rechecks = static_cast<int64_t>(fs[3]);
    return RGG_OK;
}

int rgg_gpu_set_resolver(rgg_gpu* h, const rgg_resolve_view* v) {
    if (!h || !v) return RGG_EINVAL;
    clear_stale_error();
    if (v->n_components != h->s.N) return fail(h, RGG_EINVAL, "resolver: component count differs from the layout");
    if (v->n_bodies != h->s.B) return fail(h, RGG_EINVAL, "resolver: body count differs from the layout");
    if (!v->body_half_extents || !v->pose_off || (!v->poses && v->pose_off[v->n_components] > 0))
        return fail(h, RGG_EINVAL, "resolver: null array");
    const int32_t N = v->n_components, B = v->n_bodies;
    if (v->pose_off[0] != 0) return fail(h, RGG_EINVAL, "resolver: pose_off[0] must be 0");
    for (int32_t c = 0; c < N; ++c)
        if (v->pose_off[c + 1] < v->pose_off[c]) return fail(h, RGG_EINVAL, "resolver: pose_off not ascending");
    for (int k = 0; k < 3 * B; ++k)
        if (!(v->body_half_extents[k] > 0.0)) return fail(h, RGG_EINVAL, "degenerate polytope");  // geometry.cpp:280
    const int64_t total = v->pose_off[N];
    CK(cudaSetDevice(h->device));
    cudaFree(h->d_res_he);
    cudaFree(h->d_res_off);
    cudaFree(h->d_res_pose);
    h->d_res_he = nullptr, h->d_res_off = nullptr, h->d_res_pose = nullptr;
    CK(dalloc(&h->d_res_he, static_cast<size_t>(B) * 3));
    CK(dalloc(&h->d_res_off, static_cast<size_t>(N) + 1));
    CK(dalloc(&h->d_res_pose, static_cast<size_t>(total) * B * 12));
    if (!h->d_opoly) CK(dalloc(&h->d_opoly, static_cast<size_t>(std::max(1, h->s.M))));
    if (!h->d_res_ids) CK(dalloc(&h->d_res_ids, static_cast<size_t>(N) + 1));
    if (!h->d_res_out) CK(dalloc(&h->d_res_out, static_cast<size_t>(N) + 1));
    if (!h->d_res_cnt) CK(dalloc(&h->d_res_cnt, 1));
    // stream-ordered copies: a synchronous cudaMemcpy from pageable memory runs on the
    // legacy stream and may return before its DMA lands, unordered with h->stream's kernels
    CK(cudaMemcpyAsync(h->d_res_he, v->body_half_extents, static_cast<size_t>(B) * 3 * sizeof(double),
                       cudaMemcpyHostToDevice, h->stream));
    static_assert(sizeof(long long) == sizeof(int64_t), "int64 offsets");
    CK(cudaMemcpyAsync(h->d_res_off, v->pose_off, (static_cast<size_t>(N) + 1) * sizeof(int64_t),
                       cudaMemcpyHostToDevice, h->stream));
    if (total > 0)
        CK(cudaMemcpyAsync(h->d_res_pose, v->poses, static_cast<size_t>(total) * B * 12 * sizeof(double),
                           cudaMemcpyHostToDevice, h->stream));
    CK(stream_wait(h));  // the caller's arrays may go away on return
    h->res_B = B;
    h->res_ready = true;
    ++h->gen;  // captured eager graphs hold the old resolver pointers
    return RGG_OK;
}

int rgg_gpu_set_active_obstacles(rgg_gpu* h, const int32_t* ids, const double* rt, int32_t n) {
    if (!h) return RGG_EINVAL;
    clear_stale_error();
    if (n < 0 || (n > 0 && (!ids || !rt))) return fail(h, RGG_EINVAL, "bad obstacle list");
    for (int32_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= h->s.M) return fail(h, RGG_EINVAL, "unknown obstacle id");
    const int32_t M = std::max(1, h->s.M);
    std::vector<uint8_t> act(static_cast<size_t>(M), 0);
    std::vector<double> pose(static_cast<size_t>(M) * 12, 0.0);
    for (int32_t i = 0; i < n; ++i) {  // a repeated id: the last pose wins
        act[ids[i]] = 1;
        std::copy(rt + 12 * static_cast<size_t>(i), rt + 12 * static_cast<size_t>(i) + 12, pose.begin() + 12 * ids[i]);
    }
    CK(cudaSetDevice(h->device));
    if (!h->d_res_sact) {
        CK(dalloc(&h->d_res_spose, static_cast<size_t>(M) * 12));
        CK(dalloc(&h->d_res_sact, static_cast<size_t>(M)));
        ++h->gen;  // captured eager graphs were built without these pointers
    }
    // stream-ordered after any queued resolve that still reads the old list, and before the
    // next update's (a synchronous pageable cudaMemcpy is neither: it runs on the legacy
    // stream and may return before its DMA lands)
    CK(cudaMemcpyAsync(h->d_res_spose, pose.data(), pose.size() * sizeof(double), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_res_sact, act.data(), act.size(), cudaMemcpyHostToDevice, h->stream));
    CK(stream_wait(h));
    return RGG_OK;
}

int rgg_gpu_resolve_all(rgg_gpu* h, int32_t* resolved) {
    if (!h) return RGG_EINVAL;
    clear_stale_error();
    if (!h->res_ready) return fail(h, RGG_EINVAL, "resolve_all_unknown needs rgg_gpu_set_resolver");
    CK(cudaSetDevice(h->device));
    int32_t n = 0;
    int rc = rgg_gpu_gray_ids(h, nullptr, 0, &n);  // compacts the gray list on the device
    if (rc) return rc;
    if (n > 0) {
        const Batch b = batch_of(h, 1);
        CK(rggk::launch_resolve(h->s, resolver_of(h), b, h->d_gray, h->d_ctr + 4, n, rggk::kResolve, nullptr,
                                h->stream));
        CK(stream_wait(h));
    }
    h->gray_fresh = false;
    h->gray_host_fresh = false;
    h->unknown_stale = true;
    h->last_hits_valid = false;
    rc = refresh_unknown(h);
    if (rc) return rc;
    if (resolved) *resolved = n;
    return RGG_OK;
}

int rgg_gpu_exact_check(rgg_gpu* h, const int32_t* ids, int32_t n, uint8_t* out) {
    if (!h) return RGG_EINVAL;
    clear_stale_error();
    if (!h->res_ready) return fail(h, RGG_EINVAL, "exact checks need rgg_gpu_set_resolver");
    if (n < 0 || n > h->s.N || (n > 0 && (!ids || !out))) return fail(h, RGG_EINVAL, "bad id list");
    for (int32_t i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= h->s.N) return fail(h, RGG_EINVAL, "unknown component id");
    if (n == 0) return RGG_OK;
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(h->d_res_ids, ids, static_cast<size_t>(n) * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(h->d_res_cnt, &n, sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    const Batch b = batch_of(h, 1);
    CK(rggk::launch_resolve(h->s, resolver_of(h), b, h->d_res_ids, h->d_res_cnt, n, rggk::kCheck, h->d_res_out,
                            h->stream));
    CK(cudaMemcpyAsync(out, h->d_res_out, n, cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    return RGG_OK;
}

int rgg_gpu_pair_masks(rgg_gpu* h, int32_t kind, const int32_t* cand, int32_t n, int32_t o, uint8_t* mask) {
    if (!h) return RGG_EINVAL;
    if (o < 0 || o >= h->s.M) return fail(h, RGG_EINVAL, "unknown obstacle id");
    if (kind != 0 && kind != 1) return fail(h, RGG_EINVAL, "kind must be 0 (over) or 1 (under)");
    if (n <= 0) return RGG_OK;
    for (int32_t i = 0; i < n; ++i)
        if (cand[i] < 0 || cand[i] >= h->s.N) return fail(h, RGG_EINVAL, "unknown component id");
    CK(cudaSetDevice(h->device));
    int32_t* d_c = nullptr;
    uint8_t* d_m = nullptr;
    CK(dalloc(&d_c, n));
    CK(dalloc(&d_m, n));
    CK(cudaMemcpyAsync(d_c, cand, n * sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    CK(rggk::launch_pair_masks(h->s, h->d_rank, kind, d_c, n, o, d_m, h->stream));
    CK(cudaMemcpyAsync(mask, d_m, n, cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    cudaFree(d_c);
    cudaFree(d_m);
    return RGG_OK;
}

int rgg_gpu_last_stats(rgg_gpu* h, rgg_gpu_stats* out) {
    if (!h || !out) return RGG_EINVAL;
    std::memset(out, 0, sizeof(*out));
    if (!h->timed) return RGG_OK;
    CK(cudaSetDevice(h->device));
    CK(stream_wait(h));
    float t[5] = {0, 0, 0, 0, 0};
    if (h->phase_timing)
        for (int p = 0; p < 4; ++p) CK(cudaEventElapsedTime(&t[p], h->ev[p], h->ev[p + 1]));
    CK(cudaEventElapsedTime(&t[4], h->ev[0], h->ev[4]));
    out->pose_ms = t[0];
    out->bin_ms = t[1];
    out->classify_ms = t[2];
    out->compact_ms = t[3];
    out->total_ms = t[4];
    int32_t ctr[8];
    CK(cudaMemcpy(ctr, h->d_ctr, sizeof(ctr), cudaMemcpyDeviceToHost));
    out->dirty_cells = ctr[0];
    out->overflow_cells = ctr[3];
    out->events = h->last_n;
    return RGG_OK;
}

// Re-runs the last batch's classification in counting mode (no state change):
// the reference's per-move work over the same (component, event) pairs.
int rgg_gpu_census(rgg_gpu* h, rgg_gpu_stats* out) {
    if (!h || !out) return RGG_EINVAL;
    if (h->last_n <= 0) return fail(h, RGG_EINVAL, "no update to count");
    if (h->last_single)
        return fail(h, RGG_EINVAL, "a single-move update keeps no cell lists to count: update with RGG_CENSUS");
    CK(cudaSetDevice(h->device));
    int rc = rgg_gpu_last_stats(h, out);
    if (rc) return rc;
    Batch b = batch_of(h, h->last_n);
    CK(cudaMemsetAsync(h->d_census, 0, 16 * sizeof(unsigned long long), h->stream));
    CK(rggk::launch_classify(h->s, b, rggk::kCensus, h->grid_classify, h->stream));
    unsigned long long c[16];
    CK(cudaMemcpyAsync(c, h->d_census, sizeof(c), cudaMemcpyDeviceToHost, h->stream));
    CK(stream_wait(h));
    out->over_pairs = static_cast<int64_t>(c[0]);
    out->sat_flops = static_cast<int64_t>(c[1]);
    out->under_pairs = static_cast<int64_t>(c[2]);
    out->seg_sphere_tests = static_cast<int64_t>(c[3]);
    out->over_hits = static_cast<int64_t>(c[4]);
    out->under_hits = static_cast<int64_t>(c[5]);
    // algorithmic bytes: every component of a dirty cell reads its AABB (48 B),
    // label (1 B), counters (4 B) and bit words (16 B per word) and writes them
    // back; components with an over item read their SatBoxes (B*168 B), those
    // with an under item their row offsets and real segments (56 B each).
    //   (bit words: W = 1 keeps both words of a component in registers -> 16 B read + 16 B
    //   written per component; W > 1 touches one over + one under word per touched pair)
    const int64_t dirty = static_cast<int64_t>(c[8]), box_comps = static_cast<int64_t>(c[9]),
                  sph_comps = static_cast<int64_t>(c[10]), segs = static_cast<int64_t>(c[11]),
                  touched = static_cast<int64_t>(c[12]);
    const int64_t bit_bytes = h->words == 1 ? dirty * 32 : touched * 32;
    out->bytes_components = dirty * (48 + 2 * (1 + 4)) + bit_bytes + box_comps * h->s.B * 168 +
                            sph_comps * 4 * (h->s.B * h->s.S + 1) + segs * 56;
    // per relabelled component B x 48 B of SatBox (centre + scaled
    // axes in fp32), 12 B per real-segment point (segments + rows), 8 B per row, the
    // label read and written, the counters read and written; 16 B of over / under bit
    // words read and written per touched (component, obstacle) pair; 96 B of pose per
    // move; 4 B per GRAY id of the compacted list
    const int64_t segs_all = static_cast<int64_t>(c[13]), rows = static_cast<int64_t>(h->s.B) * h->s.S;
    int32_t gray = 0;
    CK(cudaMemcpy(&gray, h->d_unknown, sizeof(int32_t), cudaMemcpyDeviceToHost));
    out->gray = gray;
    out->bytes_fp32 = dirty * (h->s.B * 48 + 8 * rows + 2 + 8) + 12 * (segs_all + dirty * rows) + 32 * touched +
                      96ll * h->last_n + 4ll * gray;
    return RGG_OK;
}

// Measured issue rates in GFLOP/s: fp64 non-FMA add/mul (the fp64-exact sequence's
// roof) and fp32 FMA (the filters' roof), best of 5 CUDA-event-timed launches.
static int peak_probe(int device, bool fp32, double* gflops) {
    rgg_gpu* h = nullptr;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    double* sink = nullptr;
    CK(cudaMalloc(&sink, 8));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int block = 256, grid = prop.multiProcessorCount * 8, iters = 4096;
    const auto run = [&]() {
        return fp32 ? rggk::launch_fp32_peak(reinterpret_cast<float*>(sink), iters, grid, block, nullptr)
                    : rggk::launch_fp64_peak(sink, iters, grid, block, nullptr);
    };
    CK(run());
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        CK(run());
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    const double flops = 2.0 * (fp32 ? 16.0 : 8.0) * iters * static_cast<double>(grid) * block;
    *gflops = flops / (best * 1e-3) / 1e9;
    return RGG_OK;
}

int rgg_gpu_fp64_peak(int device, double* gflops) { return peak_probe(device, false, gflops); }
int rgg_gpu_fp32_peak(int device, double* gflops) { return peak_probe(device, true, gflops); }

int rgg_gpu_owned(const rgg_gpu* h, int32_t* n_owned) {
    if (!h || !n_owned) return RGG_EINVAL;
    *n_owned = h->s.Np;
    return RGG_OK;
}

// exact_component_valid (roadmap.cpp:129-163) of independent configuration sets against
// a fixed obstacle list, without an engine: build_prm's node and edge checks (:69, :95-99).
int rgg_exact_valid_sets(int32_t device, int32_t n_sets, const int64_t* cfg_off, int32_t n_bodies,
                         const double* body_he, const double* poses, int32_t n_obst, const double* obst_he,
                         const double* obst_rt, uint8_t* free_out) {
    rgg_gpu* h = nullptr;
    clear_stale_error();
    if (n_sets < 0 || n_bodies < 1 || n_obst < 0) return RGG_EINVAL;
    if (n_sets == 0) return RGG_OK;
    if (!cfg_off || !body_he || !free_out || (n_obst > 0 && (!obst_he || !obst_rt))) return RGG_EINVAL;
    if (cfg_off[0] != 0) return RGG_EINVAL;
    for (int32_t c = 0; c < n_sets; ++c)
        if (cfg_off[c + 1] < cfg_off[c]) return RGG_EINVAL;
    const int64_t total = cfg_off[n_sets];
    if (total > 0 && !poses) return RGG_EINVAL;
    if (n_obst == 0) {  // exact_component_valid: no active obstacle, every set is free
        std::fill(free_out, free_out + n_sets, uint8_t{1});
        return RGG_OK;
    }
    for (int k = 0; k < 3 * n_bodies; ++k)
        if (!(body_he[k] > 0.0)) return RGG_EINVAL;  // ConvexPolytope::box: degenerate polytope
    for (int k = 0; k < 3 * n_obst; ++k)
        if (!(obst_he[k] > 0.0)) return RGG_EINVAL;
    CK(cudaSetDevice(device));
    struct Bufs {
        std::vector<void*> p;
        ~Bufs() {
            for (void* q : p) cudaFree(q);
        }
    } bufs;
    auto take = [&](auto** q, size_t n) {
        const cudaError_t e = dalloc(q, n);
        if (e == cudaSuccess) bufs.p.push_back(*q);
        return e;
    };
    double *d_bhe, *d_pose, *d_ohe, *d_spose, *d_union;
    long long* d_off;
    uint8_t *d_sact, *d_out;
    int32_t *d_ids, *d_cnt;
    rggk::ObsPoly* d_opoly;
    CK(take(&d_bhe, static_cast<size_t>(n_bodies) * 3));
    CK(take(&d_pose, static_cast<size_t>(total) * n_bodies * 12));
    CK(take(&d_off, static_cast<size_t>(n_sets) + 1));
    CK(take(&d_ohe, static_cast<size_t>(n_obst) * 3));
    CK(take(&d_spose, static_cast<size_t>(n_obst) * 12));
    CK(take(&d_union, static_cast<size_t>(n_obst) * 6));
    CK(take(&d_sact, static_cast<size_t>(n_obst)));
    CK(take(&d_opoly, static_cast<size_t>(n_obst)));
    CK(take(&d_out, static_cast<size_t>(n_sets)));
    CK(take(&d_ids, static_cast<size_t>(n_sets)));
    CK(take(&d_cnt, 1));
    std::vector<int32_t> ids(static_cast<size_t>(n_sets));
    for (int32_t i = 0; i < n_sets; ++i) ids[i] = i;
    std::vector<double> empty(static_cast<size_t>(n_obst) * 6);
    for (int32_t o = 0; o < n_obst; ++o)  // no engine moves: every obstacle is active at its listed pose
        for (int k = 0; k < 3; ++k) empty[6 * o + k] = 1.0, empty[6 * o + 3 + k] = 0.0;
    std::vector<uint8_t> act(static_cast<size_t>(n_obst), 1);
    static_assert(sizeof(long long) == sizeof(int64_t), "int64 offsets");
    CK(cudaMemcpy(d_bhe, body_he, static_cast<size_t>(n_bodies) * 3 * sizeof(double), cudaMemcpyHostToDevice));
    if (total > 0)
        CK(cudaMemcpy(d_pose, poses, static_cast<size_t>(total) * n_bodies * 12 * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_off, cfg_off, (static_cast<size_t>(n_sets) + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ohe, obst_he, static_cast<size_t>(n_obst) * 3 * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_spose, obst_rt, static_cast<size_t>(n_obst) * 12 * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_union, empty.data(), empty.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_sact, act.data(), act.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ids, ids.data(), ids.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_cnt, &n_sets, sizeof(int32_t), cudaMemcpyHostToDevice));
    rggk::Store st{};
    st.M = n_obst;
    st.ohe = d_ohe;
    st.cur_union = d_union;
    rggk::Resolver r{};
    r.B = n_bodies, r.he = d_bhe, r.off = d_off, r.pose = d_pose, r.opoly = d_opoly, r.spose = d_spose, r.sact = d_sact;
    rggk::Batch b{};
    CK(rggk::launch_resolve(st, r, b, d_ids, d_cnt, n_sets, rggk::kCheck, d_out, nullptr));
    CK(cudaMemcpy(free_out, d_out, static_cast<size_t>(n_sets), cudaMemcpyDeviceToHost));
    for (int32_t i = 0; i < n_sets; ++i) free_out[i] = free_out[i] ? 0 : 1;  // kCheck writes 1 = RED
    return RGG_OK;
}

}  // extern "C"

extern "C" int rgg_gpu_set_phase_timing(rgg_gpu* h, int32_t on) {
    if (!h) return RGG_EINVAL;
    h->phase_timing = on != 0;
    return RGG_OK;
}

extern "C" int rgg_gpu_copy_counters(rgg_gpu* h, void* dst_device, int32_t n) {
    if (!h || !dst_device) return RGG_EINVAL;
    if (n > h->last_n) return fail(h, RGG_EINVAL, "more counters than moves in the last update");
    CK(cudaSetDevice(h->device));
    CK(cudaMemcpyAsync(dst_device, h->d_mv, static_cast<size_t>(n) * 4 * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                       h->stream));
    return RGG_OK;
}
