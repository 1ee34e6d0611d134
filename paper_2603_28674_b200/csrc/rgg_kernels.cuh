// rgg_kernels.cuh — device data structures and kernel launchers shared by the
// C-ABI (rgg_capi.cu) and the kernels (rgg_kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "rgg_device.cuh"

namespace rggk {

constexpr int kMaxSpheres = 16;  // obstacle inner spheres per event (C)
constexpr int kEvS = kMaxSpheres + 1;  // float4 records per event in Batch::evs
constexpr int kEvChunk = 32;     // events staged in shared memory per pass (one bit each)
constexpr int kMaxCell = 128;
constexpr int kRecheckCap = 1 << 16;  // Batch::items_recheck entries (beyond: every over item is re-run)

// One obstacle move after re-posing (BatchLayout::update_transforms,
// proj/src/batch_layout.cpp:148-172), plus the obstacle's previous union box.
struct alignas(16) Event {
    double sat[21];  // kern::SatBox of the moved box
    double r;        // o_minus_r (shared sphere radius)
    double box[6];   // obstacle_aabb
    double sph[6];   // obstacle_sphere_aabb
    double nu[6];    // box U sph (new pose)
    double old[6];   // box U sph at the pose before this move (empty if inactive)
    double cen[kMaxSpheres * 3];
    rggd::Box32 b32;  // fp32 operand of sat (filter), L rounded up
    double rt[12];    // the pose (row-major rotation, translation): the exact resolve's obstacle
    int32_t o;
    int32_t nsph;
    int32_t move;  // index of the move in the batch
    int32_t pad;
};
static_assert(sizeof(Event) % 16 == 0, "Event must be 16-byte granular");

// Device-resident store (cell-sorted SoA).
struct Store {
    int32_t N;       // components in the roadmap
    int32_t Np;      // components owned by this handle (sorted order)
    int32_t B, S, M, C, W;
    int32_t cell, ncells, cap;
    int32_t use_under;
    int32_t prefetch;          // touch stages the narrow operands in L2 (they fit in half of it)
    const double2* aabb;       // 3 planes of Np double2: (minx,miny) (minz,maxx) (maxy,maxz)
    const double* sat;         // Np*B*22 (21 + pad)
    const rggd::Box32* sat32;  // Np*B fp32 filter operands of sat
    const int32_t* row;        // Np*B*S+1
    const double* seg;         // T*8 (a, d, dd, spline radius)
    const float4* seg32;       // T*2: the same record rounded to fp32 (narrow's filter operand)
    const double* spline_r;    // B*S
    const int32_t* orig;       // Np: sorted -> component id
    const double* cell_aabb;   // ncells*6
    const double* slice_aabb;  // ceil(Np/32)*6: union box of each 32-component slice (touch's event filter)
    // uniform grid over the cells (binning): bin (x, y, z) = floor((p - gorg) * ginv) clamped
    // to [0, gdim); the cells whose box overlaps bin g are gcell[gcell_off[g] .. gcell_off[g+1])
    double gorg[3], ginv[3];
    int32_t gdim[3];
    const int32_t* gcell_off;
    const int2* gcell;       // {cell, the cell's lowest bin per axis: x | y << 10 | z << 20} (the scatter's dedup)
    const double* ohe;         // M*3
    const double* osl;         // M*C*3
    const double* osr;         // M
    const int32_t* osn;        // M
    uint8_t* state;            // N labels (component-id order)
    uint8_t* state_c;          // Np labels (cell order): the apply kernels' coalesced working copy
    const int32_t* rank;       // N: component id -> cell-order index, -1 if another shard's
    uint32_t* cnt;             // Np: over_cnt | both_cnt << 16
    unsigned long long* over;  // W*Np, word-major
    unsigned long long* under; // W*Np
    Event* cur;                // M: obstacle operands at the current pose
    double* cur_union;         // M*6: box U sph of active obstacles (empty if inactive)
};

// Per-batch scratch.
struct Batch {
    int32_t n;
    const int32_t* ids;
    const double* rt;
    uint8_t* last;         // 1 if this is the obstacle's last move in this batch (pose kernel)
    Event* ev;             // n
    double* evbox;         // n*12: new and old union box of each event (compact, for the binning)
    double* evt;           // n*24: new union, old union, box, sphere box (the touch kernel's operands)
    float4* evs;           // n*kEvS: the narrow kernel's sphere operands (pose kernel): [0] = {fl(o_minus_r),
                           // sphere count (int bits), 0, 0}, [1 + k] = {fl(centre k), |fl(centre k)|_1}
    int32_t* cell_count;   // ncells
    int32_t* cell_list;    // ncells*cap
    int32_t* cell_ovf;     // ncells: base in pool when count > cap
    int32_t* pool;         // overflow pool (capacity pool_cap)
    int32_t pool_cap;
    int32_t* ctr;          // [0] dirty count, [1] pool top, [2] work counter, [3] overflow cells,
                           // [4] gray count, [5] hits count, [6] error flag, [8] over items, [9] under items
    int32_t* mv;           // n*4: to_green, to_red, to_gray, from_gray
    int32_t* hits;         // N: over-hit-by-last-move & still gray
    uint8_t* hits_prev;    // N: their labels before the move (eager report counts)
    unsigned long long* census;  // 16 counters: [0..5] narrow census, [8..11] touch census
    uint32_t* mpool;             // touch / over / under mask words (see touch_kernel)
    long long* mtop;             // next free word of mpool
    long long mpool_cap;
    int4* crec;                  // ncells: {count, mask base word, list address lo, hi} (bin kernel)
    int4* units;                 // touch work units {cell, chunk of 32 listed events, count, mask base}; ctr[10]
    int32_t units_cap;
    int4* items_over;            // {component, event, result word, bit}: pairs needing a SAT
    int4* items_under;           // same for the segment-sphere test
    int32_t items_cap;
    int4* items_recheck;         // over items the fp32 filter left undecided (count ctr[12])
    int32_t recheck_cap;
    int32_t recheck_queue;       // narrow_over queues its undecided pairs (else decides them inline)
    int32_t census_on;           // touch accumulates the byte census
    int32_t* unknown;      // running GRAY count, persistent across batches
    unsigned long long* tl;      // optional per-kernel timeline (RGG_DEBUG_TIMELINE), else null
    // host-mapped outputs (synchronous host updates): launch_host_out stores the
    // per-move counters (n*4) and ctr[0..23] there after the apply kernel
    int32_t* out_mv;
    int32_t* out_ctr;
    // host-mapped inputs (synchronous host updates): the pose kernel reads the moves
    // there and copies them to ids / rt; null when the moves are already in HBM
    const int32_t* src_ids;
    const double* src_rt;
    // split pipeline: the pose warps count the events whose binning boxes (evbox) are
    // stored, so the bin kernel starts before the pose kernel's remaining work ends;
    // the apply kernel resets it.  Null: bin waits for the whole pose kernel.
    int32_t* evready;
    // split pipeline, touch on published units: evready[1] = pose warps done,
    // evready[2] = cells binned (one count per cell's warp), evready[3] = next touch slice-unit, evready[4] =
    // update generation (never reset); bin stamps unit_ready[u] with the generation
    // once unit u and its cell list are stored.  Null: touch waits for the whole bin kernel.
    int32_t* unit_ready;
    int32_t bin_warps;
    // event bitmask per cell (bin_scatter_kernel -> bin_cells_kernel): cmask[cell * cmask_words + e / 32]
    // bit e % 32 = event e's new or old union box overlaps the cell's box; the cell pass
    // clears the words it reads, so they are zero between updates
    uint32_t* cmask;
    int32_t cmask_words;
};

// Exact resolve operands (rgg_resolve.cu).
struct __align__(16) ObsPoly {  // one obstacle as polytopes_intersect sees it
    double v[24];               // ConvexPolytope::box vertices
    double ax[9];               // face axes
    double ed[36];              // 12 edge directions
    double box[6];              // aabb_of_obb(world_outer())
    int32_t active;
    int32_t pad[3];
};

struct Resolver {
    int32_t B;               // robot bodies
    const double* he;        // B*3 body half extents
    const long long* off;    // N+1: configurations of component c are [off[c], off[c+1])
    const double* pose;      // off[N]*B*12: world pose of each body box per configuration
    ObsPoly* opoly;          // M
    const double* spose;     // M*12: scene pose of obstacles active before this engine moved them
    const uint8_t* sact;     // M: 1 = scene-active at spose (null: none)
};

cudaError_t launch_host_out(const Batch& b, cudaStream_t st);  // counters -> b.out_mv / b.out_ctr
// eager batches: save move i-1's report terms to rep[8(i-1)..], stage move i into slot 0
cudaError_t launch_eager_step(const Batch& b, int32_t* ids0, double* rt0, const int32_t* st_ids, const double* st_rt,
                              int32_t* rep, int i, int k, cudaStream_t st);

// The cell-sorted store built on the device (rgg_store.cu).  Inputs are the host
// arrays of rgg_layout_view; outputs are preallocated except `seg`.
struct StoreIn {
    int32_t N, B, S, T, np, cell, shards, shard_rank;
    const double* comp_aabb;  // N*6 (device when `device`, else host)
    const double* edge_sat;   // N*B*21 (idem)
    const int32_t* row_off;   // host N*B*S+1
    const double* segs;       // T*7 (idem)
    const double* spline;     // host B*S
    bool device = false;               // comp_aabb, edge_sat, segs are device arrays
    const int32_t* row_off_dev = nullptr;  // device copy of row_off when `device`
};
// sat_prep / component AABBs / seg_prep of raw components on the device (rgg_store.cu)
cudaError_t prep_components(const double* corners, int N, int B, const double* pts, int T, double* sat21,
                            double* aabb, double* segs7, cudaStream_t st);
struct StoreOut {
    double2* aabb;         // 3*np
    double* sat;           // np*B*22
    rggd::Box32* sat32;    // np*B
    int32_t* row;          // np*B*S+1
    double* seg;           // allocated here: total_segs*8
    float4* seg32;         // allocated here: total_segs*2
    double* spline;        // B*S
    int32_t* orig;         // np
    int32_t* rank;         // N
    double* cell_aabb;     // ncells*6
    double* slice_aabb;    // ceil(np/32)*6
    int32_t total_segs;
};
cudaError_t build_store(const StoreIn& in, StoreOut& out, cudaStream_t st);

// The binning's uniform grid over the cell boxes (Store::gorg / ginv / gdim / gcell_off / gcell).
struct CellGrid {
    double org[3], inv[3];
    int32_t dim[3];
    int32_t* off = nullptr;    // device, bins + 1
    int2* cells = nullptr;     // device: {cell, low bin packed}
    int64_t entries = 0;
};
cudaError_t build_cell_grid(const double* d_cell_aabb, int ncells, CellGrid& g, cudaStream_t st);

enum ResolveMode : int { kResolve = 0, kEager = 1, kCheck = 2 };
// exact check of ids[0..*count_dev) (max_count bounds the grid), after
// refreshing the obstacle polytopes
cudaError_t launch_resolve(const Store& s, const Resolver& r, const Batch& b, const int32_t* ids,
                           const int32_t* count_dev, int max_count, int mode, uint8_t* out, cudaStream_t st);

enum Flags : int32_t { kPerMove = 2, kHits = 8, kCensus = 16 };

cudaError_t launch_pose(const Store& s, const Batch& b, cudaStream_t st);
cudaError_t launch_bin(const Store& s, const Batch& b, cudaStream_t st);
cudaError_t launch_classify(const Store& s, const Batch& b, int flags, int grid, cudaStream_t st);
// single-move updates: one kernel tests the cells against the move's boxes, then runs touch,
// narrow and the transition per component of every hit cell
cudaError_t launch_single(const Store& s, const Batch& b, int flags, cudaStream_t st);
// host_out: also write the ids into mapped pinned host memory (capacity N)
cudaError_t launch_compact(const Store& s, int32_t* out_ids, int32_t* tile_cnt, int32_t* gray_n, cudaStream_t st,
                           int32_t* host_out = nullptr);
cudaError_t launch_write_states(const Store& s, const int32_t* ids, const uint8_t* st_in, int n, cudaStream_t st);
cudaError_t launch_pair_masks(const Store& s, const int32_t* rank, int kind, const int32_t* cand, int n, int o,
                              uint8_t* mask, cudaStream_t st);
cudaError_t launch_init_obstacles(const Store& s, Event* scratch, cudaStream_t st);
cudaError_t launch_fp64_peak(double* sink, int iters, int grid, int block, cudaStream_t st);
cudaError_t launch_fp32_peak(float* sink, int iters, int grid, int block, cudaStream_t st);
int classify_occupancy(int cell, int flags);
void filter_stats(unsigned long long* out, bool reset);

}  // namespace rggk
