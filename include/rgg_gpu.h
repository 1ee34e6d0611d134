/* rgg_gpu.h — C-ABI of the B200-native SerRGG edge-classification engine.
 *
 * This is the drop-in boundary.  It replaces the hot path of
 *   class rgg::BatchEngine          proj/include/rgg/engine_batch.hpp:17-63
 *   rgg::BatchEngine::update_obstacle / batch_update
 *                                   proj/src/engine_batch.cpp:145-215
 * and, below it, the per-pair plugin seam
 *   struct rgg::kern::Backend       proj/include/rgg/kernels.hpp:49-54
 * which is too fine-grained for a GPU (one host call per obstacle sphere).
 * Plain pointers and sizes only; no torch or C++ types cross it.  A handle is
 * single-host-thread (updates are not reentrant, proj/include/rgg/engine_sequential.hpp:11-12).
 *
 * Errors: every entry returns RGG_OK or an RGG_E* code; rgg_gpu_last_error()
 * gives the message.  The messages of RGG_EINVAL match the reference's
 * std::invalid_argument texts ("unknown obstacle id", engine_batch.cpp:147;
 * "obstacle bitsets support at most 64 obstacles", engine_batch.cpp:27) so the
 * C++ wrapper (include/rgg/engine_gpu.hpp) can rethrow them verbatim.
 */
#ifndef RGG_GPU_H
#define RGG_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGG_OK 0
#define RGG_EINVAL 1  /* bad argument (reference: std::invalid_argument) */
#define RGG_ECUDA 2   /* CUDA runtime failure, or no sm_100 device */
#define RGG_ENCCL 3   /* collective failure (multi-GPU plumbing) */
#define RGG_ENOMEM 4  /* device allocation failed */
#define RGG_ELOGIC 5  /* layout contract violated (reference: std::logic_error) */

/* Validity labels, numerically equal to rgg::ValidityState (proj/include/rgg/roadmap.hpp:26-30). */
#define RGG_GREEN 0
#define RGG_RED 1
#define RGG_GRAY 2

/* rgg_gpu_update flags */
#define RGG_LAZY 1      /* lazy update: over-hit components stay GRAY */
#define RGG_PER_MOVE 2  /* fill one rgg_update_report per move (finish_counts semantics) */
#define RGG_ASYNC 4     /* enqueue only; the call returns before the device finishes */
#define RGG_CENSUS 8    /* also count the algorithmic bytes of this update (read by rgg_gpu_census) */
#define RGG_GRAY_LIST 16 /* compact the GRAY ids inside the update (else lazily in rgg_gpu_gray_ids) */
#define RGG_EAGER 32    /* eager update (update_obstacle(o, pose, lazy = false), engine_batch.cpp:193-200):
                           each move's GRAY over-hits are resolved exactly on the GPU before the next move.
                           Needs rgg_gpu_set_resolver; implies PER_MOVE; not ASYNC. */

/* The serialized store, borrowed for the duration of rgg_gpu_create.  It is the
 * reference's BatchLayout (proj/include/rgg/batch_layout.hpp:23-66) with the padded
 * segment block replaced by CSR over real segments:
 *   edge_sat        N*B*21   kern::SatBox rows (center[3], e[3][3], u[3][3]) — layout.edge_sat
 *   comp_aabb       N*6      component_aabb (min xyz, max xyz)
 *   row_off         N*B*S+1  real segments of row (c, b, s) are [row_off[r], row_off[r+1]),
 *                            r = (c*B + b)*S + s  (layout.seg_count as offsets)
 *   segs            T*7      kern::SegPrep rows (a[3], d[3], dd) of the real segments
 *   spline_radius   B*S      layout.spline_radius
 *   obst_he         M*3      canonical obstacle half extents (ObstacleModel::half_extents)
 *   obst_sph_local  M*C*3    inner sphere centres in the obstacle frame
 *   obst_sph_r      M        layout.o_minus_r
 *   obst_sph_n      M        layout.o_sphere_count
 */
typedef struct rgg_layout_view {
    int32_t n_components; /* N */
    int32_t n_bodies;     /* B */
    int32_t n_slots;      /* S */
    int32_t n_obstacles;  /* M */
    int32_t max_spheres;  /* C */
    const double* edge_sat;
    const double* comp_aabb;
    const int32_t* row_off;
    const double* segs;
    const double* spline_radius;
    const double* obst_he;
    const double* obst_sph_local;
    const double* obst_sph_r;
    const int32_t* obst_sph_n;
} rgg_layout_view;

/* The same store from the components themselves, without the serialized layout:
 * the engine runs the serialize step (BatchLayout::serialize, batch_layout.cpp:55-146:
 * sat_prep of the corners, component AABBs, seg_prep of the real segments) on the
 * device.  A caller that never needs the padded host layout (12x the real segments
 * at c2) never builds it.
 *   obb_corners     N*B*24   obb_corners(components.geometry[c].over[b]) (batch_layout.cpp:10-17)
 *   row_off         N*B*S+1  real segments of row (c, b, s), as in rgg_layout_view
 *   seg_points      T*6      each real segment's end points (a, b); a single-point spline is
 *                            one degenerate segment (a, a) (batch_layout.cpp:84-90)
 *   spline_radius .. obst_sph_n: as in rgg_layout_view */
typedef struct rgg_component_view {
    int32_t n_components, n_bodies, n_slots, n_obstacles, max_spheres;
    const double* obb_corners;
    const int32_t* row_off;
    const double* seg_points;
    const double* spline_radius;
    const double* obst_he;
    const double* obst_sph_local;
    const double* obst_sph_r;
    const int32_t* obst_sph_n;
} rgg_component_view;

typedef struct rgg_gpu_options {
    int32_t device;        /* CUDA ordinal (one process per GPU) */
    int32_t use_under;     /* EngineOptions::use_under (update_report.hpp:43-46) */
    int32_t cell_size;     /* components per cell (0 -> 128; a multiple of 32, <= 128) */
    int32_t cell_capacity; /* inline event slots per cell before overflow (0 -> 64) */
    int32_t allow_wide;    /* accept M > 64 (bitsets become ceil(M/64) words) */
    int32_t shard_rank;    /* this handle owns cells c with c % shard_count == shard_rank */
    int32_t shard_count;   /* 0 or 1: unsharded */
} rgg_gpu_options;

/* Mirrors rgg::UpdateReport (proj/include/rgg/update_report.hpp:11-25).  With
 * phase timing on (rgg_gpu_set_phase_timing), the *_us fields carry
 * device-event microseconds of the batch split into the phases of this engine
 * (pose -> reval_us, binning -> over_us, classify -> under_us, compaction ->
 * resolve_us), on the last report of a batch only; otherwise they are 0. */
typedef struct rgg_update_report {
    int32_t obstacle;
    int32_t new_green;
    int32_t new_red;
    int32_t new_gray;
    int64_t reval_us;
    int64_t over_us;
    int64_t under_us;
    int64_t resolve_us;
    int32_t unknown_after_heuristic;
    int32_t residual_unknown;
    int32_t resolve_checks;
    int32_t _pad;
} rgg_update_report;

typedef struct rgg_gpu rgg_gpu;

/* BatchEngine::BatchEngine (engine_batch.cpp:20-31): uploads the store into
 * HBM (cell-sorted SoA), builds the cells, all labels GREEN, bits 0. */
int rgg_gpu_create(const rgg_layout_view* view, const rgg_gpu_options* opts, rgg_gpu** out);
/* rgg_gpu_create from raw components (rgg_component_view): same engine, same results. */
int rgg_gpu_create_from_components(const rgg_component_view* view, const rgg_gpu_options* opts, rgg_gpu** out);
void rgg_gpu_destroy(rgg_gpu* h);
const char* rgg_gpu_last_error(const rgg_gpu* h);

/* BatchEngine::batch_update (engine_batch.cpp:207-215) over n moves
 * (ids[i], pose rt12[12*i .. 12*i+11] = row-major rotation then translation).
 * Moves are applied in order; labels after the call equal the reference's after
 * the same moves.  reports (n entries, PER_MOVE) or NULL.  On an unknown id at
 * position k, moves [0, k) are applied and RGG_EINVAL is returned. */
int rgg_gpu_update(rgg_gpu* h, const int32_t* ids, const double* rt12, int32_t n, int32_t flags,
                   rgg_update_report* reports);
/* Same, with ids/rt12 already in device memory (no host copies); always async.
 * The host-side id validation is skipped: ids must be in [0, M). */
int rgg_gpu_update_device(rgg_gpu* h, const int32_t* d_ids, const double* d_rt12, int32_t n, int32_t flags);
/* The engine's pinned staging buffers for a batch of up to n moves (ids n, rt12 n*12): a
 * caller that writes its moves there and passes these pointers to rgg_gpu_update skips the
 * host copy into them (the update's host-to-device copy reads them directly).  Valid until
 * a later call grows them (a larger batch). */
int rgg_gpu_stage(rgg_gpu* h, int32_t n, int32_t** ids, double** rt12);
int rgg_gpu_sync(rgg_gpu* h);
/* Device-to-device copy (on the engine stream) of the last update's per-move
 * counters, n x {to_green, to_red, to_gray, from_gray} int32 — the per-shard
 * report terms a multi-GPU driver sums with one all-reduce. */
int rgg_gpu_copy_counters(rgg_gpu* h, void* dst_device, int32_t n);
/* Per-kernel phase events in rgg_gpu_last_stats and the reports' *_us fields
 * (default off).  Each event record between two kernels costs ~5 us of device
 * idle time and breaks their PDL overlap; off, only total_ms is filled. */
int rgg_gpu_set_phase_timing(rgg_gpu* h, int32_t on);

int rgg_gpu_count(const rgg_gpu* h, int32_t* n_components, int32_t* n_obstacles, int32_t* words_per_comp);
/* states(): N labels in component-id order (sharded handles: unowned entries are 0xFF). */
int rgg_gpu_read_states(rgg_gpu* h, uint8_t* out);
/* obstacle_bits(): N * words, component-major; word w holds obstacles [64w, 64w+64). */
int rgg_gpu_read_bits(rgg_gpu* h, uint64_t* out, int32_t words_per_comp);
int rgg_gpu_unknown_count(rgg_gpu* h, int32_t* out);
/* Ascending ids of every GRAY component (the gray list handed to the exact resolve). */
int rgg_gpu_gray_ids(rgg_gpu* h, int32_t* out, int32_t cap, int32_t* n);
/* The same list left in DEVICE memory, enqueued on the handle's stream without a host
 * wait (multi-GPU gather): the GRAY count into d_count (int32, may be null) and the
 * first cap ids into d_ids (entries past the count are unspecified).  Compacts the
 * current labels first unless the last update ran with RGG_GRAY_LIST. */
int rgg_gpu_gray_device(rgg_gpu* h, int32_t* d_count, int32_t* d_ids, int32_t cap);
/* The same list copied into a handle-owned pinned host buffer (one DMA, no staging):
 * *ids points at n ascending ids, valid until the next call on this handle. */
int rgg_gpu_gray_view(rgg_gpu* h, const int32_t** ids, int32_t* n);
/* Components over-hit by the last move of the last update that are still GRAY
 * (the over_hits the reference resolves in eager mode, engine_batch.cpp:193-200). */
int rgg_gpu_last_hits(rgg_gpu* h, int32_t* out, int32_t cap, int32_t* n);
/* Eager / resolve_all_unknown write-back: states[ids[i]] = st[i] (bits untouched). */
int rgg_gpu_write_states(rgg_gpu* h, const int32_t* ids, const uint8_t* st, int32_t n);
/* Exact resolve on the GPU (exact_component_valid, proj/src/roadmap.cpp:129-163).
 * The forward kinematics of every discretized configuration (robot.cpp:66-84) is
 * evaluated on the host once and uploaded: for component c (id order), its
 * configurations are [pose_off[c], pose_off[c+1]), and configuration k's body b
 * has the world pose poses[(k*B + b)*12 ..] (row-major rotation r[9], then t[3]),
 * i.e. forward_kinematics(robot, cfgs[c][j])[b].  Obstacles are exact-checked at
 * the poses this engine's moves gave them (active after their first move), plus
 * those rgg_gpu_set_active_obstacles lists (active in the Scene before). */
typedef struct rgg_resolve_view {
    int32_t n_components;           /* N */
    int32_t n_bodies;               /* B (the layout's) */
    const double* body_half_extents; /* B*3 */
    const int64_t* pose_off;        /* N+1 */
    const double* poses;            /* pose_off[N]*B*12 */
} rgg_resolve_view;
int rgg_gpu_set_resolver(rgg_gpu* h, const rgg_resolve_view* view);
/* The Scene's obstacles that are active before this engine moves them
 * (ObstacleModel::active + pose, proj/include/rgg/swept.hpp:43, read by
 * exact_component_valid at proj/src/roadmap.cpp:135-139).  Replaces the previous
 * list; rt = n poses of 12 doubles (r[9] row-major, t[3]); a repeated id keeps its
 * last pose.  An obstacle's own moves supersede its listed pose.  Only the exact
 * resolve reads the list: the reference's BatchEngine labels and bits do not
 * depend on obstacles it has not moved (engine_batch.cpp:145-215). */
int rgg_gpu_set_active_obstacles(rgg_gpu* h, const int32_t* ids, const double* rt, int32_t n);
/* exact_component_valid (proj/src/roadmap.cpp:129-163) of n_sets independent
 * configuration sets, without an engine: the node and edge checks of build_prm
 * (roadmap.cpp:69, :95-99; proj/src/roadmap.cpp:47-52 component_collides is its
 * negation).  Set i's configurations are [cfg_off[i], cfg_off[i+1]); poses holds
 * per configuration, per body, 12 doubles (r[9], t[3]) = forward_kinematics; the
 * n_obst obstacles are the Scene's active ones (half extents, pose rt[12]).
 * free_out[i] = 1 if set i is free.  Stateless; runs on `device`. */
int rgg_exact_valid_sets(int32_t device, int32_t n_sets, const int64_t* cfg_off, int32_t n_bodies,
                         const double* body_he, const double* poses, int32_t n_obst, const double* obst_he,
                         const double* obst_rt, uint8_t* free_out);
/* resolve_all_unknown (engine_batch.cpp:217-227): every GRAY component becomes
 * GREEN (free) or RED; *resolved = how many were GRAY. */
int rgg_gpu_resolve_all(rgg_gpu* h, int32_t* resolved);
/* exact_component_valid of ids[0..n) at the current obstacle poses, without
 * changing any label: out[i] = RGG_GREEN (free) or RGG_RED. */
int rgg_gpu_exact_check(rgg_gpu* h, const int32_t* ids, int32_t n, uint8_t* out);

/* batch_over (kind 0) / batch_under (kind 1) on explicit candidates against
 * obstacle o at its current pose (engine_batch.hpp:34-37). */
int rgg_gpu_pair_masks(rgg_gpu* h, int32_t kind, const int32_t* cand, int32_t n, int32_t o, uint8_t* mask);

/* Measurement hooks (bench.py): device time of the last update's phases and the
 * algorithmic census of the current poses. */
typedef struct rgg_gpu_stats {
    float pose_ms, bin_ms, classify_ms, compact_ms, total_ms;
    int32_t dirty_cells, events, overflow_cells;
    int64_t over_pairs, sat_flops, under_pairs, seg_sphere_tests, over_hits;
    int64_t under_hits;       /* (pair, segment) items with a hit */
    int64_t bytes_components; /* algorithmic bytes of the dirty components, fp64 records */
    int64_t bytes_fp32;       /* algorithmic bytes in SURVEY.md §8(d)'s fp32 model */
    int64_t gray;             /* GRAY components after the update */
} rgg_gpu_stats;
int rgg_gpu_last_stats(rgg_gpu* h, rgg_gpu_stats* out);
/* Full-roadmap census against all active obstacles (one untimed launch). */
int rgg_gpu_census(rgg_gpu* h, rgg_gpu_stats* out);
/* Pairs the fp32 filters could not decide and the exact fp64 sequence re-tested
 * (SAT, segment-sphere), summed over every handle of this process since the last
 * reset.  The verdicts are exact either way; this is the filters' "epsilon band". */
int rgg_gpu_filter_stats(rgg_gpu* h, int64_t* sat_rechecks, int64_t* seg_rechecks, int32_t reset);
/* The CUDA stream the engine launches on (cudaStream_t), for event timing. */
void* rgg_gpu_stream(rgg_gpu* h);
/* Measured non-FMA fp64 add/mul rate of `device` in GFLOP/s (the compute roof
 * of the fp64-exact classification). */
int rgg_gpu_fp64_peak(int device, double* gflops);
/* Measured FP32 FMA rate of `device` in GFLOP/s (2 flops per FFMA): the compute roof
 * the north star states for the geometric tests. */
int rgg_gpu_fp32_peak(int device, double* gflops);
/* Components this handle owns (its shard of the roadmap; N when unsharded). */
int rgg_gpu_owned(const rgg_gpu* h, int32_t* n_owned);

#ifdef __cplusplus
}
#endif
#endif
