/* rgg_build.h — C-ABI of the host-side roadmap producer (CPU, multithreaded).
 *
 * Produces the serialized store consumed by rgg_gpu_create (include/rgg_gpu.h)
 * from a roadmap of a free-flying box robot or a serial chain, following the reference's
 * preprocessing so the inputs have the reference's shapes:
 *   discretize_edge        proj/src/robot.cpp:39-64
 *   forward_kinematics     proj/src/robot.cpp:66-84 (free-flying and serial-chain branches)
 *   build_outer_approx     proj/src/swept.cpp:100-118 + obb_from_points geometry.cpp:134-195
 *   build_inner_approx     proj/src/swept.cpp:188-228 (+ simplify :79-92, cap_segments :125-162)
 *   build_components       proj/src/roadmap.cpp:104-127 (nodes first, then edges)
 *   BatchLayout::serialize proj/src/batch_layout.cpp:21-146 (slots, SatBox, CSR of real segments)
 * It is the step before the hot path, not part of it.
 */
#ifndef RGG_BUILD_H
#define RGG_BUILD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rgg_built rgg_built;

/* nodes: n_nodes x 6 DOFs (x, y, z, rx, ry, rz — fixed-axis XYZ Euler); edges: n_edges x 2.
 * threads <= 0: hardware concurrency.  Returns 0, or -1 (see rgg_build_last_error). */
int rgg_build_layout(const double* robot_he3, int32_t n_nodes, const double* nodes, int32_t n_edges,
                     const int32_t* edges, double eps, int32_t max_segments, int32_t threads, rgg_built** out);
/* Same, with flags: RGG_BUILD_POSES keeps forward_kinematics of every discretized
 * configuration for the GPU exact resolve (rgg_gpu_set_resolver, include/rgg_gpu.h). */
#define RGG_BUILD_POSES 1
/* fit the swept-volume boxes (obb_from_points) on the GPU, bit-identical (the calling thread's
 * current CUDA device) */
#define RGG_BUILD_GPU_FIT 2
/* also the inner approximation (spline simplification) on the GPU, bit-identical (same device);
 * slower end to end than RGG_BUILD_GPU_FIT alone while serialize stays on the host */
#define RGG_BUILD_GPU_INNER 4
/* keep the robot, the roadmap and the swept-volume geometry for rgg_built_save_roadmap */
#define RGG_BUILD_KEEP_GEOMETRY 8
int rgg_build_layout_ex(const double* robot_he3, int32_t n_nodes, const double* nodes, int32_t n_edges,
                        const int32_t* edges, double eps, int32_t max_segments, int32_t threads, int32_t flags,
                        rgg_built** out);
/* Any robot of the reference (RobotModel, proj/include/rgg/robot.hpp:13-58): free flying
 * (6 DOFs: x, y, z, rx, ry, rz; every body rides the one world frame) or a serial chain
 * (one revolute joint per body: DOF j is joint j's angle).  Its inner spheres are
 * default_body_spheres (proj/src/swept.cpp:52-65), as in the reference's scenarios. */
#define RGG_ROBOT_FREE_FLYING 0
#define RGG_ROBOT_SERIAL_CHAIN 1
typedef struct {
    int32_t kinematics;          /* RGG_ROBOT_FREE_FLYING or RGG_ROBOT_SERIAL_CHAIN */
    int32_t n_bodies;            /* >= 1 (<= 64 for a chain) */
    const double* half_extents;  /* n_bodies x 3, positive */
    const double* local;         /* n_bodies x 12 (r[9] row-major, t[3]) body frames; NULL = identity */
    const double* joint_axis;    /* serial chain: n_bodies x 3, nonzero */
    const double* joint_offset;  /* serial chain: n_bodies x 3, translation from the parent joint frame */
} rgg_robot_view;
/* rgg_build_layout_ex for any robot: nodes n_nodes x dof (6, or n_bodies for a chain).
 * The layout has B = n_bodies SatBoxes per component (body-minor) and B*S slots.
 * RGG_BUILD_GPU_FIT fits every (component, body) box on the GPU; RGG_BUILD_GPU_INNER
 * takes single-body robots only. */
int rgg_build_layout_robot(const rgg_robot_view* robot, int32_t n_nodes, const double* nodes, int32_t n_edges,
                           const int32_t* edges, double eps, int32_t max_segments, int32_t threads, int32_t flags,
                           rgg_built** out);
/* The kept poses: *n_configs = pose_off[N]; pose_off N+1; poses n_configs*B*12 (r[9], t[3];
 * body-minor per configuration).
 * Any pointer may be null. */
int rgg_built_poses(const rgg_built* b, int64_t* n_configs, int64_t* pose_off, double* poses);
/* out[0..3] = N, B, S, T (real segments) */
int rgg_built_counts(const rgg_built* b, int64_t* out);
/* Any pointer may be null.  edge_sat N*B*21, comp_aabb N*6, row_off N*B*S+1, segs T*7,
 * spline_r B*S, obb15 N*B*15 (centre, axes[3][3], half extents). */
int rgg_built_export(const rgg_built* b, double* edge_sat, double* comp_aabb, int32_t* row_off, double* segs,
                     double* spline_r, double* obb15);
void rgg_built_free(rgg_built* b);
/* save_roadmap (proj/src/roadmap_io.cpp:150-203) of a build made with RGG_BUILD_KEEP_GEOMETRY:
 * the reference's binary roadmap file, which its load_roadmap reads (and rgg_roadmap_load). */
int rgg_built_save_roadmap(const rgg_built* b, const char* path);
const char* rgg_build_last_error(void);
/* CUDA devices visible to the producer (0 without a GPU): the GPU box fit
 * (RGG_BUILD_GPU_FIT) is the Python producer's default when this is positive. */
int rgg_build_gpu_count(void);
/* The reference's binary roadmap file (save_roadmap / load_roadmap, proj/src/roadmap_io.cpp:150-301:
 * magic "RGGRDMP1", version 1, little-endian sections, a CRC-32 of the whole file), read and fully
 * verified before anything is built, straight into the component view of
 * rgg_gpu_create_from_components (include/rgg_gpu.h): no ComponentSet and no padded layout.
 * Returns 0, one of the error kinds below (RoadmapIoError, roadmap_io.hpp:10-16), or -1 (an
 * inconsistent file, e.g. an inconsistent slot radius); rgg_build_last_error has the text. */
#define RGG_ROADMAP_BAD_MAGIC 1
#define RGG_ROADMAP_BAD_VERSION 2
#define RGG_ROADMAP_TRUNCATED 3
#define RGG_ROADMAP_CHECKSUM 4
typedef struct rgg_roadmap_file rgg_roadmap_file;
int rgg_roadmap_load(const char* path, rgg_roadmap_file** out);
/* out[0..8] = n_nodes, n_edges, dof, N (components), B, S, T (real segments), kinematics, max_segments */
int rgg_roadmap_counts(const rgg_roadmap_file* f, int64_t* out);
/* the component view's arrays: obb_corners N*B*24, row_off N*B*S+1, seg_points T*6, spline_radius B*S
 * (any pointer may be null) */
int rgg_roadmap_components(const rgg_roadmap_file* f, double* obb_corners, int32_t* row_off, double* seg_points,
                           double* spline_radius);
/* the roadmap: nodes n_nodes*dof, edges n_edges*2, and the discretization resolution */
int rgg_roadmap_graph(const rgg_roadmap_file* f, double* nodes, int32_t* edges, double* eps);
/* the robot (rgg_robot_view's arrays): half extents B*3, local frames B*12, joint axes / offsets B*3 (chains) */
int rgg_roadmap_robot(const rgg_roadmap_file* f, double* he, double* local12, double* axis, double* offset);
/* the exact resolve's inputs (rgg_resolve_view): *n_configs, pose_off N+1, poses n_configs*B*12 (pass
 * poses = NULL to size them) */
int rgg_roadmap_poses(const rgg_roadmap_file* f, int64_t* n_configs, int64_t* pose_off, double* poses);
void rgg_roadmap_free(rgg_roadmap_file* f);
/* obstacle_inner_spheres (proj/src/swept.cpp:23-49): count centres (count*3) and the radius. */
int rgg_obstacle_spheres(const double* he3, int32_t count, double* centres, double* radius);

#ifdef __cplusplus
}
#endif
#endif
