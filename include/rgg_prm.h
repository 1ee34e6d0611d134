/* rgg_prm.h — C-ABI of the GPU PRM construction.
 *
 * Replaces the two halves of rgg::build_prm (proj/src/roadmap.cpp:56-102) for a
 * scene without active obstacles (the benchmark's build scene, proj/src/bench.cpp:90-91):
 *   rgg_prm_nodes      the node loop (roadmap.cpp:65-71): Rng(seed) (proj/include/rgg/rng.hpp:10-29),
 *                      dof draws per node of uniform(lo[k], hi[k]); host, sequential like mt19937_64;
 *   rgg_prm_knn_edges  the candidate loop (roadmap.cpp:73-93): the k nearest nodes of every node
 *                      under dof_distance2 (roadmap.cpp:36-43), ties by node id, as sorted unique
 *                      (min, max) pairs — the roadmap's edges when no obstacle is active (:95-101).
 * dof_bounds_for (roadmap.cpp:20-30) gives lo/hi: env then [-pi, pi]^3 for a free-flying robot,
 * [-pi, pi] per joint for a serial chain.  Lives in lib/librgg_build.so (device 0).
 * Not reentrant: one call at a time per process (the device buffers are a grow-only arena
 * reused across calls).
 */
#ifndef RGG_PRM_H
#define RGG_PRM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGG_PRM_EINVAL 1 /* std::invalid_argument in the reference (n < 1, k < 1) */
#define RGG_PRM_ECUDA 2
#define RGG_PRM_ESPACE 3 /* edges[] too small: *n_edges holds the count needed */

/* nodes: n x dof, row-major, the exact doubles build_prm samples. */
int rgg_prm_nodes(uint64_t seed, int32_t n, int32_t dof, const double* lo, const double* hi, double* nodes);
/* edges: cap x 2 int32 (first < second), sorted; cap >= n * min(k, n-1) always suffices.
 * device_ms (may be null): device time of the kNN, sort and unique (CUDA events). */
int rgg_prm_knn_edges(const double* nodes, int32_t n, int32_t dof, int32_t k, int32_t* edges, int64_t cap,
                      int64_t* n_edges, float* device_ms);
const char* rgg_prm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
