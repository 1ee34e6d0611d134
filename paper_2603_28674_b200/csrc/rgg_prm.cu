// rgg_prm.cu — PRM construction on the GPU.
//
// build_prm (proj/src/roadmap.cpp:56-102) for scenes without active obstacles:
//   * nodes: Rng(seed) draws dof uniforms per node, Rng::uniform = lo + (hi-lo)*unit()
//     with unit() = (mt19937_64() >> 11) * 2^-53 (proj/include/rgg/rng.hpp:10-29);
//     sequential by nature, so it stays on the host (n*dof draws);
//   * candidates: for every node i the k smallest (dof_distance2(node_i, node_j), j),
//     j != i, in pair order (std::partial_sort of pair<double, NodeId>, :78-90), where
//     dof_distance2 sums (b[k]-a[k])^2 in DOF order without contraction (:36-43);
//     then the (min, max) pairs sorted and made unique (:91-93).
// The reference's O(n^2) scan is the cost ("the O(n^2) kNN makes
// 1M-edge inputs slow to build").  Here (dof <= 8):
//   1. the nodes are sorted by the Morton code of their first three coordinates and
//      cut into tiles of 128; each tile and each CTA's row group gets its fp64 box;
//   2. one thread per query node keeps its k best (distance, id) in a shared-memory
//      insertion list, ordered by (distance, id) exactly as pair<double, NodeId>;
//      a CTA visits the tiles outward from its own in Morton order (the lists fill
//      with near nodes first) and skips a tile when the fp64 lower bound of the
//      distance between the two boxes — the reference's own operation sequence on
//      the per-axis gaps, which is monotone — exceeds every row's k-th distance;
//   3. a candidate's fp32 distance, against a rigorous bound (filter_bound), rejects
//      almost every non-neighbour; the rest get the reference's fp64 sum.
// Distances, ties and the resulting sets are the reference's bit for bit; only the
// work skipped differs.  dof > 8: a plain scan over all nodes in id order, split
// over CTAs for small n and merged.  Sorting and uniquing the (min, max) keys is
// CUB's radix sort + unique.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rgg_prm.h"

namespace {

thread_local std::string g_prm_err;

constexpr int kTile = 128;     // candidate nodes staged per pass (= rows per CTA of the tiled kernel)
constexpr int kMaxDof = 32;    // generic path bound
constexpr int kMaxK = 512;     // neighbours kept per node

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// d2 = sum over k of (b[k]-a[k])^2, left to right, each product and sum rounded
// (dof_distance2, roadmap.cpp:36-43); 0.0 + x == x for the first term (x >= +0).
template <int DOF>
__device__ __forceinline__ double dist2(const double* xi, const double* tile, int q, int dof) {
    const int D = DOF > 0 ? DOF : dof;
    double d = __dsub_rn(tile[q], xi[0]);
    double s = __dmul_rn(d, d);
#pragma unroll
    for (int k = 1; k < (DOF > 0 ? DOF : kMaxDof); ++k) {
        if (DOF == 0 && k >= D) break;
        d = __dsub_rn(tile[k * kTile + q], xi[k]);
        s = __dadd_rn(s, __dmul_rn(d, d));
    }
    return s;
}

// The fp32 pre-filter's threshold.  For a pair with exact difference D (real), the
// fp64 sum s64 >= |D|^2 (1 - 2^-45) (dof <= 32 roundings of 2^-53), so s64 < thr
// implies |D| < R = sqrt(thr / (1 - 2^-45)).  The fp32 operands are the coordinates
// rounded to nearest (|x32 - x| <= u|x|, u = 2^-24), so the fp32 difference d32
// has |d32 - D| <= u|D| + 2u(1+u)M_q (M_q = max |coordinate q|), and
// |d32| <= (1+u)|D| + E with E = 2u(1+u)|M| (host).  The fp32 sum of squares (one
// rounding per product / fused multiply-add) is <= |d32|^2 (1+u)^dof.  Hence
// s64 < thr  =>  s32 <= T32 = ((1+u)R + E)^2 (1+u)^dof, rounded up with a 2^-40
// margin for the fp64 evaluation of this bound: a pair with s32 > T32 cannot enter
// the list, and every other pair is decided by the exact fp64 sum.
__device__ __forceinline__ float filter_bound(double thr, double E, int dof) {
    if (!(thr < INFINITY)) return INFINITY;
    const double u = 0x1p-24;
    const double R = sqrt(thr / (1.0 - 0x1p-45)) * (1.0 + 0x1p-50);
    const double r = R * (1.0 + u) + E;
    double t = r * r;
    for (int q = 0; q < dof; ++q) t *= 1.0 + u;
    return __double2float_ru(t * (1.0 + 0x1p-40));
}

// Generic scan (dof > 8): CTA (x, y) = query rows [x*T, x*T+T) against candidates
// [y*span, (y+1)*span) in id order.  Output list t of row i at out[(y*k + t)*n + i]
// (sorted; unused slots d = +inf, j = INT32_MAX).
__global__ void __launch_bounds__(128) knn_scan_kernel(const double* __restrict__ X, int n, int dof, int k, int span,
                                                       double* __restrict__ out_d, int32_t* __restrict__ out_j) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int T = blockDim.x, tid = threadIdx.x;
    double* tile = reinterpret_cast<double*>(smem);                               // [dof][kTile]
    double* bd = tile + static_cast<size_t>(dof) * kTile;                         // [k][T]
    int32_t* bj = reinterpret_cast<int32_t*>(bd + static_cast<size_t>(k) * T);    // [k][T]
    const int i = blockIdx.x * T + tid;
    const bool live = i < n;
    double xi[kMaxDof];
    for (int q = 0; q < dof; ++q) xi[q] = live ? X[static_cast<size_t>(q) * n + i] : 0.0;
    int cnt = 0;
    double thr = INFINITY;
    const int j0 = blockIdx.y * span, j1 = min(n, j0 + span);
    for (int jb = j0; jb < j1; jb += kTile) {
        const int m = min(kTile, j1 - jb);
        __syncthreads();
        for (int t = tid; t < dof * kTile; t += T) {
            const int q = t % kTile, dd = t / kTile;
            tile[t] = q < m ? X[static_cast<size_t>(dd) * n + jb + q] : 0.0;
        }
        __syncthreads();
        if (!live) continue;
        for (int q = 0; q < m; ++q) {
            const double s = dist2<0>(xi, tile, q, dof);
            const int j = jb + q;
            if (s < thr && j != i) {  // candidates arrive in increasing j: ties keep the earlier j
                int p = cnt < k ? cnt : k - 1;
                while (p > 0 && bd[(p - 1) * T + tid] > s) {
                    bd[p * T + tid] = bd[(p - 1) * T + tid];
                    bj[p * T + tid] = bj[(p - 1) * T + tid];
                    --p;
                }
                bd[p * T + tid] = s;
                bj[p * T + tid] = j;
                if (cnt < k) ++cnt;
                if (cnt == k) thr = bd[(k - 1) * T + tid];
            }
        }
    }
    if (!live) return;
    for (int t = 0; t < k; ++t) {
        const size_t o = (static_cast<size_t>(blockIdx.y) * k + t) * n + i;
        out_d[o] = t < cnt ? bd[t * T + tid] : INFINITY;
        out_j[o] = t < cnt ? bj[t * T + tid] : INT32_MAX;
    }
}

// fp64 lower bound of dof_distance2 over two boxes (lo[q], hi[q] at b[q], b[DOF+q]):
// per axis the gap g_q (0 if the ranges overlap) satisfies |fl(xj - xi)| >= fl(g_q)
// for every pair of points (rounding is monotone), so the reference's sum of
// rounded squares over the pair is >= the same sum over the gaps.
template <int DOF>
__device__ __forceinline__ double box_lower_bound(const double* __restrict__ a, const double* __restrict__ b) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < DOF; ++q) {
        const double g1 = __dsub_rn(b[q], a[DOF + q]), g2 = __dsub_rn(a[q], b[DOF + q]);
        const double g = g1 > 0.0 ? g1 : (g2 > 0.0 ? g2 : 0.0);
        s = q == 0 ? __dmul_rn(g, g) : __dadd_rn(s, __dmul_rn(g, g));
    }
    return s;
}

// Tiled kNN (dof <= 8) over the Morton-sorted nodes: XS [DOF][n] fp64, X32 n x 8
// fp32, ids (sorted position -> node id), boxes [tiles][2*DOF] of the candidate
// tiles (kTile sorted nodes each).  A CTA of R = blockDim.x threads owns the R
// sorted rows [x*R, x*R+R).  Phase A visits the tile holding those rows and its two
// Morton neighbours, which fills every list with near nodes; phase B then bounds
// every tile against the row group's box in parallel, keeps those whose bound does
// not exceed the group's largest k-th distance, and visits them (re-checking the
// bound as the lists tighten).  Writes the row's sorted list at out[t*n + id].
// E < 0 disables the fp32 filter.
constexpr int kListCap = 1024;  // phase-B survivors per chunk of tiles

template <int DOF>
__global__ void __launch_bounds__(128) knn_tiled_kernel(const double* __restrict__ XS, const float4* __restrict__ X32,
                                                        const int32_t* __restrict__ ids,
                                                        const double* __restrict__ boxes, int n, int k, double E,
                                                        double* __restrict__ out_d, int32_t* __restrict__ out_j,
                                                        unsigned long long* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_red[4][2 * DOF];
    __shared__ double s_rbox[2 * DOF];
    __shared__ double s_bmax[4];
    __shared__ int32_t s_ids[kTile];
    __shared__ int32_t s_list[kListCap];
    __shared__ float s_lb[kListCap];
    __shared__ int s_nlist;
    const int R = blockDim.x, nw = R >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float4* t32 = reinterpret_cast<float4*>(smem);                            // [kTile][2]
    double* tile = reinterpret_cast<double*>(smem + kTile * 32);               // [DOF][kTile]
    double* bd = tile + DOF * kTile;                                           // [k][R]
    int32_t* bj = reinterpret_cast<int32_t*>(bd + static_cast<size_t>(k) * R);  // [k][R]
    const int ntiles = (n + kTile - 1) / kTile;
    const int pos = blockIdx.x * R + tid;
    const bool live = pos < n;
    const int me = live ? ids[pos] : -1;
    const int home = (blockIdx.x * R) / kTile;
    double xi[DOF];
    float xf[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < DOF; ++q) xi[q] = live ? XS[static_cast<size_t>(q) * n + pos] : 0.0;
    if (live) {
        const float4 a = X32[2 * static_cast<size_t>(pos)], b = X32[2 * static_cast<size_t>(pos) + 1];
        xf[0] = a.x, xf[1] = a.y, xf[2] = a.z, xf[3] = a.w, xf[4] = b.x, xf[5] = b.y, xf[6] = b.z, xf[7] = b.w;
    }
    // the row group's box
#pragma unroll
    for (int q = 0; q < DOF; ++q) {
        double lo = live ? xi[q] : INFINITY, hi = live ? xi[q] : -INFINITY;
        for (int o = 16; o; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) s_red[warp][q] = lo, s_red[warp][DOF + q] = hi;
    }
    __syncthreads();
    if (tid < DOF) {
        double lo = s_red[0][tid], hi = s_red[0][DOF + tid];
        for (int w = 1; w < nw; ++w) lo = fmin(lo, s_red[w][tid]), hi = fmax(hi, s_red[w][DOF + tid]);
        s_rbox[tid] = lo;
        s_rbox[DOF + tid] = hi;
    }
    const bool use_filter = E >= 0.0;
    int cnt = 0;
    double thr = INFINITY;
    int32_t thr_j = INT32_MAX;
    float t32max = INFINITY;
    unsigned long long visited = 0;

    // block-wide largest k-th distance (every thread calls; ends with a barrier)
    auto group_max = [&]() -> double {
        double mx = live ? thr : -INFINITY;
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        __syncthreads();
        if (lane == 0) s_bmax[warp] = mx;
        __syncthreads();
        double b = s_bmax[0];
        for (int w = 1; w < nw; ++w) b = fmax(b, s_bmax[w]);
        return b;
    };
    // stage tile tt and test it against every live row (block-uniform call)
    auto visit = [&](int tt) {
        __syncthreads();  // the previous tile's operands are no longer read
        const int jb = tt * kTile, m = min(kTile, n - jb);
        for (int t = tid; t < kTile; t += R) {
#pragma unroll
            for (int q = 0; q < DOF; ++q) tile[q * kTile + t] = t < m ? XS[static_cast<size_t>(q) * n + jb + t] : 0.0;
            s_ids[t] = t < m ? ids[jb + t] : -1;
        }
        for (int t = tid; t < 2 * kTile; t += R)
            t32[t] = t < 2 * m ? X32[2 * static_cast<size_t>(jb) + t] : make_float4(0, 0, 0, 0);
        __syncthreads();
        ++visited;
        if (!live) return;
        for (int q = 0; q < m; ++q) {
            if (use_filter) {
                const float4 a = t32[2 * q];
                float d = __fsub_rn(a.x, xf[0]);
                float s = __fmul_rn(d, d);
                if (DOF > 1) d = __fsub_rn(a.y, xf[1]), s = __fmaf_rn(d, d, s);
                if (DOF > 2) d = __fsub_rn(a.z, xf[2]), s = __fmaf_rn(d, d, s);
                if (DOF > 3) d = __fsub_rn(a.w, xf[3]), s = __fmaf_rn(d, d, s);
                if (DOF > 4) {
                    const float4 b = t32[2 * q + 1];
                    d = __fsub_rn(b.x, xf[4]), s = __fmaf_rn(d, d, s);
                    if (DOF > 5) d = __fsub_rn(b.y, xf[5]), s = __fmaf_rn(d, d, s);
                    if (DOF > 6) d = __fsub_rn(b.z, xf[6]), s = __fmaf_rn(d, d, s);
                    if (DOF > 7) d = __fsub_rn(b.w, xf[7]), s = __fmaf_rn(d, d, s);
                }
                if (s > t32max) continue;  // cannot enter the list (filter_bound)
            }
            const double s = dist2<DOF>(xi, tile, q, DOF);
            const int32_t j = s_ids[q];
            // pair<double, NodeId> order: (s, j) < (thr, thr_j)
            if ((s < thr || (s == thr && j < thr_j)) && j != me) {
                int p = cnt < k ? cnt : k - 1;
                while (p > 0) {
                    const double pd = bd[(p - 1) * R + tid];
                    if (!(pd > s || (pd == s && bj[(p - 1) * R + tid] > j))) break;
                    bd[p * R + tid] = pd;
                    bj[p * R + tid] = bj[(p - 1) * R + tid];
                    --p;
                }
                bd[p * R + tid] = s;
                bj[p * R + tid] = j;
                if (cnt < k) ++cnt;
                if (cnt == k) {
                    const double nt = bd[(k - 1) * R + tid];
                    thr_j = bj[(k - 1) * R + tid];
                    if (use_filter && nt != thr) t32max = filter_bound(nt, E, DOF);
                    thr = nt;
                }
            }
        }
    };

    // phase A: the home tile and its Morton neighbours
    const int a0 = max(0, home - 1), a1 = min(ntiles - 1, home + 1);
    for (int tt = a0; tt <= a1; ++tt) visit(tt);
    // phase B: every other tile whose box bound does not exceed the group's k-th distance
    for (int c0 = 0; c0 < ntiles; c0 += kListCap) {
        double bmax = group_max();
        if (tid == 0) s_nlist = 0;
        __syncthreads();
        double rb[2 * DOF];
#pragma unroll
        for (int q = 0; q < 2 * DOF; ++q) rb[q] = s_rbox[q];
        for (int tt = c0 + tid; tt < min(ntiles, c0 + kListCap); tt += R) {
            if (tt >= a0 && tt <= a1) continue;
            const double lb = box_lower_bound<DOF>(rb, boxes + static_cast<size_t>(tt) * 2 * DOF);
            if (lb > bmax) continue;
            const int at = atomicAdd(&s_nlist, 1);
            s_list[at] = tt;
            s_lb[at] = __double2float_rd(lb);  // <= lb: a valid (weaker) bound for the re-check
        }
        __syncthreads();
        const int nl = s_nlist;
        for (int e = 0; e < nl; ++e) {
            bmax = group_max();
            if (s_lb[e] > bmax) continue;  // block-uniform
            visit(s_list[e]);
        }
        __syncthreads();
    }
    if (stats && tid == 0) atomicAdd(stats, visited);
    if (!live) return;
    for (int t = 0; t < k; ++t) {
        const size_t o = static_cast<size_t>(t) * n + me;
        out_d[o] = t < cnt ? bd[t * R + tid] : INFINITY;
        out_j[o] = t < cnt ? bj[t * R + tid] : INT32_MAX;
    }
}

// Row-major n x dof -> SoA [dof][n] (fp64), for the generic scan.
__global__ void soa_kernel(const double* __restrict__ rows, int n, int dof, double* __restrict__ X) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int q = 0; q < dof; ++q) X[static_cast<size_t>(q) * n + i] = rows[static_cast<size_t>(i) * dof + q];
}

__device__ __forceinline__ unsigned long long spread3(unsigned long long x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

// Morton key of the first min(3, dof) coordinates over [lo, hi] (a locality heuristic
// only: any order gives the same lists).
__global__ void morton_kernel(const double* __restrict__ rows, int n, int dof, double3 lo, double3 inv,
                              unsigned long long* __restrict__ key, int32_t* __restrict__ val) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double l[3] = {lo.x, lo.y, lo.z}, iv[3] = {inv.x, inv.y, inv.z};
    unsigned long long code = 0;
    for (int q = 0; q < 3 && q < dof; ++q) {
        double f = (rows[static_cast<size_t>(i) * dof + q] - l[q]) * iv[q];
        f = f == f ? fmin(fmax(f, 0.0), 1.0) : 0.0;
        code |= spread3(static_cast<unsigned long long>(f * 2097151.0)) << q;
    }
    key[i] = code;
    val[i] = i;
}

// Sorted position p <- node ids[p]: fp64 SoA, fp32 (round to nearest, zero padded).
__global__ void gather_sorted_kernel(const double* __restrict__ rows, int n, int dof, const int32_t* __restrict__ ids,
                                     double* __restrict__ XS, float* __restrict__ X32) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int i = ids[p];
    for (int q = 0; q < dof; ++q) {
        const double v = rows[static_cast<size_t>(i) * dof + q];
        XS[static_cast<size_t>(q) * n + p] = v;
        X32[8 * static_cast<size_t>(p) + q] = __double2float_rn(v);
    }
    for (int q = dof; q < 8; ++q) X32[8 * static_cast<size_t>(p) + q] = 0.0f;
}

// fp64 box (min, max per coordinate) of each tile of kTile sorted nodes.
__global__ void tile_box_kernel(const double* __restrict__ XS, int n, int dof, double* __restrict__ boxes) {
    const int t = blockIdx.x, lane = threadIdx.x;  // one warp per tile
    const int p0 = t * kTile, p1 = min(n, p0 + kTile);
    for (int q = 0; q < dof; ++q) {
        double lo = INFINITY, hi = -INFINITY;
        for (int p = p0 + lane; p < p1; p += 32) {
            const double v = XS[static_cast<size_t>(q) * n + p];
            lo = fmin(lo, v);
            hi = fmax(hi, v);
        }
        for (int o = 16; o; o >>= 1) {
            lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            boxes[static_cast<size_t>(t) * 2 * dof + q] = lo;
            boxes[static_cast<size_t>(t) * 2 * dof + dof + q] = hi;
        }
    }
}

// Merge the per-split lists of row i (each sorted by (d, j), j disjoint across
// splits) into its kk best and emit the (min, max) keys.
__global__ void merge_kernel(const double* __restrict__ pd, const int32_t* __restrict__ pj, int n, int k, int kk,
                             int splits, unsigned long long* __restrict__ keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int head[64];
    for (int s = 0; s < splits; ++s) head[s] = 0;
    for (int t = 0; t < kk; ++t) {
        int best = -1;
        double bd = INFINITY;
        int32_t bj = INT32_MAX;
        for (int s = 0; s < splits; ++s) {
            if (head[s] >= k) continue;
            const size_t o = (static_cast<size_t>(s) * k + head[s]) * n + i;
            const double d = pd[o];
            const int32_t j = pj[o];
            if (j == INT32_MAX) continue;
            if (best < 0 || d < bd || (d == bd && j < bj)) {
                best = s;
                bd = d;
                bj = j;
            }
        }
        unsigned long long key = ~0ull;  // cannot happen for t < kk = min(k, n-1)
        if (best >= 0) {
            ++head[best];
            const unsigned a = static_cast<unsigned>(min(i, bj)), b = static_cast<unsigned>(max(i, bj));
            key = (static_cast<unsigned long long>(a) << 32) | b;
        }
        keys[static_cast<size_t>(i) * kk + t] = key;
    }
}

__global__ void keys_to_pairs_kernel(const unsigned long long* __restrict__ keys, const int* __restrict__ n_unique,
                                     int2* __restrict__ pairs) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= *n_unique) return;
    const unsigned long long key = keys[e];
    pairs[e] = make_int2(static_cast<int>(key >> 32), static_cast<int>(key & 0xffffffffu));
}

template <int DOF>
void launch_tiled(const double* XS, const float* X32, const int32_t* ids, const double* boxes, int n, int k, int R,
                  size_t smem, double E, double* pd, int32_t* pj, unsigned long long* stats, cudaStream_t st) {
    auto kern = knn_tiled_kernel<DOF>;
    ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    kern<<<(n + R - 1) / R, R, smem, st>>>(XS, reinterpret_cast<const float4*>(X32), ids, boxes, n, k, E, pd, pj,
                                           stats);
    ck(cudaGetLastError(), "knn_tiled_kernel");
}

int sm_count() {
    static int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return sms;
}

// Grow-only device arena reused across calls (the API is not reentrant).
struct Arena {
    unsigned char* p = nullptr;
    size_t cap = 0;
    unsigned char* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
            cap = bytes;
        }
        return p;
    }
};
Arena g_arena;

struct Carve {  // 256-byte aligned sub-allocations of one arena block
    size_t off = 0;
    size_t take(size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~size_t(255);
        return o;
    }
};

constexpr size_t kTiledSmemMax = 200 * 1024;

int64_t knn_edges(const double* nodes, int n, int dof, int k, int32_t* edges, int64_t cap, float* kernel_ms) {
    const int kk = std::min(k, n - 1);
    if (kk <= 0) return 0;
    k = kk;
    // tiled: rows per CTA R so that about four CTAs per SM are available
    int R = 128;
    while (R > 32 && (n + R - 1) / R < 4 * sm_count()) R >>= 1;
    const size_t tiled_smem = kTile * 32 + static_cast<size_t>(dof) * kTile * 8 + static_cast<size_t>(k) * R * 12;
    const bool tiled = dof <= 8 && tiled_smem <= kTiledSmemMax;
    // generic scan: threads per CTA so the insertion lists (k*T*12 bytes) fit; the
    // candidate range split until the grid covers the GPU about twice
    int T = 128;
    while (T > 32 && static_cast<size_t>(k) * T * 12 > 96 * 1024) T >>= 1;
    const size_t scan_smem = static_cast<size_t>(dof) * kTile * 8 + static_cast<size_t>(k) * T * 12;
    int splits = 1;
    if (!tiled) {
        const int row_ctas = (n + T - 1) / T;
        const int want = 2 * sm_count() * std::max(1, static_cast<int>((228 * 1024) / (scan_smem + 1024)));
        splits = std::max(1, std::min(64, want / std::max(1, row_ctas)));
        splits = std::max(1, std::min(splits, n / (4 * kTile)));
    }
    const int span = (n + splits - 1) / splits;

    // host pass: Morton bounds of the first three coordinates, and the fp32 filter's
    // E = 2u(1+u)|M| (filter_bound) from the per-coordinate max |x|; the filter is off
    // (E < 0) for non-finite or huge coordinates (fp32 overflow)
    double E = -1.0;
    double lo3[3] = {0, 0, 0}, hi3[3] = {0, 0, 0};
    if (tiled) {
        std::vector<double> M(dof, 0.0);
        bool finite = true;
        for (int q = 0; q < 3; ++q) lo3[q] = INFINITY, hi3[q] = -INFINITY;
        for (size_t t = 0; t < static_cast<size_t>(n) * dof; ++t) {
            const double v = nodes[t], a = std::fabs(v);
            const int q = static_cast<int>(t % dof);
            if (!(a <= 1e15)) finite = false;
            if (a > M[q]) M[q] = a;
            if (q < 3 && v == v) {
                lo3[q] = std::min(lo3[q], v);
                hi3[q] = std::max(hi3[q], v);
            }
        }
        if (finite) {
            double m2 = 0.0;
            for (double m : M) m2 += m * m;
            E = 2.0 * 0x1p-24 * (1.0 + 0x1p-24) * std::sqrt(m2) * (1.0 + 0x1p-40) + 1e-30;
        }
    }
    double inv3[3];
    for (int q = 0; q < 3; ++q) {
        const double w = hi3[q] - lo3[q];
        inv3[q] = w > 0 && std::isfinite(w) ? 1.0 / w : 0.0;
        if (!std::isfinite(lo3[q])) lo3[q] = 0.0;
    }

    cudaStream_t st = nullptr;
    const size_t nkeys = static_cast<size_t>(n) * kk;
    const size_t lists = static_cast<size_t>(splits) * k * n;
    const int ntiles = (n + kTile - 1) / kTile;
    int hb = 1;
    while ((1ll << hb) < n) ++hb;
    size_t tmp_sort = 0, tmp_uniq = 0, tmp_pairs = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, static_cast<unsigned long long*>(nullptr),
                                   static_cast<unsigned long long*>(nullptr), static_cast<int64_t>(nkeys), 0, 32 + hb, st);
    cub::DeviceSelect::Unique(nullptr, tmp_uniq, static_cast<unsigned long long*>(nullptr),
                              static_cast<unsigned long long*>(nullptr), static_cast<int*>(nullptr),
                              static_cast<int64_t>(nkeys), st);
    if (tiled)
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_pairs, static_cast<unsigned long long*>(nullptr),
                                        static_cast<unsigned long long*>(nullptr), static_cast<int32_t*>(nullptr),
                                        static_cast<int32_t*>(nullptr), n, 0, 63, st);
    Carve cv;
    const size_t o_rows = cv.take(static_cast<size_t>(n) * dof * 8);
    const size_t o_X = cv.take(static_cast<size_t>(n) * dof * 8);
    const size_t o_X32 = cv.take(tiled ? static_cast<size_t>(n) * 32 : 0);
    const size_t o_mk = cv.take(tiled ? static_cast<size_t>(n) * 8 * 2 : 0);
    const size_t o_mv = cv.take(tiled ? static_cast<size_t>(n) * 4 * 2 : 0);
    const size_t o_box = cv.take(tiled ? static_cast<size_t>(ntiles) * 2 * dof * 8 : 0);
    const size_t o_pd = cv.take(lists * 8);
    const size_t o_pj = cv.take(lists * 4);
    const size_t o_keys = cv.take(nkeys * 8);
    const size_t o_sorted = cv.take(nkeys * 8);
    const size_t o_cnt = cv.take(16);
    const size_t o_tmp = cv.take(std::max(std::max(tmp_sort, tmp_uniq), tmp_pairs));
    unsigned char* base = g_arena.get(cv.off);
    double* rows = reinterpret_cast<double*>(base + o_rows);
    double* X = reinterpret_cast<double*>(base + o_X);
    float* X32 = reinterpret_cast<float*>(base + o_X32);
    auto* mk = reinterpret_cast<unsigned long long*>(base + o_mk);
    auto* mv = reinterpret_cast<int32_t*>(base + o_mv);
    double* boxes = reinterpret_cast<double*>(base + o_box);
    double* pd = reinterpret_cast<double*>(base + o_pd);
    int32_t* pj = reinterpret_cast<int32_t*>(base + o_pj);
    auto* keys = reinterpret_cast<unsigned long long*>(base + o_keys);
    auto* sorted = reinterpret_cast<unsigned long long*>(base + o_sorted);
    int* nuniq = reinterpret_cast<int*>(base + o_cnt);
    auto* stats = reinterpret_cast<unsigned long long*>(base + o_cnt + 8);
    void* tmp = base + o_tmp;

    ck(cudaMemcpyAsync(rows, nodes, static_cast<size_t>(n) * dof * 8, cudaMemcpyHostToDevice, st), "upload nodes");
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    cudaEventRecord(e0, st);
    const unsigned g = static_cast<unsigned>((n + 127) / 128);
    if (tiled) {
        cudaMemsetAsync(stats, 0, 8, st);
        morton_kernel<<<g, 128, 0, st>>>(rows, n, dof, make_double3(lo3[0], lo3[1], lo3[2]),
                                         make_double3(inv3[0], inv3[1], inv3[2]), mk, mv);
        ck(cudaGetLastError(), "morton_kernel");
        ck(cub::DeviceRadixSort::SortPairs(tmp, tmp_pairs, mk, mk + n, mv, mv + n, n, 0, 63, st), "morton sort");
        const int32_t* ids = mv + n;
        gather_sorted_kernel<<<g, 128, 0, st>>>(rows, n, dof, ids, X, X32);
        ck(cudaGetLastError(), "gather_sorted_kernel");
        tile_box_kernel<<<ntiles, 32, 0, st>>>(X, n, dof, boxes);
        ck(cudaGetLastError(), "tile_box_kernel");
        switch (dof) {
            case 1: launch_tiled<1>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 2: launch_tiled<2>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 3: launch_tiled<3>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 4: launch_tiled<4>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 5: launch_tiled<5>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 6: launch_tiled<6>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            case 7: launch_tiled<7>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
            default: launch_tiled<8>(X, X32, ids, boxes, n, k, R, tiled_smem, E, pd, pj, stats, st); break;
        }
    } else {
        soa_kernel<<<g, 128, 0, st>>>(rows, n, dof, X);
        ck(cudaGetLastError(), "soa_kernel");
        ck(cudaFuncSetAttribute(knn_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(scan_smem)),
           "cudaFuncSetAttribute");
        knn_scan_kernel<<<dim3((n + T - 1) / T, splits), T, scan_smem, st>>>(X, n, dof, k, span, pd, pj);
        ck(cudaGetLastError(), "knn_scan_kernel");
    }
    merge_kernel<<<g, 128, 0, st>>>(pd, pj, n, k, kk, splits, keys);
    ck(cudaGetLastError(), "merge_kernel");
    // candidates.sort + unique (roadmap.cpp:91-93): bits above the largest id never vary
    ck(cub::DeviceRadixSort::SortKeys(tmp, tmp_sort, keys, sorted, static_cast<int64_t>(nkeys), 0, 32 + hb, st),
       "radix sort");
    ck(cub::DeviceSelect::Unique(tmp, tmp_uniq, sorted, keys, nuniq, static_cast<int64_t>(nkeys), st), "unique");
    int2* pairs = reinterpret_cast<int2*>(sorted);  // reuse: nkeys * 8 bytes
    keys_to_pairs_kernel<<<static_cast<unsigned>((nkeys + 255) / 256), 256, 0, st>>>(keys, nuniq, pairs);
    ck(cudaGetLastError(), "keys_to_pairs_kernel");
    cudaEventRecord(e1, st);
    int nu = 0;
    ck(cudaMemcpy(&nu, nuniq, sizeof(int), cudaMemcpyDeviceToHost), "read count");
    if (kernel_ms) cudaEventElapsedTime(kernel_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (tiled && std::getenv("RGG_PRM_STATS")) {
        unsigned long long v = 0;
        cudaMemcpy(&v, stats, 8, cudaMemcpyDeviceToHost);
        std::fprintf(stderr, "[prm] n=%d k=%d R=%d tiles visited %.1f of %d per row group\n", n, k, R,
                     static_cast<double>(v) / ((n + R - 1) / R), ntiles);
    }
    if (nu > cap) return -static_cast<int64_t>(nu) - 1;
    if (nu) ck(cudaMemcpy(edges, pairs, static_cast<size_t>(nu) * sizeof(int2), cudaMemcpyDeviceToHost), "download");
    return nu;
}

}  // namespace

extern "C" {

const char* rgg_prm_last_error(void) { return g_prm_err.c_str(); }

int rgg_prm_nodes(uint64_t seed, int32_t n, int32_t dof, const double* lo, const double* hi, double* nodes) {
    if (n < 1 || dof < 1 || !lo || !hi || !nodes) {
        g_prm_err = n < 1 ? "node count must be >= 1" : "bad arguments";
        return RGG_PRM_EINVAL;
    }
    std::mt19937_64 gen(seed);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t q = 0; q < dof; ++q) {
            const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
            const double span = hi[q] - lo[q];
            const double v = span * u;  // two roundings, as lo + (hi - lo) * unit() (no FMA on the host ISA)
            nodes[static_cast<size_t>(i) * dof + q] = lo[q] + v;
        }
    return 0;
}

int rgg_prm_knn_edges(const double* nodes, int32_t n, int32_t dof, int32_t k, int32_t* edges, int64_t cap,
                      int64_t* n_edges, float* device_ms) {
    try {
        if (n < 1) throw std::invalid_argument("node count must be >= 1");
        if (k < 1) throw std::invalid_argument("neighbor count must be >= 1");
        if (dof < 1 || dof > kMaxDof) throw std::invalid_argument("dof must be in [1, 32]");
        if (std::min(k, n - 1) > kMaxK) throw std::invalid_argument("neighbor count above 512 is not supported on the GPU");
        if (!nodes || (!edges && cap > 0)) throw std::invalid_argument("null pointer");
        if (device_ms) *device_ms = 0.0f;
        const int64_t r = knn_edges(nodes, n, dof, std::max(1, std::min(k, n - 1)), edges, cap, device_ms);
        if (r < 0) {
            if (n_edges) *n_edges = -r - 1;
            g_prm_err = "edge buffer too small";
            return RGG_PRM_ESPACE;
        }
        if (n_edges) *n_edges = r;
        return 0;
    } catch (const std::invalid_argument& e) {
        g_prm_err = e.what();
        return RGG_PRM_EINVAL;
    } catch (const std::exception& e) {
        g_prm_err = e.what();
        return RGG_PRM_ECUDA;
    }
}

}  // extern "C"
