// rgg_resolve.cu — exact resolve of GRAY components on the GPU.
//
// exact_component_valid (proj/src/roadmap.cpp:129-163): a component is free iff
// no robot body, at any of its discretized configurations, intersects an active
// obstacle.  Per (configuration, body) the reference builds the body box
// (apply_transform + aabb_of_obb, geometry.cpp:205-213 and :307-313), gates every
// active obstacle by closed AABB overlap, and runs polytopes_intersect
// (geometry.cpp:256-303) on ConvexPolytope::box of both (:228-254).
//
// The forward kinematics (proj/src/robot.cpp:66-84) of every configuration is
// computed once on the host (libm sin/cos, as the reference) and uploaded as
// per-(configuration, body) world poses; everything from the pose on runs here,
// in fp64 with the reference's operation order and no contraction, so the
// verdict is the reference's bit for bit:
//   * Box vertices: obb_corners of {centre = pose.t, axes = pose.rotate(e_k)}.
//   * Face axes: the reference tests +/-axes; a negated axis negates every
//     projection exactly, so it separates iff the positive one does.
//   * Edge axes: the reference crosses the 24 ring-edge directions of each box
//     (each box edge once per orientation, v[q] - v[p] or its exact negation);
//     cross products of negated operands are exact negations too, so the 12 x
//     12 canonical edge pairs decide exactly what the 24 x 24 ring pairs decide.
//   * Every axis is a pure predicate, so testing them in any order (32 lanes
//     at a time) gives the reference's early-exit result.
#include "rgg_device.cuh"
#include "rgg_kernels.cuh"

namespace rggk {
namespace {

using rggd::add;
using rggd::mul;
using rggd::sub;

// box edges (p, q = p | bit): along axis 0, 1, 2
__constant__ int kEdgeP[12] = {0, 2, 4, 6, 0, 1, 4, 5, 0, 1, 2, 3};
__constant__ int kEdgeBit[12] = {1, 1, 1, 1, 2, 2, 2, 2, 4, 4, 4, 4};

// pose.rotate(e_k), component i (vec3.hpp:79-84)
__device__ __forceinline__ double rot_unit(const double* r, int k, int i) {
    const double x = k == 0 ? 1.0 : 0.0, y = k == 1 ? 1.0 : 0.0, z = k == 2 ? 1.0 : 0.0;
    return add(add(mul(r[3 * i], x), mul(r[3 * i + 1], y)), mul(r[3 * i + 2], z));
}

// Coordinate j of corner i of ConvexPolytope::box(he, pose) (geometry.cpp:228-254
// + obb_corners :50-62): centre = pose.t, e_k = pose.rotate(unit_k) * he_k.
__device__ __forceinline__ double corner(const double* rt, const double* he, int i, int j) {
    const double e0 = mul(rot_unit(rt, 0, j), he[0]);
    const double e1 = mul(rot_unit(rt, 1, j), he[1]);
    const double e2 = mul(rot_unit(rt, 2, j), he[2]);
    double p = (i & 1) ? add(rt[9 + j], e0) : sub(rt[9 + j], e0);
    p = (i & 2) ? add(p, e1) : sub(p, e1);
    return (i & 4) ? add(p, e2) : sub(p, e2);
}

// One box as polytopes_intersect sees it (warp-shared).
struct PolyS {
    double v[24];   // vertices
    double ax[9];   // face axes (+ side)
    double ed[36];  // 12 edge directions
    double box[6];  // aabb_of_obb
};

// Fill a PolyS from a pose (12 doubles) and half extents, all 32 lanes.
// The AABB is the min/max of the vertices: aabb_of_obb uses centre
// pose.apply(0) instead of pose.t, which differ at most in the sign of a zero,
// and no comparison can tell those apart.
__device__ void build_poly(PolyS& P, const double* rt, const double* he, int lane) {
    if (lane < 24) P.v[lane] = corner(rt, he, lane / 3, lane % 3);
    if (lane < 9) P.ax[lane] = rot_unit(rt, lane / 3, lane % 3);
    __syncwarp();
    for (int t = lane; t < 36; t += 32) {
        const int e = t / 3, j = t % 3, p = kEdgeP[e], q = p | kEdgeBit[e];
        P.ed[t] = sub(P.v[3 * q + j], P.v[3 * p + j]);
    }
    if (lane < 3) {
        double lo = P.v[lane], hi = P.v[lane];
        for (int i = 1; i < 8; ++i) {
            lo = fmin(lo, P.v[3 * i + lane]);
            hi = fmax(hi, P.v[3 * i + lane]);
        }
        P.box[lane] = lo;
        P.box[3 + lane] = hi;
    }
    __syncwarp();
}

__device__ __forceinline__ double dot3(const double* v, const double* a) {
    return add(add(mul(v[0], a[0]), mul(v[1], a[1])), mul(v[2], a[2]));
}

// separates (geometry.cpp:268-273): projections of both vertex sets disjoint.
__device__ __forceinline__ bool separates(const PolyS& A, const PolyS& B, const double* ax) {
    double alo = dot3(A.v, ax), ahi = alo, blo = dot3(B.v, ax), bhi = blo;
#pragma unroll
    for (int i = 1; i < 8; ++i) {
        const double ta = dot3(A.v + 3 * i, ax), tb = dot3(B.v + 3 * i, ax);
        alo = fmin(alo, ta);
        ahi = fmax(ahi, ta);
        blo = fmin(blo, tb);
        bhi = fmax(bhi, tb);
    }
    return ahi < blo || bhi < alo;
}

// polytopes_intersect (geometry.cpp:278-303) over the warp: 6 face axes + 144
// edge-pair axes, 32 at a time; false as soon as any lane separates.
__device__ bool boxes_intersect(const PolyS& A, const PolyS& B, int lane) {
    for (int base = 0; base < 150; base += 32) {
        const int j = base + lane;
        bool sep = false;
        if (j < 3) {
            sep = separates(A, B, A.ax + 3 * j);
        } else if (j < 6) {
            sep = separates(A, B, B.ax + 3 * (j - 3));
        } else if (j < 150) {
            const double* da = A.ed + 3 * ((j - 6) / 12);
            const double* db = B.ed + 3 * ((j - 6) % 12);
            const double ax[3] = {sub(mul(da[1], db[2]), mul(da[2], db[1])), sub(mul(da[2], db[0]), mul(da[0], db[2])),
                                  sub(mul(da[0], db[1]), mul(da[1], db[0]))};
            if (dot3(ax, ax) > 0.0) sep = separates(A, B, ax);
        }
        if (__any_sync(0xffffffffu, sep)) return false;
    }
    return true;
}

__device__ __forceinline__ bool box_overlap(const double* a, const double* b) {
    return a[0] <= b[3] && b[0] <= a[3] && a[1] <= b[4] && b[1] <= a[4] && a[2] <= b[5] && b[2] <= a[5];
}

// The active obstacles' polytopes at their current poses (Event::rt).  An
// obstacle this engine has not moved yet is active at its scene pose when the
// host listed it (rgg_gpu_set_active_obstacles: ObstacleModel::active before the
// engine's first move, the `if (!o.active) continue;` of roadmap.cpp:135-136).
__global__ void resolve_prep_kernel(Store s, Resolver r) {
    const int o = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (o >= s.M) return;
    __shared__ PolyS sp[4];
    PolyS& P = sp[threadIdx.x >> 5];
    const double* un = s.cur_union + 6 * o;
    const bool moved = un[0] <= un[3];  // inactive obstacles keep an empty union box
    const bool scene = !moved && r.sact && r.sact[o];
    const bool active = moved || scene;
    build_poly(P, scene ? r.spose + 12 * static_cast<size_t>(o) : s.cur[o].rt, s.ohe + 3 * o, lane);
    ObsPoly& out = r.opoly[o];
    for (int t = lane; t < 24; t += 32) out.v[t] = P.v[t];
    for (int t = lane; t < 9; t += 32) out.ax[t] = P.ax[t];
    for (int t = lane; t < 36; t += 32) out.ed[t] = P.ed[t];
    if (lane < 6) out.box[lane] = P.box[lane];
    if (lane == 0) out.active = active ? 1 : 0;
}

constexpr int kResolveWarps = 4;

// SPLIT (eager moves: a few hundred gray over-hits, too few warps to fill the GPU):
// one CTA per listed component; its warps split the component's configurations
// (warp w takes configurations c0 + w, c0 + w + kResolveWarps, ...) and stop as soon
// as any warp finds an intersection (a shared flag).  Otherwise (resolve_all_unknown,
// exact checks: thousands of components) one warp per component.  The verdict is the
// OR over (configuration, body, obstacle) of polytopes_intersect, so the mapping
// does not change it.  MODE kResolve: the listed (GRAY) components become GREEN or RED.
// kEager (one-move eager update): the list is the move's gray over-hits with their
// pre-move labels, and the report deltas of finish_counts (engine_batch.cpp:41-53)
// go to ctr[20..23].  kCheck: verdicts to out[], no label changes.
template <int MODE, bool SPLIT>
__global__ void __launch_bounds__(32 * kResolveWarps) resolve_kernel(Store s, Resolver r, Batch b, const int32_t* ids,
                                                                     const int32_t* count_ptr, uint8_t* out) {
    constexpr bool EAGER = MODE == kEager;
    __shared__ PolyS sa[kResolveWarps], sb[kResolveWarps];
    __shared__ int hits[kResolveWarps];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    volatile int* hit = hits + (SPLIT ? 0 : wi);
    const bool leader = SPLIT ? threadIdx.x == 0 : lane == 0;
    const int unit0 = SPLIT ? blockIdx.x : blockIdx.x * kResolveWarps + wi;
    const int ustride = SPLIT ? gridDim.x : gridDim.x * kResolveWarps;
    const int cfg0 = SPLIT ? wi : 0, cstride = SPLIT ? kResolveWarps : 1;
    auto sync = [&]() {
        if (SPLIT)
            __syncthreads();
        else
            __syncwarp();
    };
    PolyS& A = sa[wi];
    PolyS& Bo = sb[wi];
    const int count = *count_ptr;
    int d[4] = {0, 0, 0, 0};
    for (int k = unit0; k < count; k += ustride) {
        const int id = ids[k];
        if (leader) *hit = 0;
        sync();
        const long long c0 = r.off[id], c1 = r.off[id + 1];
        bool free = true;
        for (long long cfg = c0 + cfg0; cfg < c1 && free; cfg += cstride) {
            for (int body = 0; body < r.B && free; ++body) {
                // another warp found an intersection: stop (warp-uniform)
                if (SPLIT && __any_sync(0xffffffffu, *hit != 0)) free = false;
                if (!free) break;
                const double* pose = r.pose + (cfg * r.B + body) * 12;
                __syncwarp();
                build_poly(A, pose, r.he + 3 * body, lane);
                for (int base = 0; base < s.M && free; base += 32) {
                    const int o = base + lane;
                    bool cand = false;
                    if (o < s.M) {
                        const ObsPoly& op = r.opoly[o];
                        cand = op.active && box_overlap(A.box, op.box);
                    }
                    for (unsigned m = __ballot_sync(0xffffffffu, cand); m && free; m &= m - 1) {
                        const ObsPoly& op = r.opoly[base + __ffs(m) - 1];
                        __syncwarp();
                        for (int t = lane; t < 24; t += 32) Bo.v[t] = op.v[t];
                        for (int t = lane; t < 9; t += 32) Bo.ax[t] = op.ax[t];
                        for (int t = lane; t < 36; t += 32) Bo.ed[t] = op.ed[t];
                        __syncwarp();
                        if (boxes_intersect(A, Bo, lane)) {
                            free = false;
                            if (lane == 0) *hit = 1;
                        }
                    }
                }
            }
        }
        sync();
        const bool is_free = *hit == 0;
        if (leader && MODE == kCheck) out[k] = is_free ? 0 : 1;
        if (leader && MODE != kCheck) {
            const uint8_t fin = is_free ? 0 : 1;  // GREEN : RED
            s.state[id] = fin;
            const int c = s.rank[id];
            if (c >= 0) s.state_c[c] = fin;
            if (EAGER) {
                const int prev = b.hits_prev[k];
                d[0] += (fin == 0 && prev != 0);
                d[1] += (fin == 1 && prev != 1);
                d[2] -= (prev != 2);
                d[3] += (prev == 2);
            }
        }
        sync();  // the flag is reset for the next component only after every thread read it
    }
    if (leader && MODE != kCheck) {
        int n = 0;
        for (int k = unit0; k < count; k += ustride) ++n;
        if (n) atomicAdd(b.unknown, -n);  // every listed component was GRAY
        if (EAGER)
            for (int q = 0; q < 4; ++q)
                if (d[q]) atomicAdd(&b.ctr[20 + q], d[q]);
    }
}

}  // namespace

cudaError_t launch_resolve(const Store& s, const Resolver& r, const Batch& b, const int32_t* ids,
                           const int32_t* count_dev, int max_count, int mode, uint8_t* out, cudaStream_t st) {
    if (s.M > 0) {
        resolve_prep_kernel<<<(s.M + 3) / 4, 128, 0, st>>>(s, r);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // eager: one CTA per component (max_count bounds the grid); otherwise one warp per component
    const int need = mode == kEager ? max_count : (max_count + kResolveWarps - 1) / kResolveWarps;
    const int grid = need < 1 ? 1 : (need < 8 * sms ? need : 8 * sms);
    if (mode == kEager)
        resolve_kernel<kEager, true><<<grid, 32 * kResolveWarps, 0, st>>>(s, r, b, ids, count_dev, out);
    else if (mode == kCheck)
        resolve_kernel<kCheck, false><<<grid, 32 * kResolveWarps, 0, st>>>(s, r, b, ids, count_dev, out);
    else
        resolve_kernel<kResolve, false><<<grid, 32 * kResolveWarps, 0, st>>>(s, r, b, ids, count_dev, out);
    return cudaGetLastError();
}

}  // namespace rggk
