// rgg_kernels.cu — the SerRGG update pipeline for sm_100a.
//
//   pose      one thread per move: BatchLayout::update_transforms
//             (proj/src/batch_layout.cpp:148-172) on device, fp64-exact.
//   bin       one warp per cell: closed AABB test of every event's new and old
//             box against the cell's box, ordered warp-ballot compaction into a
//             fixed-capacity cell list + overflow pool, dirty-cell list.
//             Replaces SpatialGrid::candidates (proj/src/spatial_grid.cpp:114-135).
//   classify  one CTA per dirty cell, one thread per component: the cell's event
//             list staged in shared memory, each event applied in move order with
//             the reference's per-move state transition (engine_batch.cpp:114-188):
//             15-axis SAT (over) and segment-sphere (under) narrow tests.
//   commit    one thread per move: the moved obstacles' resident operands.
//   compact   ordered ballot/prefix compaction of the GRAY component ids.
#include <cstdio>

#include "rgg_device.cuh"
#include "rgg_kernels.cuh"

namespace rggk {

using rggd::add;
using rggd::mul;
using rggd::sub;

namespace {

__device__ __forceinline__ void aabb_empty(double* a) {
    a[0] = a[1] = a[2] = __longlong_as_double(0x7ff0000000000000ll);   // +inf
    a[3] = a[4] = a[5] = __longlong_as_double(0xfff0000000000000ll);   // -inf
}

__device__ __forceinline__ void aabb_expand(double* a, double x, double y, double z) {
    a[0] = fmin(a[0], x);
    a[1] = fmin(a[1], y);
    a[2] = fmin(a[2], z);
    a[3] = fmax(a[3], x);
    a[4] = fmax(a[4], y);
    a[5] = fmax(a[5], z);
}

__device__ __forceinline__ void aabb_union(const double* a, const double* b, double* out) {
    for (int k = 0; k < 3; ++k) out[k] = fmin(a[k], b[k]);
    for (int k = 3; k < 6; ++k) out[k] = fmax(a[k], b[k]);
}

// Obstacle box + spheres at pose rt (batch_layout.cpp:148-172 with
// apply_transform(Obb) geometry.cpp:307-313, obb_corners :50-62, aabb_of_obb :205-213).
// When SAT is false only the two boxes are produced.
template <bool FULL>
__device__ void obstacle_at(const Store& s, int o, const double* rt, double* sat21, double* box, double* sph,
                            double* cen, int* nsph_out) {
    const double he0 = s.ohe[3 * o], he1 = s.ohe[3 * o + 1], he2 = s.ohe[3 * o + 2];
    double center[3];
    rggd::tf_apply(rt, 0.0, 0.0, 0.0, center);
    // Transform::rotate of the unit axes, then Vec3 * half extent.
    double e[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double r0 = rt[3 * i], r1 = rt[3 * i + 1], r2 = rt[3 * i + 2];
        e[0][i] = mul(add(add(mul(r0, 1.0), mul(r1, 0.0)), mul(r2, 0.0)), he0);
        e[1][i] = mul(add(add(mul(r0, 0.0), mul(r1, 1.0)), mul(r2, 0.0)), he1);
        e[2][i] = mul(add(add(mul(r0, 0.0), mul(r1, 0.0)), mul(r2, 1.0)), he2);
    }
    double corners[24];
    aabb_empty(box);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        double p[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) p[i] = (c & 1) ? add(center[i], e[0][i]) : sub(center[i], e[0][i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) p[i] = (c & 2) ? add(p[i], e[1][i]) : sub(p[i], e[1][i]);
#pragma unroll
        for (int i = 0; i < 3; ++i) p[i] = (c & 4) ? add(p[i], e[2][i]) : sub(p[i], e[2][i]);
        corners[3 * c] = p[0];
        corners[3 * c + 1] = p[1];
        corners[3 * c + 2] = p[2];
        aabb_expand(box, p[0], p[1], p[2]);
    }
    if (FULL) rggd::sat_prep(corners, sat21);
    const int n = s.osn[o];
    const double r = s.osr[o];
    aabb_empty(sph);
    for (int k = 0; k < n; ++k) {
        const double* l = s.osl + (static_cast<size_t>(o) * s.C + k) * 3;
        double c3[3];
        rggd::tf_apply(rt, l[0], l[1], l[2], c3);
        if (FULL) {
            cen[3 * k] = c3[0];
            cen[3 * k + 1] = c3[1];
            cen[3 * k + 2] = c3[2];
        }
        aabb_expand(sph, sub(c3[0], r), sub(c3[1], r), sub(c3[2], r));
        aabb_expand(sph, add(c3[0], r), add(c3[1], r), add(c3[2], r));
    }
    if (nsph_out) *nsph_out = n;
}

// One warp per move: BatchLayout::update_transforms (batch_layout.cpp:148-172)
// spread over the lanes.  Lanes 0-7 build the 8 corners of the new box, lanes
// 8-15 those of the pose before this move (for the binning's old box), lanes
// 16.. the sphere centres; AABBs are warp min/max reductions (min/max are exact,
// so the order of the reduction does not change a value); lanes 0-2 run
// sat_prep's three axes in parallel.
__device__ __forceinline__ double shfl(double v, int src, int width = 32) {
    return __shfl_sync(0xffffffffu, v, src, width);
}

__device__ __forceinline__ void box_of(const double* rt, const double* he, int corner, double* p) {
    double center[3];
    rggd::tf_apply(rt, 0.0, 0.0, 0.0, center);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double r0 = rt[3 * i], r1 = rt[3 * i + 1], r2 = rt[3 * i + 2];
        // Transform::rotate of the unit axes, then Vec3 * half extent (geometry.cpp:307-313, :50-54)
        const double e0 = mul(add(add(mul(r0, 1.0), mul(r1, 0.0)), mul(r2, 0.0)), he[0]);
        const double e1 = mul(add(add(mul(r0, 0.0), mul(r1, 1.0)), mul(r2, 0.0)), he[1]);
        const double e2 = mul(add(add(mul(r0, 0.0), mul(r1, 0.0)), mul(r2, 1.0)), he[2]);
        double v = (corner & 1) ? add(center[i], e0) : sub(center[i], e0);
        v = (corner & 2) ? add(v, e1) : sub(v, e1);
        p[i] = (corner & 4) ? add(v, e2) : sub(v, e2);
    }
}

__global__ void pose_kernel(Store s, Batch b) {
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i == 0 && lane < 8) {
        b.ctr[lane] = 0;
        b.census[lane] = 0;
    }
    if (i >= b.n) return;
    const int o = b.ids[i];
    // prev / last links: the same obstacle moved earlier / later in this batch
    int p = -1;
    bool is_last = true;
    for (int base = 0; base < b.n; base += 32) {
        const int j = base + lane;
        const bool same = j < b.n && b.ids[j] == o;
        const unsigned before = __ballot_sync(0xffffffffu, same && j < i);
        const unsigned after = __ballot_sync(0xffffffffu, same && j > i);
        if (before) p = base + 31 - __clz(before);
        if (after) is_last = false;
    }
    const double he[3] = {s.ohe[3 * o], s.ohe[3 * o + 1], s.ohe[3 * o + 2]};
    const double* rt_new = b.rt + 12 * static_cast<size_t>(i);
    const double* rt_old = p >= 0 ? b.rt + 12 * static_cast<size_t>(p) : rt_new;
    const double* rt = lane < 8 ? rt_new : (lane < 16 ? rt_old : rt_new);
    double rtl[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) rtl[k] = rt[k];
    // corners (lanes 0-15) and sphere centres (lanes 16-31)
    const int nsph = s.osn[o];
    const double r = s.osr[o];
    double lo[3], hi[3], pt[3] = {0, 0, 0};
    if (lane < 16) {
        box_of(rtl, he, lane & 7, pt);
#pragma unroll
        for (int k = 0; k < 3; ++k) lo[k] = hi[k] = pt[k];
    } else {
        const int sp = lane - 16;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = __longlong_as_double(0x7ff0000000000000ll);
            hi[k] = __longlong_as_double(0xfff0000000000000ll);
        }
        if (sp < nsph) {
            const double* l = s.osl + (static_cast<size_t>(o) * s.C + sp) * 3;
            rggd::tf_apply(rtl, l[0], l[1], l[2], pt);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                lo[k] = sub(pt[k], r);
                hi[k] = add(pt[k], r);
            }
        }
    }
    // min/max over groups of 8 (corners) or 16 (spheres)
    const int width = lane < 16 ? 8 : 16;
#pragma unroll
    for (int off = 1; off < 16; off <<= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double a = __shfl_xor_sync(0xffffffffu, lo[k], off);
            const double c = __shfl_xor_sync(0xffffffffu, hi[k], off);
            if (off < width) {
                lo[k] = fmin(lo[k], a);
                hi[k] = fmax(hi[k], c);
            }
        }
    }
    // sat_prep (kernels_scalar.cpp:7-30): lane k < 3 derives axis k
    const int src = lane < 3 ? (1 << lane) : 0;
    double c0[3], ch[3], e[3], u[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        c0[k] = shfl(pt[k], 0);
        ch[k] = shfl(pt[k], src);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) e[k] = mul(0.5, sub(ch[k], c0[k]));
    const double n2 = add(add(mul(e[0], e[0]), mul(e[1], e[1])), mul(e[2], e[2]));
    if (lane < 3) {
        if (n2 > 0.0) {
            const double len = __dsqrt_rn(n2);
#pragma unroll
            for (int k = 0; k < 3; ++k) u[k] = __ddiv_rn(e[k], len);
        } else {
            u[0] = u[1] = u[2] = 0.0;
        }
    }
    // centre_j = ((c0_j + e0_j) + e1_j) + e2_j on lane j
    double ej[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double vx = shfl(e[0], k), vy = shfl(e[1], k), vz = shfl(e[2], k);
        ej[k] = lane == 0 ? vx : (lane == 1 ? vy : vz);
    }
    const double cj = lane == 0 ? c0[0] : (lane == 1 ? c0[1] : c0[2]);
    Event& ev = b.ev[i];
    if (lane < 3) {
        ev.sat[lane] = add(add(add(cj, ej[0]), ej[1]), ej[2]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ev.sat[3 + 3 * lane + k] = e[k];
            ev.sat[12 + 3 * lane + k] = u[k];
        }
    }
    // boxes: new corners on lane 0, old corners on lane 8, spheres on lane 16
    double bn[6], bo[6], bs[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        bn[k] = shfl(lo[k], 0), bn[3 + k] = shfl(hi[k], 0);
        bo[k] = shfl(lo[k], 8), bo[3 + k] = shfl(hi[k], 8);
        bs[k] = shfl(lo[k], 16), bs[3 + k] = shfl(hi[k], 16);
    }
    // the old spheres' box: recompute on lanes 16.. only when the obstacle moved earlier in this batch
    double os[6];
    if (p >= 0) {
        double olo[3], ohi[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            olo[k] = __longlong_as_double(0x7ff0000000000000ll);
            ohi[k] = __longlong_as_double(0xfff0000000000000ll);
        }
        if (lane >= 16 && lane - 16 < nsph) {
            const double* l = s.osl + (static_cast<size_t>(o) * s.C + (lane - 16)) * 3;
            double q[3];
            rggd::tf_apply(rt_old, l[0], l[1], l[2], q);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                olo[k] = sub(q[k], r);
                ohi[k] = add(q[k], r);
            }
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                olo[k] = fmin(olo[k], __shfl_xor_sync(0xffffffffu, olo[k], off));
                ohi[k] = fmax(ohi[k], __shfl_xor_sync(0xffffffffu, ohi[k], off));
            }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            os[k] = fmin(bo[k], olo[k]);
            os[3 + k] = fmax(bo[3 + k], ohi[k]);
        }
    }
    if (lane < 6) {
        ev.box[lane] = bn[lane];
        ev.sph[lane] = bs[lane];
        ev.nu[lane] = lane < 3 ? fmin(bn[lane], bs[lane]) : fmax(bn[lane], bs[lane]);
        ev.old[lane] = p >= 0 ? os[lane] : s.cur_union[6 * o + lane];
    }
    if (lane >= 16 && lane - 16 < nsph) {
        ev.cen[3 * (lane - 16)] = pt[0];
        ev.cen[3 * (lane - 16) + 1] = pt[1];
        ev.cen[3 * (lane - 16) + 2] = pt[2];
    }
    if (lane == 0) {
        ev.r = r;
        ev.o = o;
        ev.nsph = nsph;
        ev.move = i;
        b.last[i] = is_last ? 1 : 0;
        reinterpret_cast<int4*>(b.mv)[i] = make_int4(0, 0, 0, 0);
    }
}

// Identity pose for every obstacle: serialize() poses obstacles at their
// canonical pose (batch_layout.cpp:117-136); they stay inactive (empty union).
__global__ void init_obstacles_kernel(Store s) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= s.M) return;
    const double id[12] = {1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0};
    Event& e = s.cur[o];
    int nsph = 0;
    obstacle_at<true>(s, o, id, e.sat, e.box, e.sph, e.cen, &nsph);
    e.r = s.osr[o];
    e.o = o;
    e.nsph = nsph;
    e.move = -1;
    aabb_union(e.box, e.sph, e.nu);
    aabb_empty(e.old);
    aabb_empty(s.cur_union + 6 * o);
}

// ------------------------------------------------------------------ binning

constexpr int kBinThreads = 512;  // 16 warps = 16 cells per CTA
constexpr int kBinChunk = 256;    // event boxes staged per pass

__global__ void __launch_bounds__(kBinThreads) bin_kernel(Store s, Batch b) {
    __shared__ double sbox[kBinChunk][12];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * (kBinThreads / 32) + warp;
    const bool live = cell < s.ncells;
    double cb[6];
    if (live)
        for (int k = 0; k < 6; ++k) cb[k] = s.cell_aabb[6 * static_cast<size_t>(cell) + k];
    int count = 0;
    int32_t* inl = b.cell_list + static_cast<size_t>(cell) * s.cap;
    for (int base = 0; base < b.n; base += kBinChunk) {
        __syncthreads();
        const int m = min(kBinChunk, b.n - base);
        for (int t = threadIdx.x; t < m * 12; t += kBinThreads) {
            const int e = t / 12, k = t % 12;
            sbox[e][k] = k < 6 ? b.ev[base + e].nu[k] : b.ev[base + e].old[k - 6];
        }
        __syncthreads();
        if (!live) continue;
        for (int j = 0; j < m; j += 32) {
            const int e = j + lane;
            const bool hit = e < m && (rggd::overlaps(cb, sbox[e]) || rggd::overlaps(cb, sbox[e] + 6));
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int pos = count + __popc(bal & ((1u << lane) - 1u));
                if (pos < s.cap) inl[pos] = base + e;
            }
            count += __popc(bal);
        }
    }
    if (!live) return;
    if (count > s.cap) {
        // Overflow: the full ordered list goes to the pool (second pass).
        int pbase = 0;
        if (lane == 0) {
            pbase = atomicAdd(&b.ctr[1], count);
            atomicAdd(&b.ctr[3], 1);
        }
        pbase = __shfl_sync(0xffffffffu, pbase, 0);
        if (pbase + count > b.pool_cap) {
            if (lane == 0) atomicExch(&b.ctr[6], 1);
            count = s.cap;  // truncated: reported as an error by the host
        } else {
            int at = 0;
            for (int e0 = 0; e0 < b.n; e0 += 32) {
                const int e = e0 + lane;
                bool hit = false;
                if (e < b.n) {
                    const Event& ev = b.ev[e];
                    hit = rggd::overlaps(cb, ev.nu) || rggd::overlaps(cb, ev.old);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (hit) b.pool[pbase + at + __popc(bal & ((1u << lane) - 1u))] = e;
                at += __popc(bal);
            }
            if (lane == 0) b.cell_ovf[cell] = pbase;
        }
    }
    if (lane == 0) {
        b.cell_count[cell] = count;
        if (count > 0) b.dirty[atomicAdd(&b.ctr[0], 1)] = cell;
    }
}

// ----------------------------------------------------------------- classify

// batch_over for one (component, obstacle) pair: any body intersects (engine_batch.cpp:55-74).
template <bool COUNT>
__device__ __forceinline__ bool over_test(const Store& s, int c, const double* osat, long long* cost) {
    bool hit = false;
    for (int b = 0; b < s.B; ++b) {
        const double* a = s.sat + (static_cast<size_t>(c) * s.B + b) * 22;
        double ar[21];
#pragma unroll
        for (int k = 0; k < 20; k += 2) {
            const double2 v = *reinterpret_cast<const double2*>(a + k);
            ar[k] = v.x;
            ar[k + 1] = v.y;
        }
        ar[20] = a[20];
        const bool h = rggd::sat_boxes<COUNT>(ar, osat, cost);
        hit = hit || h;
        if (hit && !COUNT) break;
    }
    return hit;
}

// batch_under for one pair (engine_batch.cpp:76-112): any real segment of any
// (body, slot) row within o_minus_r + spline_radius of any obstacle sphere.
template <bool COUNT>
__device__ __forceinline__ bool under_test(const Store& s, int c, const Event& ev, long long* tests) {
    const int rows = s.B * s.S;
    const int r0 = c * rows;
    bool hit = false;
    for (int rr = 0; rr < rows; ++rr) {
        const int k0 = s.row[r0 + rr], k1 = s.row[r0 + rr + 1];
        if (k0 == k1) continue;
        const double r_total = add(ev.r, s.spline_r[rr]);
        for (int k = k0; k < k1; ++k) {
            const double2* p = reinterpret_cast<const double2*>(s.seg + 8 * static_cast<size_t>(k));
            const double2 v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
            const double seg[7] = {v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, v3.x};
            for (int sp = 0; sp < ev.nsph; ++sp) {
                // the reference evaluates every (segment, sphere); the verdict is their OR
                if (COUNT) *tests += 1;
                if (rggd::seg_sphere(seg, ev.cen + 3 * sp, r_total)) {
                    hit = true;
                    if (!COUNT) return true;
                }
            }
        }
    }
    return hit;
}

// One CTA per dirty cell (persistent, dynamic cell queue), one thread per
// component.  Per chunk of <= 32 events staged in shared memory:
//   A. each thread builds its touch / box / sphere overlap masks over the chunk;
//   B. the CTA evaluates the narrow-test work list (over items, then under
//      items) with all its threads — the (component, event) pairs that
//      actually need a SAT or a segment-sphere test — into result masks;
//   C. each thread applies its events in move order with the reference's
//      per-move transition (engine_batch.cpp:114-188) from the result masks.
// B is where the fp64 work is; spreading it over the CTA keeps the lanes busy
// where the v1 event loop left 18 of 32 idle (profiles/r1_v1_summary.md).
// One lane's share (segments g, g+G, ...) of batch_under for one pair.  A
// component's real segments are contiguous (rows (c, b, s) in order), so the
// lanes walk [row[c*B*S], row[(c+1)*B*S]) and look up each segment's row for
// its slot radius (engine_batch.cpp:97).
template <bool COUNT>
__device__ __forceinline__ bool under_part(const Store& s, int c, const Event& ev, int g, int G, long long* tests) {
    const int rows = s.B * s.S;
    const int r0 = c * rows;
    const int lo = s.row[r0], hi = s.row[r0 + rows];
    int rr = 0, rend = s.row[r0 + 1];
    bool hit = false;
    for (int j = lo + g; j < hi; j += G) {
        while (j >= rend) rend = s.row[r0 + (++rr) + 1];
        const double r_total = add(ev.r, s.spline_r[rr]);
        const double2* p = reinterpret_cast<const double2*>(s.seg + 8 * static_cast<size_t>(j));
        const double2 v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
        const double seg[7] = {v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, v3.x};
        for (int sp = 0; sp < ev.nsph; ++sp) {
            if (COUNT) *tests += 1;
            if (rggd::seg_sphere_fast(seg, ev.cen + 3 * sp, r_total)) {
                hit = true;
                if (!COUNT) return true;
            }
        }
    }
    return hit;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

constexpr int kUnderLanes = 4;  // lanes per under-approximation work item
constexpr int kOverLanes = 1;   // lanes per SAT work item (4 was slower: operands re-read per lane)

template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(kMaxCell, 4) classify_kernel(Store s, Batch b) {
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    constexpr bool HITS = (FLAGS & kHits) != 0;
    constexpr bool CENSUS = (FLAGS & kCensus) != 0;
    __shared__ Event sev[kEvChunk];
    __shared__ int scnt[kEvChunk][4];
    __shared__ uint32_t s_over[kMaxCell], s_under[kMaxCell];
    __shared__ uint16_t q_over[kMaxCell * kEvChunk], q_under[kMaxCell * kEvChunk];
    __shared__ int s_wo[kMaxCell / 32], s_wu[kMaxCell / 32];
    __shared__ int s_cell, s_no, s_nu;
    __shared__ unsigned long long scensus[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (CENSUS && tid < 8) scensus[tid] = 0;
    long long c_over_pairs = 0, c_sat = 0, c_under_pairs = 0, c_tests = 0, c_over_hits = 0, c_under_hits = 0,
              c_narrow = 0, c_narrow_segs = 0;
    unsigned long long t0 = 0;
    for (;;) {
        __syncthreads();
        if (b.dbg && tid == 0) t0 = gtimer();
        if (tid == 0) {
            const int di = atomicAdd(&b.ctr[2], 1);
            s_cell = di < b.ctr[0] ? b.dirty[di] : -1;
        }
        __syncthreads();
        const int cell = s_cell;
        if (cell < 0) break;
        unsigned long long* dbg = b.dbg ? b.dbg + 8 * static_cast<size_t>(cell) : nullptr;
        if (dbg && tid == 0) dbg[0] = t0, dbg[1] = gtimer();
        const int count = b.cell_count[cell];
        const int32_t* list = count <= s.cap ? b.cell_list + static_cast<size_t>(cell) * s.cap : b.pool + b.cell_ovf[cell];
        const int c = cell * s.cell + tid;
        const bool valid = c < s.Np;
        double aabb[6];
        int label = 0, oc = 0, bc = 0, id = -1;
        unsigned long long OW = 0, UW = 0;
        if (valid) {
            const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
            aabb[0] = a0.x, aabb[1] = a0.y, aabb[2] = a1.x, aabb[3] = a1.y, aabb[4] = a2.x, aabb[5] = a2.y;
            id = s.orig[c];
            label = s.state[id];
            const uint32_t cw = s.cnt[c];
            oc = cw & 0xffff;
            bc = cw >> 16;
            if (!WIDE) {
                OW = s.over[c];
                UW = s.under[c];
            }
        }
        const int label0 = label;
        const uint32_t cnt0 = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
        const unsigned long long OW0 = OW, UW0 = UW;
        bool hit_last = false, narrow_any = false;
        if (dbg) {
            __syncthreads();
            if (tid == 0) dbg[2] = gtimer(), dbg[7] = count;
        }
        int dgray = 0;
        for (int base = 0; base < count; base += kEvChunk) {
            const int m = min(kEvChunk, count - base);
            __syncthreads();
            {
                constexpr int kVec = sizeof(Event) / 16;
                for (int t = tid; t < m * kVec; t += blockDim.x) {
                    const int e = t / kVec, k = t % kVec;
                    reinterpret_cast<int4*>(&sev[e])[k] = reinterpret_cast<const int4*>(&b.ev[list[base + e]])[k];
                }
                if (PER_MOVE)
                    for (int t = tid; t < m * 4; t += blockDim.x) scnt[t >> 2][t & 3] = 0;
            }
            __syncthreads();
            if (dbg && tid == 0 && base == 0) dbg[3] = gtimer();
            // ---- A: overlap masks
            uint32_t tm = 0, bm = 0, sm = 0;
            if (valid) {
                for (int k = 0; k < m; ++k) {
                    const Event& ev = sev[k];
                    if (rggd::overlaps(aabb, ev.nu) || rggd::overlaps(aabb, ev.old)) {
                        tm |= 1u << k;
                        if (rggd::overlaps(aabb, ev.box)) bm |= 1u << k;
                        if (s.use_under && rggd::overlaps(aabb, ev.sph)) sm |= 1u << k;
                    }
                }
            }
            narrow_any = narrow_any || (bm | sm) != 0;
            if (bm) {
                const char* a = reinterpret_cast<const char*>(s.sat + static_cast<size_t>(c) * s.B * 22);
                for (int off = 0; off < s.B * 176; off += 128) prefetch_l2(a + off);
            }
            if (sm) {
                const int rows = s.B * s.S;
                const char* a = reinterpret_cast<const char*>(s.seg + 8 * static_cast<size_t>(s.row[c * rows]));
                const char* e = reinterpret_cast<const char*>(s.seg + 8 * static_cast<size_t>(s.row[(c + 1) * rows]));
                for (; a < e; a += 128) prefetch_l2(a);
            }
            s_over[tid] = 0;
            s_under[tid] = 0;
            // block-exclusive offsets of the work items
            const int no = __popc(bm), nu = __popc(sm);
            int xo = no, xu = nu;
            for (int off = 1; off < 32; off <<= 1) {
                const int yo = __shfl_up_sync(0xffffffffu, xo, off), yu = __shfl_up_sync(0xffffffffu, xu, off);
                if (lane >= off) xo += yo, xu += yu;
            }
            if (lane == 31) s_wo[warp] = xo, s_wu[warp] = xu;
            __syncthreads();
            if (tid == 0) {
                int ao = 0, au = 0;
                for (int w = 0; w < nwarps; ++w) {
                    const int to = s_wo[w], tu = s_wu[w];
                    s_wo[w] = ao, s_wu[w] = au;
                    ao += to, au += tu;
                }
                s_no = ao;
                s_nu = au;
            }
            __syncthreads();
            {
                int po = s_wo[warp] + xo - no, pu = s_wu[warp] + xu - nu;
                for (uint32_t x = bm; x; x &= x - 1) q_over[po++] = static_cast<uint16_t>((tid << 5) | (__ffs(x) - 1));
                for (uint32_t x = sm; x; x &= x - 1) q_under[pu++] = static_cast<uint16_t>((tid << 5) | (__ffs(x) - 1));
            }
            __syncthreads();
            if (dbg && tid == 0 && base == 0) dbg[4] = gtimer();
            // ---- B: narrow tests spread over the CTA
            const int n_over_items = s_no, n_under_items = s_nu;
            if (CENSUS) {
                for (int i = tid; i < n_over_items; i += blockDim.x) {
                    const int it = q_over[i], t = it >> 5, k = it & 31;
                    const bool h = over_test<true>(s, cell * s.cell + t, sev[k].sat, &c_sat);
                    c_over_pairs += s.B, c_over_hits += h;
                    if (h) atomicOr(&s_over[t], 1u << k);
                }
            } else {
                // over items on groups of kOverLanes lanes: the 15 axes split across the group
                const int g = tid % kOverLanes, groups = blockDim.x / kOverLanes;
                const unsigned gmask = ((1u << kOverLanes) - 1u) << (lane & ~(kOverLanes - 1));
                for (int ob = 0; ob < n_over_items; ob += groups) {
                    const int i = ob + tid / kOverLanes;
                    bool sep_all = true;  // over any body: hit iff some body is not separated
                    int t = 0, k = 0;
                    if (i < n_over_items) {
                        const int it = q_over[i];
                        t = it >> 5;
                        k = it & 31;
                        const double* osat = sev[k].sat;
                        const int c = cell * s.cell + t;
                        for (int bb = 0; bb < s.B; ++bb) {
                            bool sep = rggd::sat_separated_part(s.sat + (static_cast<size_t>(c) * s.B + bb) * 22, osat, g,
                                                                kOverLanes);
#pragma unroll
                            for (int off = 1; off < kOverLanes; off <<= 1) {
                                const bool other = __shfl_xor_sync(gmask, sep, off);  // the group's 4 lanes
                                sep = sep || other;
                            }
                            if (!sep) {
                                sep_all = false;
                                break;
                            }
                        }
                    }
                    if (i < n_over_items && g == 0 && !sep_all) atomicOr(&s_over[t], 1u << k);
                }
            }
            {
                // under items on groups of kUnderLanes lanes, taken from the top
                // thread index down so they overlap the over items above
                const int rt = blockDim.x - 1 - tid, g = rt % kUnderLanes, groups = blockDim.x / kUnderLanes;
                for (int ub = 0; ub < n_under_items; ub += groups) {
                    const int i = ub + rt / kUnderLanes;
                    bool h = false;
                    int t = 0, k = 0;
                    if (i < n_under_items) {
                        const int it = q_under[i];
                        t = it >> 5;
                        k = it & 31;
                        h = under_part<CENSUS>(s, cell * s.cell + t, sev[k], g, kUnderLanes, &c_tests);
                    }
#pragma unroll
                    for (int off = 1; off < kUnderLanes; off <<= 1) {
                        const bool other = __shfl_xor_sync(0xffffffffu, h, off);  // every lane must shuffle
                        h = h || other;
                    }
                    if (i < n_under_items && g == 0) {
                        if (CENSUS) c_under_pairs += 1, c_under_hits += h;
                        if (h) atomicOr(&s_under[t], 1u << k);
                    }
                }
            }
            __syncthreads();
            if (dbg && tid == 0 && base == 0) dbg[5] = gtimer();
            if (CENSUS) continue;
            // ---- C: transitions in move order
            const uint32_t ro = s_over[tid], ru = s_under[tid];
            for (int k = 0; k < m; ++k) {
                const int before = label;
                if ((tm >> k) & 1u) {
                    const Event& ev = sev[k];
                    const int w = ev.o >> 6;
                    const unsigned long long bit = 1ull << (ev.o & 63);
                    unsigned long long ow, uw;
                    if (WIDE) {
                        ow = s.over[static_cast<size_t>(w) * s.Np + c];
                        uw = s.under[static_cast<size_t>(w) * s.Np + c];
                    } else {
                        ow = OW;
                        uw = UW;
                    }
                    const bool old_over = (ow & bit) != 0, old_under = (uw & bit) != 0;
                    const bool n_over = (ro >> k) & 1u, n_under = (ru >> k) & 1u;
                    // revalidate_old_intersections (engine_batch.cpp:114-143)
                    if (old_over) {
                        oc -= 1;
                        const int rest = bc - (old_under ? 1 : 0);
                        label = oc == 0 ? 0 : ((s.use_under && rest > 0) ? 1 : 2);
                    }
                    // over phase (engine_batch.cpp:163-177)
                    if (n_over) {
                        if (label == 0) label = 2;
                        oc += 1;
                    }
                    // under phase (engine_batch.cpp:181-188)
                    if (n_under) label = 1;
                    bc += (n_over && n_under ? 1 : 0) - (old_over && old_under ? 1 : 0);
                    const unsigned long long nw = n_over ? (ow | bit) : (ow & ~bit);
                    const unsigned long long nuw = n_under ? (uw | bit) : (uw & ~bit);
                    if (WIDE) {
                        if (nw != ow) s.over[static_cast<size_t>(w) * s.Np + c] = nw;
                        if (nuw != uw) s.under[static_cast<size_t>(w) * s.Np + c] = nuw;
                    } else {
                        OW = nw;
                        UW = nuw;
                    }
                    if (HITS && ev.move == b.n - 1) hit_last = n_over;
                }
                if (PER_MOVE) {
                    const bool ch = label != before;
                    const unsigned g = __ballot_sync(0xffffffffu, ch && label == 0);
                    const unsigned r = __ballot_sync(0xffffffffu, ch && label == 1);
                    const unsigned y = __ballot_sync(0xffffffffu, ch && label == 2);
                    const unsigned f = __ballot_sync(0xffffffffu, ch && before == 2);
                    if (lane == 0 && (g | r | y | f)) {
                        if (g) atomicAdd(&scnt[k][0], __popc(g));
                        if (r) atomicAdd(&scnt[k][1], __popc(r));
                        if (y) atomicAdd(&scnt[k][2], __popc(y));
                        if (f) atomicAdd(&scnt[k][3], __popc(f));
                    }
                }
            }
            if (PER_MOVE) {
                __syncthreads();
                for (int t = tid; t < m * 4; t += blockDim.x) {
                    const int v = scnt[t >> 2][t & 3];
                    if (v) atomicAdd(&b.mv[4 * sev[t >> 2].move + (t & 3)], v);
                }
            }
        }
        if (CENSUS) {
            if (narrow_any && valid) {
                c_narrow += 1;
                c_narrow_segs += s.row[(c + 1) * s.B * s.S] - s.row[c * s.B * s.S];
            }
            continue;
        }
        if (valid) {
            if (label != label0) {
                s.state[id] = static_cast<uint8_t>(label);
                dgray = (label == 2) - (label0 == 2);
            }
            const uint32_t cw = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
            if (cw != cnt0) s.cnt[c] = cw;
            if (!WIDE) {
                if (OW != OW0) s.over[c] = OW;
                if (UW != UW0) s.under[c] = UW;
            }
        }
        if (dbg) {
            __syncthreads();
            if (tid == 0) dbg[6] = gtimer();
        }
        // running gray count (the unknown_count of the reference)
        for (int off = 16; off; off >>= 1) dgray += __shfl_down_sync(0xffffffffu, dgray, off);
        if (lane == 0 && dgray) atomicAdd(b.unknown, dgray);
        if (HITS) {
            const bool h = valid && hit_last && label == 2;
            const unsigned bal = __ballot_sync(0xffffffffu, h);
            int pos = 0;
            if (lane == 0 && bal) pos = atomicAdd(&b.ctr[5], __popc(bal));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (h) b.hits[pos + __popc(bal & ((1u << lane) - 1u))] = id;
        }
    }
    if (CENSUS) {
        long long v[8] = {c_over_pairs, c_sat, c_under_pairs, c_tests, c_over_hits, c_under_hits, c_narrow,
                          c_narrow_segs};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&scensus[k], static_cast<unsigned long long>(x));
        }
        __syncthreads();
        if (tid < 8 && scensus[tid]) atomicAdd(&b.census[tid], scensus[tid]);
    }
}

// Commit the moved obstacles' operands (one warp per move, 16-byte lanes).
__global__ void commit_kernel(Store s, Batch b) {
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= b.n || !b.last[i]) return;
    const int o = b.ids[i];
    constexpr int kVec = sizeof(Event) / 16;
    const int4* src = reinterpret_cast<const int4*>(&b.ev[i]);
    int4* dst = reinterpret_cast<int4*>(&s.cur[o]);
    for (int k = lane; k < kVec; k += 32) dst[k] = src[k];
    if (lane < 6) s.cur_union[6 * o + lane] = b.ev[i].nu[lane];
}

// --------------------------------------------------------------- compaction

constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 16;  // labels per thread (one uint4)
constexpr int kTile = kCompactThreads * kCompactPer;

__device__ __forceinline__ int gray_count16(uint4 v) {
    // a byte equals 2 (GRAY) iff it is 0x02; count such bytes
    int n = 0;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t x = w[i] ^ 0x02020202u;  // zero byte where label == 2
        const uint32_t z = (x - 0x01010101u) & ~x & 0x80808080u;
        n += __popc(z);
    }
    return n;
}

__device__ __forceinline__ uint4 load_labels(const uint8_t* st, int N, int base) {
    if (base + 16 <= N && (reinterpret_cast<uintptr_t>(st + base) & 15) == 0)
        return *reinterpret_cast<const uint4*>(st + base);
    uint8_t tmp[16];
    for (int i = 0; i < 16; ++i) tmp[i] = base + i < N ? st[base + i] : 0;
    return *reinterpret_cast<uint4*>(tmp);
}

__global__ void __launch_bounds__(kCompactThreads) gray_count_kernel(const uint8_t* st, int N, int32_t* tile_cnt) {
    const int base = blockIdx.x * kTile + threadIdx.x * kCompactPer;
    const int n = base < N ? gray_count16(load_labels(st, N, base)) : 0;
    int x = n;
    for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
    __shared__ int ws[kCompactThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < kCompactThreads / 32; ++i) t += ws[i];
        tile_cnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kCompactThreads) gray_write_kernel(const uint8_t* st, int N, const int32_t* tile_cnt,
                                                                     int ntiles, int32_t* out, int32_t* gray_n) {
    __shared__ int ws[kCompactThreads / 32];
    __shared__ int s_base;
    // tile base = sum of earlier tiles
    int acc = 0;
    for (int t = threadIdx.x; t < blockIdx.x; t += kCompactThreads) acc += tile_cnt[t];
    for (int off = 16; off; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int i = 0; i < kCompactThreads / 32; ++i) t += ws[i];
        s_base = t;
        if (blockIdx.x == ntiles - 1) *gray_n = t + tile_cnt[blockIdx.x];
    }
    __syncthreads();
    const int base = blockIdx.x * kTile + threadIdx.x * kCompactPer;
    uint4 v = base < N ? load_labels(st, N, base) : make_uint4(0, 0, 0, 0);
    const int n = base < N ? gray_count16(v) : 0;
    // block-exclusive scan of n
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = n;
    for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    __syncthreads();
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kCompactThreads / 32 ? ws[lane] : 0;
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        if (lane < kCompactThreads / 32) ws[lane] = w;
    }
    __syncthreads();
    int pos = s_base + x - n + (warp > 0 ? ws[warp - 1] : 0);
    if (n) {
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
        for (int i = 0; i < 16; ++i)
            if (b[i] == 2) out[pos++] = base + i;
    }
}

__global__ void write_states_kernel(uint8_t* state, const int32_t* ids, const uint8_t* st, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) state[ids[i]] = st[i];
}

__global__ void pair_masks_kernel(Store s, const int32_t* rank, int kind, const int32_t* cand, int n, int o,
                                  uint8_t* mask) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = rank[cand[i]];
    if (c < 0) {
        mask[i] = 0;
        return;
    }
    const Event& ev = s.cur[o];
    bool h;
    if (kind == 0) {
        double osat[21];
        for (int k = 0; k < 21; ++k) osat[k] = ev.sat[k];
        h = over_test<false>(s, c, osat, nullptr);
    } else {
        h = under_test<false>(s, c, ev, nullptr);
    }
    mask[i] = h ? 1 : 0;
}

// Non-FMA fp64 issue-rate probe: 8 independent mul/add chains per thread.
__global__ void fp64_peak_kernel(double* sink, int iters) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = 1.0 + 1e-9 * (threadIdx.x + k);
    const double a = 0.999999999, c = 1e-12;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(__dmul_rn(x[k], a), c);
    }
    double t = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += x[k];
    if (t == 12345.0) sink[0] = t;
}

}  // namespace

// ------------------------------------------------------------------ launchers

cudaError_t launch_pose(const Store& s, const Batch& b, cudaStream_t st) {
    const int warps = 4;  // moves per CTA
    pose_kernel<<<(b.n + warps - 1) / warps, 32 * warps, 0, st>>>(s, b);
    return cudaGetLastError();
}

cudaError_t launch_init_obstacles(const Store& s, Event*, cudaStream_t st) {
    if (s.M == 0) return cudaSuccess;
    init_obstacles_kernel<<<(s.M + 127) / 128, 128, 0, st>>>(s);
    return cudaGetLastError();
}

cudaError_t launch_bin(const Store& s, const Batch& b, cudaStream_t st) {
    const int cells_per = kBinThreads / 32;
    bin_kernel<<<(s.ncells + cells_per - 1) / cells_per, kBinThreads, 0, st>>>(s, b);
    return cudaGetLastError();
}

template <int F, bool W>
static cudaError_t classify_t(const Store& s, const Batch& b, int grid, cudaStream_t st) {
    classify_kernel<F, W><<<grid, s.cell, 0, st>>>(s, b);
    return cudaGetLastError();
}

cudaError_t launch_classify(const Store& s, const Batch& b, int flags, int grid, cudaStream_t st) {
    const bool wide = s.W > 1;
    const int f = flags & (kPerMove | kHits | kCensus);
#define RGG_CASE(F)                                                           \
    case F:                                                                   \
        return wide ? classify_t<F, true>(s, b, grid, st) : classify_t<F, false>(s, b, grid, st);
    switch (f) {
        RGG_CASE(0)
        RGG_CASE(kPerMove)
        RGG_CASE(kHits)
        RGG_CASE(kPerMove | kHits)
        case kCensus:
        case kCensus | kPerMove:
        case kCensus | kHits:
        case kCensus | kPerMove | kHits:
            return wide ? classify_t<kCensus, true>(s, b, grid, st) : classify_t<kCensus, false>(s, b, grid, st);
    }
#undef RGG_CASE
    return cudaErrorInvalidValue;
}

int classify_occupancy(int cell, int flags) {
    int n = 0;
    if (flags & kCensus)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, classify_kernel<kCensus, false>, cell, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, classify_kernel<kPerMove, false>, cell, 0);
    return n < 1 ? 1 : n;
}

cudaError_t launch_commit(const Store& s, const Batch& b, cudaStream_t st) {
    commit_kernel<<<(b.n + 3) / 4, 128, 0, st>>>(s, b);
    return cudaGetLastError();
}

cudaError_t launch_compact(const Store& s, int32_t* out_ids, int32_t* tile_cnt, int32_t* gray_n, cudaStream_t st) {
    const int ntiles = (s.N + kTile - 1) / kTile;
    if (ntiles == 0) return cudaMemsetAsync(gray_n, 0, sizeof(int32_t), st);
    gray_count_kernel<<<ntiles, kCompactThreads, 0, st>>>(s.state, s.N, tile_cnt);
    gray_write_kernel<<<ntiles, kCompactThreads, 0, st>>>(s.state, s.N, tile_cnt, ntiles, out_ids, gray_n);
    return cudaGetLastError();
}

cudaError_t launch_write_states(const Store& s, const int32_t* ids, const uint8_t* st_in, int n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    write_states_kernel<<<(n + 255) / 256, 256, 0, st>>>(s.state, ids, st_in, n);
    return cudaGetLastError();
}

cudaError_t launch_pair_masks(const Store& s, const int32_t* rank, int kind, const int32_t* cand, int n, int o,
                              uint8_t* mask, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    pair_masks_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, rank, kind, cand, n, o, mask);
    return cudaGetLastError();
}

cudaError_t launch_fp64_peak(double* sink, int iters, int grid, int block, cudaStream_t st) {
    fp64_peak_kernel<<<grid, block, 0, st>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace rggk
