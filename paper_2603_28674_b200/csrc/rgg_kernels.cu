// rgg_kernels.cu — the SerRGG update pipeline for sm_100a.
//
// One update = one CUDA graph of programmatically dependent launches:
//   pose          one warp per move: BatchLayout::update_transforms
//                 (proj/src/batch_layout.cpp:148-172) on the device, fp64-exact; the
//                 event boxes (widened by 2^-40), SAT operands, Box32 filter line and the
//                 fp32 sphere operands of every move.
//   bin           bin_scatter_kernel (a CTA per event over a uniform grid of the cell
//                 boxes, event bitmask per cell; below 512 moves it derives the event's
//                 boxes itself, overlapping the pose kernel) + bin_cells_kernel (a warp per cell:
//                 ordered lists by popcount / prefix scan, fixed capacity + overflow
//                 pool, work units), or bin_small_kernel for <= 64 moves.  Replaces
//                 SpatialGrid::build / candidates (proj/src/spatial_grid.cpp:50-135).
//   touch         touch_cta_kernel: a CTA per cell chunk, a warp per 32-component slice:
//                 the closed AABB tests that decide which (component, event) pairs need
//                 the narrow tests, queued as over / under items.
//   narrow        narrow_over_kernel (the 15-axis SAT, kernels_scalar.cpp:37-69) and
//                 narrow_under_kernel (segment-sphere, :81-96): fp32 filters with
//                 rigorous bounds, the reference's fp64 sequence for undecided pairs
//                 (undecided SAT pairs queued, then a warp each in narrow_under's tail).
//   apply         apply_warp_kernel: a warp per slice, the reference's per-move
//                 transitions in move order (engine_batch.cpp:114-188), per-move
//                 report counters, the moved obstacles' operands committed.
//   compact       gray_count / gray_write: ordered compaction of the GRAY ids.
// Single moves (update_obstacle, eager updates) run single_cells_kernel after pose
// instead of bin .. apply.
#include <cstdio>
#include <cstdlib>

#include "rgg_device.cuh"
#include "rgg_kernels.cuh"

namespace rggk {

using rggd::add;
using rggd::mul;
using rggd::sub;

namespace {

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; pdl_wait() blocks until the predecessor's writes are
// visible, pdl_trigger() lets the successor's CTAs be scheduled early.
// Both are no-ops for ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// In-kernel handoffs (Batch::evready, unit_ready) spin on counters another kernel
// raises; a spin that outlasts ~1 s (2^23 polls with back-off) gives up with status 4
// (ctr[6]) instead of hanging the GPU, and the host fails the update.
__device__ __forceinline__ bool handoff_timeout(const Batch& b, unsigned spins) {
    if (spins < (1u << 23)) return false;
    atomicExch(&b.ctr[6], 4);
    return true;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Update timeline (RGG_DEBUG_TIMELINE): per kernel k, 8 words at b.tl + 8k:
// ~first start, last start, ~first end, last end, sum of warp durations, warps
// (all max-reduced from zero; "first" stored complemented).
__device__ __forceinline__ unsigned long long tl_start(const unsigned long long* tl) { return tl ? gtimer() : 0; }
__device__ __forceinline__ void tl_stop(unsigned long long* tl, int k, unsigned long long t0) {
    if (!tl || (threadIdx.x & 31) != 0) return;
    const unsigned long long t1 = gtimer();
    unsigned long long* p = tl + 8 * k;
    atomicMax(p + 0, ~t0);
    atomicMax(p + 1, t0);
    atomicMax(p + 2, ~t1);
    atomicMax(p + 3, t1);
    atomicAdd(p + 4, t1 - t0);
    atomicAdd(p + 5, 1ull);
}

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

// The candidate filter's widening of an obstacle box face: 2^-40 relative (plus 2^-40
// absolute near zero), far above the fp64 rounding of the SAT margins and the AABB
// corners (~1e-16 relative) and far below any geometric scale.  +-inf (empty boxes)
// stay as they are.
__device__ __forceinline__ double widen_lo(double v) { return isfinite(v) ? v - (fabs(v) + 1.0) * 0x1p-40 : v; }
__device__ __forceinline__ double widen_hi(double v) { return isfinite(v) ? v + (fabs(v) + 1.0) * 0x1p-40 : v; }

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

constexpr int kBinSmallMax = 64;  // bin_small_kernel takes batches up to this many moves

__global__ void pose_kernel(Store s, Batch b) {
    const unsigned long long t0 = tl_start(b.tl);
    pdl_trigger();  // the bin kernel's CTAs may land now; they wait for these events in pdl_wait()
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i == 0 && lane < 16) {
        b.ctr[lane] = 0;
        b.census[lane] = 0;
        if (lane < 4) b.ctr[20 + lane] = 0;  // eager resolve report deltas
        if (lane == 0) *b.mtop = 0;
        if (lane == 0 && b.unit_ready) b.evready[4] += 1;  // this update's generation (released below)
    }
    if (i >= b.n) return;
    // moves straight from mapped host memory (synchronous host updates) or from HBM
    const int32_t* mids = b.src_ids ? b.src_ids : b.ids;
    const double* mrt = b.src_ids ? b.src_rt : b.rt;
    const double* rt_new = mrt + 12 * static_cast<size_t>(i);
    double rtl[12];  // the move's pose does not depend on its id: both loads in flight together
#pragma unroll
    for (int k = 0; k < 12; ++k) rtl[k] = rt_new[k];
    const int o = mids[i];
    // prev / last links: the same obstacle moved earlier / later in this batch
    int p = -1;
    bool is_last = true;
    for (int base = 0; base < b.n; base += 256) {  // eight ids per lane in flight, then the ballots
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + 32 * u + lane;
            v[u] = j < b.n ? mids[j] : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + 32 * u + lane;
            const bool same = v[u] == o;
            const unsigned before = __ballot_sync(0xffffffffu, same && j < i);
            const unsigned after = __ballot_sync(0xffffffffu, same && j > i);
            if (before) p = base + 32 * u + 31 - __clz(before);
            if (after) is_last = false;
        }
    }
    const double he[3] = {s.ohe[3 * o], s.ohe[3 * o + 1], s.ohe[3 * o + 2]};
    const double cu = lane < 6 ? s.cur_union[6 * o + lane] : 0.0;  // the old union box when p < 0
    const double* rt_old = p >= 0 ? mrt + 12 * static_cast<size_t>(p) : rt_new;
    if (p >= 0 && lane >= 8 && lane < 16)  // lanes 8-15 place the old corners
#pragma unroll
        for (int k = 0; k < 12; ++k) rtl[k] = rt_old[k];
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
    // boxes: new corners on lane 0, old corners on lane 8, spheres on lane 16, each
    // widened by a relative 2^-40 (candidate_widen): the reference tests every grid
    // candidate, and the fp64 SAT / segment-sphere test can report contact for a pair
    // whose exact AABBs miss by an ulp, so the AABB filter keeps those pairs too
    double bn[6], bo[6], bs[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        bn[k] = widen_lo(shfl(lo[k], 0)), bn[3 + k] = widen_hi(shfl(hi[k], 0));
        bo[k] = widen_lo(shfl(lo[k], 8)), bo[3 + k] = widen_hi(shfl(hi[k], 8));
        bs[k] = widen_lo(shfl(lo[k], 16)), bs[3 + k] = widen_hi(shfl(hi[k], 16));
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
            os[k] = fmin(bo[k], widen_lo(olo[k]));
            os[3 + k] = fmax(bo[3 + k], widen_hi(ohi[k]));
        }
    }
    // the binning boxes first: the bin kernel starts on them (Batch::evready)
    double nu6 = 0.0, ol6 = 0.0;
    if (lane < 6) {
        nu6 = lane < 3 ? fmin(bn[lane], bs[lane]) : fmax(bn[lane], bs[lane]);
        ol6 = p >= 0 ? os[lane] : cu;
        b.evbox[12 * static_cast<size_t>(i) + lane] = nu6;  // compact copy for the binning
        b.evbox[12 * static_cast<size_t>(i) + 6 + lane] = ol6;
    }
    // release: the warp's stores (evbox, and the counter resets of warp 0), then the count; only
    // bin_small_kernel and the touch on published units poll it (bin_scatter takes the PDL wait)
    if (b.evready && (b.n <= kBinSmallMax || b.unit_ready)) {
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(b.evready, 1);
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
            for (int k = 0; k < 3; ++k) u[k] = rggd::div_pos(e[k], len);
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
    __syncwarp();
    if (lane == 0) {  // the filter operands of the obstacle box
        rggd::box32_terms(ev.sat, ev.b32);
        for (int k = 0; k < 3; ++k) ev.b32.c[k] = ev.sat[k];
    }
    if (lane < 6) {
        ev.box[lane] = bn[lane];
        ev.sph[lane] = bs[lane];
        ev.nu[lane] = nu6;
        ev.old[lane] = ol6;
        double* et = b.evt + 24 * static_cast<size_t>(i);
        et[lane] = nu6, et[6 + lane] = ol6, et[12 + lane] = bn[lane], et[18 + lane] = bs[lane];
    }
    double rtk = 0.0;  // the new pose's element k on lane k (lane 0 holds it in registers)
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const double v = shfl(rtl[k], 0);
        if (lane == k) rtk = v;
    }
    if (lane < 12) ev.rt[lane] = rtk;
    if (b.src_ids) {  // the HBM copy the later kernels (and a replay) read
        if (lane == 0) const_cast<int32_t*>(b.ids)[i] = o;
        if (lane < 12) const_cast<double*>(b.rt)[12 * static_cast<size_t>(i) + lane] = rtk;
    }
    if (lane >= 16 && lane - 16 < nsph) {
        ev.cen[3 * (lane - 16)] = pt[0];
        ev.cen[3 * (lane - 16) + 1] = pt[1];
        ev.cen[3 * (lane - 16) + 2] = pt[2];
        const float cx = __double2float_rn(pt[0]), cy = __double2float_rn(pt[1]), cz = __double2float_rn(pt[2]);
        b.evs[kEvS * static_cast<size_t>(i) + 1 + (lane - 16)] = make_float4(cx, cy, cz, (fabsf(cx) + fabsf(cy)) + fabsf(cz));
    }
    if (lane == 0) b.evs[kEvS * static_cast<size_t>(i)] = make_float4(__double2float_rn(r), __int_as_float(nsph), 0.0f, 0.0f);
    if (lane == 0) {
        ev.r = r;
        ev.o = o;
        ev.nsph = nsph;
        ev.move = i;
        b.last[i] = is_last ? 1 : 0;
        reinterpret_cast<int4*>(b.mv)[i] = make_int4(0, 0, 0, 0);
    }
    if (b.unit_ready) {  // release this event's operands to the touch kernel
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(b.evready + 1, 1);
        }
    }
    tl_stop(b.tl, 0, t0);
}

// The binning boxes of move i (Batch::evbox: the new box U spheres, then the old), by one
// warp with pose_kernel's exact operations, so bin_scatter_kernel starts without waiting for
// the pose kernel (lanes < 6 store out[lane] and out[6 + lane]).
__device__ __forceinline__ void binning_boxes_warp(const Store& s, const Batch& b, int i, int lane, double* out) {
    const int32_t* mids = b.src_ids ? b.src_ids : b.ids;
    const double* mrt = b.src_ids ? b.src_rt : b.rt;
    const double* rt_new = mrt + 12 * static_cast<size_t>(i);
    double rtl[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) rtl[k] = rt_new[k];
    const int o = mids[i];
    int p = -1;
    for (int base = 0; base < b.n; base += 256) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + 32 * u + lane;
            v[u] = j < b.n ? mids[j] : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int j = base + 32 * u + lane;
            const unsigned before = __ballot_sync(0xffffffffu, v[u] == o && j < i);
            if (before) p = base + 32 * u + 31 - __clz(before);
        }
    }
    const double he[3] = {s.ohe[3 * o], s.ohe[3 * o + 1], s.ohe[3 * o + 2]};
    const double cu = lane < 6 ? s.cur_union[6 * o + lane] : 0.0;
    const double* rt_old = p >= 0 ? mrt + 12 * static_cast<size_t>(p) : rt_new;
    if (p >= 0 && lane >= 8 && lane < 16)
#pragma unroll
        for (int k = 0; k < 12; ++k) rtl[k] = rt_old[k];
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
    double bn[6], bo[6], bs[6];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        bn[k] = widen_lo(shfl(lo[k], 0)), bn[3 + k] = widen_hi(shfl(hi[k], 0));
        bo[k] = widen_lo(shfl(lo[k], 8)), bo[3 + k] = widen_hi(shfl(hi[k], 8));
        bs[k] = widen_lo(shfl(lo[k], 16)), bs[3 + k] = widen_hi(shfl(hi[k], 16));
    }
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
            os[k] = fmin(bo[k], widen_lo(olo[k]));
            os[3 + k] = fmax(bo[3 + k], widen_hi(ohi[k]));
        }
    }
    if (lane < 6) {
        out[lane] = lane < 3 ? fmin(bn[lane], bs[lane]) : fmax(bn[lane], bs[lane]);
        out[6 + lane] = p >= 0 ? os[lane] : cu;
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
    rggd::box32_terms(e.sat, e.b32);
    for (int k = 0; k < 3; ++k) e.b32.c[k] = e.sat[k];

    e.r = s.osr[o];
    e.o = o;
    e.nsph = nsph;
    e.move = -1;
    for (int k = 0; k < 12; ++k) e.rt[k] = id[k];
    aabb_union(e.box, e.sph, e.nu);
    aabb_empty(e.old);
    aabb_empty(s.cur_union + 6 * o);
}

// Commit the moved obstacles' operands for the next batch (s.cur, s.cur_union):
// one 16-byte word per thread over the whole grid.  Nothing between the pose
// kernel and the end of the update reads s.cur / s.cur_union.
__device__ __forceinline__ void commit_grid(const Store& s, const Batch& b) {
    constexpr int kVec = sizeof(Event) / 16 + 1;  // + the 6-double union box
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    for (int w = gt; w < b.n * kVec; w += gridDim.x * blockDim.x) {
        const int i = w / kVec, k = w % kVec;
        if (!b.last[i]) continue;
        const int o = b.ids[i];
        if (k < kVec - 1)
            reinterpret_cast<int4*>(&s.cur[o])[k] = reinterpret_cast<const int4*>(&b.ev[i])[k];
        else
            for (int j = 0; j < 6; ++j) s.cur_union[6 * o + j] = b.ev[i].nu[j];
    }
}

// ------------------------------------------------------------------ binning
//
// Event-centric counting sort of the events into the cells' lists (replaces
// SpatialGrid::build / candidates, proj/src/spatial_grid.cpp:50-135):
//   bin_scatter_kernel  one warp per event: the bins of a uniform grid over the
//                       cell boxes (Store::gcell*) that the event's new and old
//                       union boxes cover; the lanes test those bins' cells
//                       (closed fp64 box test) and set bit e of each overlapping
//                       cell's event mask (atomicOr);
//   bin_cells_kernel    one warp per cell: popcount + warp prefix scan of the
//                       cell's mask words gives the count and every event's list
//                       position, so the list is written in move order without
//                       a sort; then the fixed-capacity list (overflow -> pool),
//                       the dirty list and the cell's touch work units.
// Work is O(events x bins x cells per bin + cells x n/32), not O(cells x events).

// The per-cell records of the CTA's listed cells (WARPS cells per CTA, one warp
// each; every warp of the CTA calls this, count = 0 past the last cell): count,
// the 16-byte cell record {count, mask base, list address}, one touch work unit
// per chunk of 32 listed events, and the unit stamps of the early-touch handoff.
// The dirty count and the unit list are reserved with one atomic per CTA; each
// cell's mask block (3 * ceil(count/32) words per component) sits at a fixed
// offset of the mask pool, sized for the batch capacity.
template <int WARPS>
__device__ __forceinline__ void bin_cells_tail(const Store& s, const Batch& b, int cell, int count,
                                               const int32_t* inl, int lane, int warp) {
    __shared__ int s_units[WARPS];
    __shared__ int s_ub;
    const int W = (count + 31) >> 5;
    if (lane == 0) s_units[warp] = W;
    __syncthreads();  // also orders every lane's list entries before the stamps below
    if (threadIdx.x == 0) {
        int tot = 0, nd = 0;
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            const int t = s_units[w];
            s_units[w] = tot;
            tot += t;
            nd += t > 0;
        }
        s_ub = tot ? atomicAdd(&b.ctr[10], tot) : 0;
        if (nd) atomicAdd(&b.ctr[0], nd);
    }
    __syncthreads();
    if (cell >= s.ncells) return;
    const int ub = s_ub + s_units[warp];
    const int mbase = cell * 3 * s.cell * b.cmask_words;
    if (lane == 0) {
        b.cell_count[cell] = count;
        const int32_t* list = count <= s.cap ? inl : b.pool + b.cell_ovf[cell];
        const unsigned long long a = reinterpret_cast<unsigned long long>(list);
        b.crec[cell] = make_int4(count, mbase, static_cast<int>(a & 0xffffffffu), static_cast<int>(a >> 32));
    }
    for (int w = lane; w < W && ub + w < b.units_cap; w += 32) b.units[ub + w] = make_int4(cell, w, count, mbase);
    if (b.unit_ready && count > 0) {  // release the cell's units (record, list, mask base) to touch
        __syncwarp();
        const int gen = reinterpret_cast<volatile int32_t*>(b.evready)[4];
        __threadfence();
        for (int w = lane; w < W && ub + w < b.units_cap; w += 32) b.unit_ready[ub + w] = gen;
    }
}

// a cell's warp has released all its units (touch on published units waits for
// every cell: Batch::bin_warps = ncells)
__device__ __forceinline__ void bin_warp_done(const Batch& b, int lane) {
    if (!b.unit_ready) return;
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        atomicAdd(b.evready + 2, 1);
    }
}

__device__ __forceinline__ int grid_bin(const Store& s, double v, int k) {
    const double f = floor((v - s.gorg[k]) * s.ginv[k]);
    return f < 0.0 ? 0 : (f >= s.gdim[k] ? s.gdim[k] - 1 : static_cast<int>(f));
}

// Waits until the pose warps have published every event's binning boxes
// (Batch::evready: release by each pose warp, acquire here), else the whole pose kernel.
__device__ __forceinline__ void wait_event_boxes(const Batch& b) {
    if (b.evready) {
        pdl_trigger();
        if (threadIdx.x == 0) {
            for (unsigned spins = 0;; ++spins) {
                int r;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(b.evready) : "memory");
                if (r >= b.n || handoff_timeout(b, spins)) break;
                __nanosleep(32);
            }
        }
        __syncthreads();
    } else {
        pdl_wait();
        pdl_trigger();
    }
}

// One CTA per event.  For each of the event's two boxes the CTA flattens the
// (bin, cell) entries of the bins the box covers: the bins' entry counts are
// scanned in shared memory, then every thread takes entries, so a box's ~10^2-10^3
// entries cost about three memory round trips.  A cell listed in several of the
// box's bins is tested in one of them only: the bin at the low corner of the
// intersection of the cell's and the box's bin ranges (the cell's low bin rides in
// its grid entry).
constexpr int kScatterThreads = 256;
constexpr int kScatterSelfBox = 512;  // batches below this many moves: bin_scatter_kernel<true>

template <bool SELF_BOX>
__global__ void __launch_bounds__(kScatterThreads) bin_scatter_kernel(Store s, Batch b) {
    // a plain PDL wait for the pose kernel: a thousand CTAs polling the pose warps' count
    // (Batch::evready) slowed those warps' own release atomics more than it saved
    // SELF_BOX (batches under kScatterSelfBox moves): no wait for the pose kernel; warp 0
    // derives this event's binning boxes itself with the pose kernel's operations
    // (binning_boxes_warp), and the grid waits for the pose kernel only before it exits, so
    // the next kernels' waits still cover the pose kernel's outputs.  Larger batches wait
    // and read the pose kernel's boxes (a thousand CTAs redoing the pose work cost more
    // than the overlap saves).
    if (!SELF_BOX) pdl_wait();
    pdl_trigger();
    const unsigned long long t0 = tl_start(b.tl);
    __shared__ int s_pre[kScatterThreads + 1];
    __shared__ int s_tot;
    __shared__ double s_bx[12];
    const int tid = threadIdx.x;
    const int e = blockIdx.x;
    if (SELF_BOX) {
        if (tid < 32) binning_boxes_warp(s, b, e, tid, s_bx);
    } else if (tid < 12) {
        s_bx[tid] = b.evbox[12 * static_cast<size_t>(e) + tid];
    }
    __syncthreads();
    double bx[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) bx[k] = s_bx[k];
    uint32_t* col = b.cmask + (e >> 5);
    const uint32_t bit = 1u << (e & 31);
    for (int h = 0; h < 2; ++h) {
        const double* q = bx + 6 * h;
        if (!(q[0] <= q[3] && q[1] <= q[4] && q[2] <= q[5])) continue;  // empty (inactive obstacle)
        if (h == 1 && q[0] >= bx[0] && q[1] >= bx[1] && q[2] >= bx[2] && q[3] <= bx[3] && q[4] <= bx[4] && q[5] <= bx[5])
            continue;  // the old box lies inside the new one
        const int x0 = grid_bin(s, q[0], 0), x1 = grid_bin(s, q[3], 0);
        const int y0 = grid_bin(s, q[1], 1), y1 = grid_bin(s, q[4], 1);
        const int z0 = grid_bin(s, q[2], 2), z1 = grid_bin(s, q[5], 2);
        const int nx = x1 - x0 + 1, ny = y1 - y0 + 1, nb = nx * ny * (z1 - z0 + 1);
        for (int b0 = 0; b0 < nb; b0 += kScatterThreads) {  // bins in passes of one per thread
            const int nbp = min(kScatterThreads, nb - b0);
            int lo = 0, cnt = 0;
            if (tid < nbp) {
                const int i = b0 + tid;
                const int g = ((z0 + i / (nx * ny)) * s.gdim[1] + y0 + (i / nx) % ny) * s.gdim[0] + x0 + i % nx;
                lo = s.gcell_off[g];
                cnt = s.gcell_off[g + 1] - lo;
            }
            // exclusive scan of the bins' entry counts
            int x = cnt;
            const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, off);
                if (lane >= off) x += y;
            }
            __syncthreads();  // the previous pass's readers of s_pre are done
            if (lane == 31) s_pre[warp] = x;
            __syncthreads();
            if (tid == 0) {
                int acc = 0;
                for (int w = 0; w < kScatterThreads / 32; ++w) {
                    const int t = s_pre[w];
                    s_pre[w] = acc;
                    acc += t;
                }
                s_tot = acc;
            }
            __syncthreads();
            const int excl = s_pre[warp] + x - cnt;
            const int tot = s_tot;
            __syncthreads();
            if (tid < nbp) s_pre[tid] = excl;
            s_pre[kScatterThreads] = tot;  // (every thread stores the same value)
            __shared__ int s_lo[kScatterThreads];
            if (tid < nbp) s_lo[tid] = lo;
            __syncthreads();
            for (int j = tid; j < tot; j += kScatterThreads) {
                // the bin of entry j: the last bin whose exclusive prefix is <= j
                int a = 0, z = nbp - 1;
                while (a < z) {
                    const int mid = (a + z + 1) >> 1;
                    if (s_pre[mid] <= j) a = mid;
                    else z = mid - 1;
                }
                const int i = b0 + a;
                const int xb = x0 + i % nx, yb = y0 + (i / nx) % ny, zb = z0 + i / (nx * ny);
                const int2 ent = s.gcell[s_lo[a] + j - s_pre[a]];  // {cell, low bin x | y << 10 | z << 20}
                const int c = ent.x;
                if (xb != max(ent.y & 1023, x0) || yb != max((ent.y >> 10) & 1023, y0) ||
                    zb != max((ent.y >> 20) & 1023, z0))
                    continue;
                const double* cb = s.cell_aabb + 6 * static_cast<size_t>(c);
                double cbox[6];
#pragma unroll
                for (int k = 0; k < 6; ++k) cbox[k] = cb[k];
                if (rggd::overlaps(cbox, q)) atomicOr(col + static_cast<size_t>(c) * b.cmask_words, bit);
            }
        }
    }
    tl_stop(b.tl, 9, t0);
    if (SELF_BOX) pdl_wait();  // the pose kernel is complete before this grid is
}

constexpr int kCellWarps = 32;

__global__ void __launch_bounds__(32 * kCellWarps) bin_cells_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
    pdl_wait();
    pdl_trigger();
    tl_stop(b.tl, 10, tw);
    const unsigned long long t0 = tl_start(b.tl);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int cell = blockIdx.x * kCellWarps + warp;
    const bool live = cell < s.ncells;
    uint32_t* m = b.cmask + static_cast<size_t>(live ? cell : 0) * b.cmask_words;
    const int nw = live ? (b.n + 31) >> 5 : 0;
    // count: popcounts of the mask words (lane j: words j, j + 32, ...)
    int count = 0;
    for (int w = lane; w < nw; w += 32) count += __popc(m[w]);
    count = __reduce_add_sync(0xffffffffu, count);
    int32_t* inl = b.cell_list + static_cast<size_t>(cell) * s.cap;
    int32_t* dst = inl;
    int lim = count;
    if (count > s.cap) {  // the ordered list goes to the overflow pool
        int pbase = 0;
        if (lane == 0) {
            pbase = atomicAdd(&b.ctr[1], count);
            atomicAdd(&b.ctr[3], 1);
        }
        pbase = __shfl_sync(0xffffffffu, pbase, 0);
        if (pbase + count > b.pool_cap) {
            if (lane == 0) atomicExch(&b.ctr[6], 1);
            lim = count = s.cap;  // truncated: reported as an error by the host
        } else {
            dst = b.pool + pbase;
            if (lane == 0) b.cell_ovf[cell] = pbase;
        }
    }
    if (count > 0) {
        // positions: exclusive warp scan of the popcounts, 32 words per pass; each lane
        // writes its word's events in bit (= move) order, then clears the word
        int at = 0;
        for (int w0 = 0; w0 < nw; w0 += 32) {
            const int w = w0 + lane;
            uint32_t x = w < nw ? m[w] : 0u;
            const int c = __popc(x);
            int incl = c;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += y;
            }
            int pos = at + incl - c;
            if (x) m[w] = 0u;
            for (; x; x &= x - 1, ++pos)
                if (pos < lim) dst[pos] = 32 * w + __ffs(x) - 1;
            at += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
    bin_cells_tail<kCellWarps>(s, b, cell, count, inl, lane, warp);
    tl_stop(b.tl, 1, t0);
    if (live) bin_warp_done(b, lane);
}

// Small batches (n <= 64 moves): one warp per cell, no scatter stage.  Lane l
// tests events l and l + 32 (exact fp64 closed-box tests of the new and old
// boxes), two ordered ballots build the list.  Small warps-per-CTA so every cell's
// warp is resident in one wave even for a million components (c4: 8400 cells).
constexpr int kBinSmallWarps = 8;

__global__ void __launch_bounds__(32 * kBinSmallWarps) bin_small_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
    wait_event_boxes(b);
    const unsigned long long t0 = tl_start(b.tl);
    tl_stop(b.tl, 5, tw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * kBinSmallWarps + warp;
    const bool live = cell < s.ncells;
    double cb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) cb[k] = live ? s.cell_aabb[6 * static_cast<size_t>(cell) + k] : 0.0;
    unsigned bal[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = 32 * h + lane;
        bool hit = false;
        if (live && e < b.n) {
            const double* bx = b.evbox + 12 * static_cast<size_t>(e);
            hit = rggd::overlaps(cb, bx) | rggd::overlaps(cb, bx + 6);
        }
        bal[h] = __ballot_sync(0xffffffffu, hit);
    }
    int count = __popc(bal[0]) + __popc(bal[1]);
    int32_t* inl = b.cell_list + static_cast<size_t>(live ? cell : 0) * s.cap;
    int32_t* dst = inl;
    if (count > s.cap) {  // the ordered list goes to the pool
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
            dst = b.pool + pbase;
            if (lane == 0) b.cell_ovf[cell] = pbase;
        }
    }
    const int lim = count;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int pos = (h ? __popc(bal[0]) : 0) + __popc(bal[h] & ((1u << lane) - 1u));
        if (((bal[h] >> lane) & 1u) && pos < lim) dst[pos] = 32 * h + lane;
    }
    bin_cells_tail<kBinSmallWarps>(s, b, cell, count, inl, lane, warp);
    tl_stop(b.tl, 1, t0);
    if (live) bin_warp_done(b, lane);
    if (b.evready) pdl_wait();
}

// ----------------------------------------------------------------- classify

// batch_over for one (component, obstacle) pair: any body intersects (engine_batch.cpp:55-74).
// filter outcome counters (tests, rgg_gpu_filter_stats): [0] SAT filtered, [1] SAT rechecked in
// fp64, [2] seg-sphere filtered, [3] seg-sphere rechecked
__device__ unsigned long long g_filter_stats[4];

// The exact fp64 rechecks run for a handful of pairs per update; kept out of
// line so their register footprint does not cap the classify kernel's occupancy.
__device__ __noinline__ bool sat_exact(const double* a, const double* b) {
    atomicAdd(&g_filter_stats[1], 1ull);
    return rggd::sat_boxes<false>(a, b, nullptr);
}
__device__ __noinline__ bool seg_exact(const double* seg, const double* c, double r_total) {
    atomicAdd(&g_filter_stats[3], 1ull);
    return rggd::seg_sphere_fast(seg, c, r_total);
}

template <bool COUNT>
__device__ __forceinline__ bool over_test(const Store& s, int c, const Event& ev, long long* cost) {
    const double* osat = ev.sat;
    if (!COUNT) {
        // fp32 filter with an exact fp64 recheck of undecided pairs (rgg_device.cuh)
        bool hit = false;
        for (int b = 0; b < s.B && !hit; ++b) {
            const size_t i = static_cast<size_t>(c) * s.B + b;
            const rggd::Box32G a32 = rggd::load_box32g(s.sat32 + i), o32 = rggd::load_box32g(&ev.b32);
            const int f = rggd::sat_filter32g(a32, o32.c, o32);
            hit = f == 2 ? sat_exact(s.sat + i * 22, osat) : f == 1;
        }
        return hit;
    }
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

// The fp32 filter alone: 1 some body surely intersects, 0 every body surely separates,
// 2 undecided (queued: narrow_under_kernel's tail runs the exact fp64 test; keeping that
// path out of narrow_over_kernel<true> leaves it 71 registers instead of 122, 7 CTAs per SM,
// not 4; batches under Batch::recheck_queue's threshold run narrow_over_kernel<false>)
__device__ __forceinline__ int over_filter(const Store& s, int c, const Event& ev) {
    int r = 0;
    const rggd::Box32G o32 = rggd::load_box32g(&ev.b32);
    for (int b = 0; b < s.B; ++b) {
        const rggd::Box32G a32 = rggd::load_box32g(s.sat32 + static_cast<size_t>(c) * s.B + b);
        const int f = rggd::sat_filter32g(a32, o32.c, o32);
        if (f == 1) return 1;
        if (f == 2) r = 2;
    }
    return r;
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

// batch_under for one pair from its item (narrow kernel): the component's real
// segments [lo, hi); word 7 of each segment record carries its row's spline
// radius (rgg_capi.cu upload), so no row lookup is needed.  Lanes g, g+G, ...
template <bool COUNT>
__device__ __forceinline__ bool under_range(const Store& s, int lo, int hi, const Event& ev, int g, int G,
                                            long long* tests) {
    bool hit = false;
    for (int j = lo + g; j < hi; j += G) {
        const double2* p = reinterpret_cast<const double2*>(s.seg + 8 * static_cast<size_t>(j));
        const double2 v0 = p[0], v1 = p[1], v2 = p[2], v3 = p[3];
        const double seg[7] = {v0.x, v0.y, v1.x, v1.y, v2.x, v2.y, v3.x};
        const double r_total = add(ev.r, v3.y);  // o_minus_r + spline_radius[row] (engine_batch.cpp:97)
        if (COUNT) {
            for (int sp = 0; sp < ev.nsph; ++sp) {
                *tests += 1;
                hit |= rggd::seg_sphere_fast(seg, ev.cen + 3 * sp, r_total);
            }
            continue;
        }
        // every sphere through the filter first (independent chains), then the
        // exact fp64 check of the undecided ones only if none hit for sure
        const rggd::Seg32 g32 = rggd::seg32_prep(seg, r_total);
        const int nsph = ev.nsph;
        bool sure = false;
        uint32_t und = 0;
#pragma unroll 4
        for (int sp = 0; sp < nsph; ++sp) {
            const int f = rggd::seg_filter32_pre(seg, g32, ev.cen + 3 * sp);
            sure |= f == 1;
            und |= static_cast<uint32_t>(f == 2) << sp;
        }
        if (sure) return true;
        for (; und; und &= und - 1)
            if (seg_exact(seg, ev.cen + 3 * (__ffs(und) - 1), r_total)) return true;
    }
    return hit;
}

// under_range over the compact fp32 records (rggd::segf_filter): the fp64 record
// is read only when a sphere is undecided.  es: the event's sphere operands
// (Batch::evs).  Verdicts are the reference's.
__device__ __forceinline__ bool under_range32(const Store& s, int lo, int hi, const float4* es, const Event& ev) {
    const float4 hd = es[0];
    const int nsph = __float_as_int(hd.y);
    for (int j = lo; j < hi; ++j) {
        const float4 v0 = s.seg32[2 * static_cast<size_t>(j)], v1 = s.seg32[2 * static_cast<size_t>(j) + 1];
        const rggd::SegF g = rggd::segf_prep(v0, v1, hd.x);
        bool sure = false;
        uint32_t und = 0;
#pragma unroll 4
        for (int sp = 0; sp < nsph; ++sp) {
            const float4 c = es[1 + sp];
            const int f = rggd::segf_filter(g, c.x, c.y, c.z, c.w);
            sure |= f == 1;
            und |= static_cast<uint32_t>(f == 2) << sp;
        }
        if (sure) return true;
        if (und) {
            const double2* p = reinterpret_cast<const double2*>(s.seg + 8 * static_cast<size_t>(j));
            const double2 w0 = p[0], w1 = p[1], w2 = p[2], w3 = p[3];
            const double seg[7] = {w0.x, w0.y, w1.x, w1.y, w2.x, w2.y, w3.x};
            const double r_total = add(ev.r, w3.y);  // o_minus_r + spline_radius[row] (engine_batch.cpp:97)
            for (; und; und &= und - 1)
                if (seg_exact(seg, ev.cen + 3 * (__ffs(und) - 1), r_total)) return true;
        }
    }
    return false;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// Stream a byte range towards the SM (L1) or the L2, one request per 128-byte line.
__device__ __forceinline__ void prefetch_range(const void* a, const void* e, bool l1) {
    const char* p = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(127));
    for (; p < reinterpret_cast<const char*>(e); p += 128) l1 ? prefetch_l1(p) : prefetch_l2(p);
}


// ------------------------------------------------------- mask blocks of touch / narrow / apply
//
// Per cell with L listed events the bin kernel reserves a mask block of
// 3 * ceil(L/32) * cell words: touch[w][t], over[w][t], under[w][t] (bit k of
// word w = the cell's event at list position 32w + k, for component t of the
// cell).  touch fills the touch words and emits one work item per (component,
// event) pair whose boxes overlap; narrow evaluates every item with the whole
// GPU and ORs the verdicts into the result words; apply replays each
// component's events in move order from the three words.

// the moved obstacles' operands, alone (a store without components)
__global__ void commit_kernel(Store s, Batch b) { commit_grid(s, b); }

__device__ __forceinline__ const int32_t* rec_list(int4 r) {
    return reinterpret_cast<const int32_t*>((static_cast<unsigned long long>(static_cast<uint32_t>(r.w)) << 32) |
                                            static_cast<uint32_t>(r.z));
}


// The reference's operation census of the last update's narrow items (rgg_gpu_census),
// GPU-wide, one thread per item.  Over items {component, event, result word, bit}: the
// 15-axis SAT per body.  Under items {segment, the pair's first segment, result word,
// event << 5 | bit}: one real segment of the component against the event's spheres.
// The verdicts themselves come from narrow_over_kernel / narrow_under_kernel below.
__global__ void __launch_bounds__(128) narrow_census_kernel(Store s, Batch b) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int n_over = min(b.ctr[8], b.items_cap), n_under = min(b.ctr[9], b.items_cap);
    long long c_sat = 0, c_tests = 0, c_op = 0, c_up = 0, c_oh = 0, c_uh = 0;
    for (int i = gt; i < n_over; i += nthreads) {
        const int4 it = b.items_over[i];  // component, event, result word, bit
        const bool h = over_test<true>(s, it.x, b.ev[it.y], &c_sat);
        c_op += s.B, c_oh += h;
    }
    for (int i = gt; i < n_under; i += nthreads) {  // per (pair, segment) items: pairs = first segments
        const int4 it = b.items_under[i];
        const bool h = under_range<true>(s, it.x, it.x + 1, b.ev[it.w >> 5], 0, 1, &c_tests);
        c_up += it.x == it.y, c_uh += h;
    }
    long long v[6] = {c_op, c_sat, c_up, c_tests, c_oh, c_uh};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        long long x = v[k];
        for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
        if (lane == 0 && x) atomicAdd(&b.census[k], static_cast<unsigned long long>(x));
    }
}

// The narrow tests split by item kind, so each kernel gets the registers (and hence the
// occupancy) its own test needs: the SAT filter of the over items, the segment-sphere
// filter of the under items.  narrow_over_kernel waits for touch (PDL) and triggers
// right away; narrow_under_kernel's CTAs therefore start only after every over CTA is
// past its wait (touch complete, its items visible), run without a wait of their own,
// and wait for narrow_over_kernel before they exit, so the apply kernel's wait on
// narrow_under_kernel covers both.  The over pairs the fp32 filter leaves undecided are
// queued (Batch::items_recheck) and decided in fp64 by narrow_under_kernel after that wait
// (narrow_recheck), so narrow_over_kernel carries only the filter's registers.
template <bool QUEUE>
__global__ void __launch_bounds__(128) narrow_over_kernel(Store s, Batch b) {
    pdl_wait();
    pdl_trigger();
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const int total = min(b.ctr[8], b.items_cap);
    int i = gt;
    int4 it = i < total ? b.items_over[i] : make_int4(0, 0, 0, 0);
    int4 nx = i + nthreads < total ? b.items_over[i + nthreads] : make_int4(0, 0, 0, 0);
    while (i < total) {
        const int inext = i + nthreads, i2 = inext + nthreads;
        const int4 nn = i2 < total ? b.items_over[i2] : make_int4(0, 0, 0, 0);
        if (inext < total) {
            prefetch_l1(s.sat32 + static_cast<size_t>(nx.x) * s.B);
            prefetch_l1(&b.ev[nx.y].b32);
        }
        if (QUEUE) {
            const int f = over_filter(s, it.x, b.ev[it.y]);
            if (f == 1) atomicOr(&b.mpool[it.z], static_cast<uint32_t>(it.w));
            if (f == 2) {
                const int q = atomicAdd(&b.ctr[12], 1);
                if (q < b.recheck_cap) b.items_recheck[q] = it;
            }
        } else if (over_test<false>(s, it.x, b.ev[it.y], nullptr)) {  // small batches: the fp64 path inline
            atomicOr(&b.mpool[it.z], static_cast<uint32_t>(it.w));
        }
        it = nx;
        nx = nn;
        i = inext;
    }
}

// over_test<false> for one pair by a whole warp: the filter per body, and for an undecided
// body the exact fp64 test with its 15 axes split over lanes (rggd::sat_separated_part:
// the pair is separated iff some lane finds a separating tested axis, so the verdict is
// sat_boxes' whatever the order)
__device__ __forceinline__ bool over_test_warp(const Store& s, int c, const Event& ev, int lane) {
    const rggd::Box32G o32 = rggd::load_box32g(&ev.b32);
    for (int b = 0; b < s.B; ++b) {
        const size_t i = static_cast<size_t>(c) * s.B + b;
        const int f = rggd::sat_filter32g(rggd::load_box32g(s.sat32 + i), o32.c, o32);
        if (f == 1) return true;
        if (f == 2) {
            if (lane == 0) atomicAdd(&g_filter_stats[1], 1ull);
            const bool sep = lane < 15 && rggd::sat_separated_part(s.sat + i * 22, ev.sat, lane, 15);
            if (!__any_sync(0xffffffffu, sep)) return true;
        }
    }
    return false;
}

// The over items narrow_over_kernel's filter left undecided (Batch::items_recheck, count
// ctr[12]), a warp per item, by narrow_under_kernel once narrow_over_kernel is complete;
// past recheck_cap queued items every over item is re-run.
__device__ __forceinline__ void narrow_recheck(const Store& s, const Batch& b) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int n = b.ctr[12];
    const bool all = n > b.recheck_cap;
    const int total = all ? min(b.ctr[8], b.items_cap) : n;
    const int4* items = all ? b.items_over : b.items_recheck;
    for (int i = gw; i < total; i += nwarps) {
        const int4 it = items[i];
        if (over_test_warp(s, it.x, b.ev[it.y], lane) && lane == 0)
            atomicOr(&b.mpool[it.z], static_cast<uint32_t>(it.w));
    }
}

__global__ void __launch_bounds__(128, 9) narrow_under_kernel(Store s, Batch b) {
    pdl_trigger();
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const int total = min(b.ctr[9], b.items_cap);
    int i = gt;
    int4 it = i < total ? b.items_under[i] : make_int4(0, 0, 0, 0);
    int4 nx = i + nthreads < total ? b.items_under[i + nthreads] : make_int4(0, 0, 0, 0);
    while (i < total) {
        const int inext = i + nthreads, i2 = inext + nthreads;
        const int4 nn = i2 < total ? b.items_under[i2] : make_int4(0, 0, 0, 0);
        if (inext < total) {
            prefetch_l1(s.seg32 + 2 * static_cast<size_t>(nx.x));
            prefetch_l1(b.evs + kEvS * static_cast<size_t>(nx.w >> 5));
        }
        if (under_range32(s, it.x, it.x + 1, b.evs + kEvS * static_cast<size_t>(it.w >> 5), b.ev[it.w >> 5]))
            atomicOr(&b.mpool[it.z], 1u << (it.w & 31));  // a pair's segments OR into one bit
        it = nx;
        nx = nn;
        i = inext;
    }
    pdl_wait();  // narrow_over_kernel is complete before this grid is
    narrow_recheck(s, b);
}

// ------------------------------------------------- warp-slice touch / GPU-wide narrow / warp-slice apply
constexpr int kWarpsPerCta = 4;   // warps per CTA of the slice kernels (touch, apply)
constexpr int kStageIds = 1024;  // apply stages the moved obstacle ids of batches up to this size
//
// A warp owns a 32-component slice for the touch masks and for the transitions;
// the narrow tests of all slices are drained by one GPU-wide kernel (one
// (component, event) item per thread), so a slice next to an obstacle does not
// serialise its SAT / segment rounds on one warp.  Masks live in the per-cell
// mask blocks the bin kernel reserves (word (kind*W + w)*cell + t).

template <bool CENSUS>
__global__ void __launch_bounds__(32 * kWarpsPerCta) touch_warp_kernel(Store s, Batch b) {
    const unsigned long long tw = CENSUS ? 0 : tl_start(b.tl);
    // touch on published units (Batch::unit_ready): the event operands once every pose
    // warp released them, then each unit once bin stamped it; otherwise the whole bin kernel
    const bool flow = !CENSUS && b.unit_ready != nullptr;
    if (flow) {
        pdl_trigger();
        if (threadIdx.x == 0) {
            for (unsigned spins = 0;; ++spins) {
                int r;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(b.evready + 1) : "memory");
                if (r >= b.n || handoff_timeout(b, spins)) break;
                __nanosleep(32);
            }
        }
        __syncthreads();
    } else {
        pdl_wait();
        pdl_trigger();
    }
    const unsigned long long t0 = CENSUS ? 0 : tl_start(b.tl);
    if (!CENSUS) tl_stop(b.tl, 6, tw);
    // each warp stages its current chunk of 32 listed events; the batch's operands
    // are prefetched into this SM's L1 first (read per chunk below)
    __shared__ double sbx[kWarpsPerCta * 32][24];
    __shared__ int sev[kWarpsPerCta][32];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = (s.Np + 31) >> 5;
    {
        const char* p = reinterpret_cast<const char*>(b.evt);
        const int lines = (b.n * 24 * 8 + 127) >> 7;
        for (int l = threadIdx.x; l < min(lines, 256); l += blockDim.x) prefetch_l1(p + (static_cast<size_t>(l) << 7));
    }
    unsigned long long c_dirty = 0, c_box = 0, c_sph = 0, c_segs = 0, c_touch = 0, c_segs_all = 0;
    // Work units: (slice, chunk of <= 32 listed events) from the bin kernel's unit
    // list, so a cell with many events spreads over several warps.  The census
    // walks every slice with all its chunks.
    const int spc = s.cell >> 5;  // slices per cell
    const int n_units = CENSUS ? nslices : min(b.ctr[10], b.units_cap) * spc;
    const int gen = flow ? reinterpret_cast<volatile int32_t*>(b.evready)[4] : 0;
    // flow: slice-units are taken one at a time from a counter, and a unit is used once
    // its stamp is this update's generation; the list ends when every bin warp is done
    // and the index is past the final unit count
    auto take = [&]() {
        int v = 0;
        if (lane == 0) v = atomicAdd(b.evready + 3, 1);
        return __shfl_sync(0xffffffffu, v, 0);
    };
    auto available = [&](int u) {
        if (!flow) return u < n_units;
        const int unit = u / spc;
        for (unsigned spins = 0;; ++spins) {
            int st = 0;
            if (lane == 0) {
                int r;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(b.unit_ready + min(unit, b.units_cap - 1)) : "memory");
                if (unit < b.units_cap && r == gen) {
                    st = 1;
                } else {
                    int d;
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(d) : "l"(b.evready + 2) : "memory");
                    if (d >= b.bin_warps) {
                        const int cnt = min(reinterpret_cast<volatile int32_t*>(b.ctr)[10], b.units_cap);
                        if (unit >= cnt) st = 2;  // past the end
                    }
                }
                if (st == 0 && handoff_timeout(b, spins)) st = 2;
            }
            st = __shfl_sync(0xffffffffu, st, 0);
            if (st == 1) return true;
            if (st == 2) return false;
            __nanosleep(64);
        }
    };
    for (int u = flow ? take() : blockIdx.x * kWarpsPerCta + wi; available(u);
         u = flow ? take() : u + gridDim.x * kWarpsPerCta) {
        int q = u, w_first = 0, w_last = 1 << 30;
        int4 rec;
        if (!CENSUS) {
            const int4 un = b.units[u / spc];  // {cell, chunk, count, mask base}
            q = un.x * spc + u % spc;
            w_first = un.y;
            w_last = un.y + 1;
            rec = make_int4(un.z, un.w, 0, 0);
        }
        const int c0 = q << 5;
        if (c0 >= s.Np) continue;
        const int cell = c0 / s.cell;
        if (CENSUS) rec = b.crec[cell];
        const int count = rec.x;
        if (count == 0) continue;  // warp-uniform: clean cell
        const int c = c0 + lane, t = c - cell * s.cell;
        const bool valid = c < s.Np;
        double aabb[6], sbox[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) sbox[j] = s.slice_aabb[6 * static_cast<size_t>(q) + j];
        int seg_lo = 0, seg_hi = 0;
        if (valid) {
            const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
            aabb[0] = a0.x, aabb[1] = a0.y, aabb[2] = a1.x, aabb[3] = a1.y, aabb[4] = a2.x, aabb[5] = a2.y;
            seg_lo = s.row[c * s.B * s.S];
            seg_hi = s.row[(c + 1) * s.B * s.S];
        }
        const int32_t* list = CENSUS ? rec_list(rec)
                                     : (count <= s.cap ? b.cell_list + static_cast<size_t>(cell) * s.cap
                                                       : b.pool + b.cell_ovf[cell]);
        const int W = (count + 31) >> 5;
        bool any_box = false, any_sph = false;
        for (int w = w_first; w < min(W, w_last); ++w) {
            const int base = 32 * w;
            const int m = min(32, count - base);
            const int myev = lane < m ? list[base + lane] : 0;
            sev[wi][lane] = myev;
            if (lane < m) {
                const double2* src = reinterpret_cast<const double2*>(b.evt + 24 * static_cast<size_t>(myev));
#pragma unroll
                for (int j = 0; j < 12; ++j) {
                    const double2 v = src[j];
                    sbx[32 * wi + lane][2 * j] = v.x;
                    sbx[32 * wi + lane][2 * j + 1] = v.y;
                }
            }
            __syncwarp();
            // the chunk's events whose new or old box meets the slice's box: the cell's list
            // is coarser than a slice, and the other events touch none of its components
            bool near = false;
            if (lane < m) {
                const double* bx = sbx[32 * wi + lane];
                near = rggd::overlaps(sbox, bx) | rggd::overlaps(sbox, bx + 6);
            }
            const uint32_t smask = __ballot_sync(0xffffffffu, near);
            uint32_t tm = 0, bm = 0, sm = 0;
            if (valid) {
                for (uint32_t x = smask; x; x &= x - 1) {
                    const int k = __ffs(x) - 1;
                    const double* bx = sbx[32 * wi + k];
                    const bool touch = rggd::overlaps(aabb, bx) | rggd::overlaps(aabb, bx + 6);
                    tm |= static_cast<uint32_t>(touch) << k;
                    bm |= static_cast<uint32_t>(touch & rggd::overlaps(aabb, bx + 12)) << k;
                    sm |= static_cast<uint32_t>(touch & (s.use_under != 0) & rggd::overlaps(aabb, bx + 18)) << k;
                }
            }
            any_box |= bm != 0;
            any_sph |= sm != 0;
            if (CENSUS) {
                c_touch += __popc(tm);
                __syncwarp();
                continue;
            }
            // the narrow kernel (next launch) reads exactly these operands: stage them in L2
            // now, when the roadmap's operands fit the L2 (else the prefetches evict each other)
            if (bm && w == 0 && s.prefetch) {
                const size_t i0 = static_cast<size_t>(c) * s.B;
                prefetch_range(s.sat32 + i0, s.sat32 + i0 + s.B, false);
            }
            if (sm && w == 0 && s.prefetch)
                prefetch_range(s.seg32 + 2 * static_cast<size_t>(seg_lo), s.seg32 + 2 * static_cast<size_t>(seg_hi), false);
            const int wt = rec.y + (0 * W + w) * s.cell + t, wo = rec.y + (1 * W + w) * s.cell + t,
                      wu = rec.y + (2 * W + w) * s.cell + t;
            if (valid) {
                b.mpool[wt] = tm;
                b.mpool[wo] = 0;
                b.mpool[wu] = 0;
            }
            // one warp-aggregated reservation per queue and chunk
            // one packed reservation for both queues (ctr[8] over count, ctr[9] under count);
            // a full queue is reported through ctr[6] = 3 (the apply kernel then applies nothing)
            int at, atu;
            {
                // under work is queued per (pair, segment): the narrow threads then test one
                // segment each, so a pair's segment count no longer diverges a warp
                const unsigned long long mine = static_cast<unsigned long long>(__popc(bm)) |
                                                (static_cast<unsigned long long>(__popc(sm) * (seg_hi - seg_lo)) << 32);
                unsigned long long x = mine;
                for (int off = 1; off < 32; off <<= 1) {
                    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, off);
                    if (lane >= off) x += y;
                }
                const unsigned long long total = __shfl_sync(0xffffffffu, x, 31);
                unsigned long long base = 0;
                if (lane == 31 && total) base = atomicAdd(reinterpret_cast<unsigned long long*>(&b.ctr[8]), total);
                base = __shfl_sync(0xffffffffu, base, 31) + x - mine;
                at = static_cast<int>(base & 0xffffffffu);
                atu = static_cast<int>(base >> 32);
            }
            for (uint32_t x = bm; x; x &= x - 1, ++at) {
                const int k = __ffs(x) - 1;
                if (at < b.items_cap) b.items_over[at] = make_int4(c, sev[wi][k], wo, 1 << k);
                else b.ctr[6] = 3;
            }
            at = atu;
            for (uint32_t x = sm; x; x &= x - 1) {
                const int k = __ffs(x) - 1;
                const int w4 = (sev[wi][k] << 5) | k;
                for (int j = seg_lo; j < seg_hi; ++j, ++at) {  // {segment, the pair's first segment, word, event|bit}
                    if (at < b.items_cap) b.items_under[at] = make_int4(j, seg_lo, wu, w4);
                    else b.ctr[6] = 3;
                }
            }
            __syncwarp();
        }
        if (CENSUS && valid) {
            c_dirty += 1;
            c_box += any_box;
            c_sph += any_sph;
            if (any_sph) c_segs += seg_hi - seg_lo;
            c_segs_all += seg_hi - seg_lo;
        }
    }
    if (!CENSUS) tl_stop(b.tl, 2, t0);
    if (flow) pdl_wait();  // the grid ends after bin's (narrow waits on this grid only)
    if (CENSUS) {
        unsigned long long v[6] = {c_dirty, c_box, c_sph, c_segs, c_touch, c_segs_all};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            unsigned long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&b.census[8 + k], x);
        }
    }
}

// touch, one CTA per work unit (a cell's chunk of <= 32 listed events): warp w takes the
// cell's slice w (kWarpsPerCta == slices per cell at 128-component cells), so the chunk's
// event boxes are staged once per CTA (all 128 threads load them) instead of once per
// slice.  The tests and items are touch_warp_kernel's; that kernel remains for the census
// and for the published-unit handoff (Batch::unit_ready).
__global__ void __launch_bounds__(32 * kWarpsPerCta) touch_cta_kernel(Store s, Batch b) {
    __shared__ double sbx[32][24];
    __shared__ int sev[32];
    const int tid = threadIdx.x, wi = tid >> 5, lane = tid & 31;
    {  // the pose kernel's event boxes are complete once this grid's CTAs run (every kernel
       // since waited on its predecessor): into this SM's L1 before the wait
        const char* p = reinterpret_cast<const char*>(b.evt);
        const int lines = (b.n * 24 * 8 + 127) >> 7;
        for (int l = tid; l < min(lines, 256); l += blockDim.x) prefetch_l1(p + (static_cast<size_t>(l) << 7));
    }
    pdl_wait();
    pdl_trigger();
    const int spc = s.cell >> 5;  // slices per cell (<= kWarpsPerCta)
    const int n_rec = min(b.ctr[10], b.units_cap);
    for (int r = blockIdx.x; r < n_rec; r += gridDim.x) {
        const int4 un = b.units[r];  // {cell, chunk, count, mask base}
        const int cell = un.x, w = un.y, count = un.z;
        const int q = cell * spc + wi, c0 = q << 5;
        const bool has_slice = wi < spc && c0 < s.Np;
        const int c = c0 + lane, t = c - cell * s.cell;
        const bool valid = has_slice && c < s.Np;
        // this warp's slice operands (independent of the staging below)
        double aabb[6], sbox[6];
        int seg_lo = 0, seg_hi = 0;
        if (has_slice) {
#pragma unroll
            for (int j = 0; j < 6; ++j) sbox[j] = s.slice_aabb[6 * static_cast<size_t>(q) + j];
        }
        if (valid) {
            const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
            aabb[0] = a0.x, aabb[1] = a0.y, aabb[2] = a1.x, aabb[3] = a1.y, aabb[4] = a2.x, aabb[5] = a2.y;
            seg_lo = s.row[c * s.B * s.S];
            seg_hi = s.row[(c + 1) * s.B * s.S];
        }
        // stage the chunk's event boxes: 12 double2 per event over the CTA's threads
        const int32_t* list = count <= s.cap ? b.cell_list + static_cast<size_t>(cell) * s.cap : b.pool + b.cell_ovf[cell];
        const int W = (count + 31) >> 5, base = 32 * w, m = min(32, count - base);
        for (int x = tid; x < m * 12; x += blockDim.x) {
            const int e = x / 12, j = x - 12 * e;
            const int ev = list[base + e];
            const double2 v = reinterpret_cast<const double2*>(b.evt + 24 * static_cast<size_t>(ev))[j];
            sbx[e][2 * j] = v.x;
            sbx[e][2 * j + 1] = v.y;
            if (j == 0) sev[e] = ev;
        }
        __syncthreads();
        uint32_t tm = 0, bm = 0, sm = 0;
        if (has_slice) {
            // the chunk's events whose new or old box meets the slice's box
            bool near = false;
            if (lane < m) near = rggd::overlaps(sbox, sbx[lane]) | rggd::overlaps(sbox, sbx[lane] + 6);
            const uint32_t smask = __ballot_sync(0xffffffffu, near);
            if (valid) {
                for (uint32_t x = smask; x; x &= x - 1) {
                    const int kk = __ffs(x) - 1;
                    const double* bx = sbx[kk];
                    const bool touch = rggd::overlaps(aabb, bx) | rggd::overlaps(aabb, bx + 6);
                    tm |= static_cast<uint32_t>(touch) << kk;
                    bm |= static_cast<uint32_t>(touch & rggd::overlaps(aabb, bx + 12)) << kk;
                    sm |= static_cast<uint32_t>(touch & (s.use_under != 0) & rggd::overlaps(aabb, bx + 18)) << kk;
                }
            }
            // the narrow kernels (next launches) read exactly these operands: stage them in L2
            if (bm && w == 0 && s.prefetch) {
                const size_t i0 = static_cast<size_t>(c) * s.B;
                prefetch_range(s.sat32 + i0, s.sat32 + i0 + s.B, false);
            }
            if (sm && w == 0 && s.prefetch)
                prefetch_range(s.seg32 + 2 * static_cast<size_t>(seg_lo), s.seg32 + 2 * static_cast<size_t>(seg_hi), false);
        }
        const int wt = un.w + (0 * W + w) * s.cell + t, wo = un.w + (1 * W + w) * s.cell + t,
                  wu = un.w + (2 * W + w) * s.cell + t;
        if (valid) {
            b.mpool[wt] = tm;
            b.mpool[wo] = 0;
            b.mpool[wu] = 0;
        }
        // one packed reservation per warp for both queues (ctr[8] over items, ctr[9] under
        // items per (pair, segment)); a full queue is reported through ctr[6] = 3.  (One per
        // CTA, by thread 0 between two barriers, was slower.)
        const unsigned long long mine = static_cast<unsigned long long>(__popc(bm)) |
                                        (static_cast<unsigned long long>(__popc(sm) * (seg_hi - seg_lo)) << 32);
        unsigned long long x = mine;
        for (int off = 1; off < 32; off <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, off);
            if (lane >= off) x += y;
        }
        const unsigned long long wtot = __shfl_sync(0xffffffffu, x, 31);
        unsigned long long wbase = 0;
        if (lane == 31 && wtot) wbase = atomicAdd(reinterpret_cast<unsigned long long*>(&b.ctr[8]), wtot);
        wbase = __shfl_sync(0xffffffffu, wbase, 31);
        const unsigned long long at64 = wbase + x - mine;
        int at = static_cast<int>(at64 & 0xffffffffu);
        for (uint32_t y = bm; y; y &= y - 1, ++at) {
            const int kk = __ffs(y) - 1;
            if (at < b.items_cap) b.items_over[at] = make_int4(c, sev[kk], wo, 1 << kk);
            else b.ctr[6] = 3;
        }
        at = static_cast<int>(at64 >> 32);
        for (uint32_t y = sm; y; y &= y - 1) {
            const int kk = __ffs(y) - 1;
            const int w4 = (sev[kk] << 5) | kk;
            for (int j = seg_lo; j < seg_hi; ++j, ++at) {  // {segment, the pair's first segment, word, event|bit}
                if (at < b.items_cap) b.items_under[at] = make_int4(j, seg_lo, wu, w4);
                else b.ctr[6] = 3;
            }
        }
        __syncthreads();  // sbx / sev are restaged by the next unit
    }
}

// Per-move transitions (engine_batch.cpp:114-188) of every component of a dirty
// slice, in list (= move) order, from the touch / over / under words.  WIDE (M > 64 obstacles, ceil(M/64) bit words per
// component): the old over / under bits of every event touching a lane are loaded
// up front, four at a time, before the walk, and changed bits are written back with
// fire-and-forget atomics, so the walk has no memory round trip per event.  A batch
// that moves an obstacle twice keeps the sequential read-modify-write (the second
// move's old bits are the first one's new bits).
// 9 CTAs per SM (<= 56 registers, a few spilled): more resident warps hide the walk's
// bit-word round trips better than the registers save (c5: 0.263 -> 0.253 ms)
template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(32 * kWarpsPerCta, 9) apply_warp_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    constexpr bool HITS = (FLAGS & kHits) != 0;
    __shared__ int2 som[kWarpsPerCta][32];
    __shared__ int s_ids[kStageIds];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = (s.Np + 31) >> 5;
    const bool staged = b.n <= kStageIds;
    // the pose kernel's outputs (ids, last) are complete once this grid's CTAs run: every
    // kernel since has waited on its predecessor, so stage them before the wait, while
    // the narrow kernels drain
    int rep = 0;  // some obstacle moves twice in this batch (b.last from the pose kernel)
    for (int t = threadIdx.x; t < b.n; t += blockDim.x) {
        if (staged) s_ids[t] = b.ids[t];
        rep |= b.last[t] == 0;
    }
    const bool repeats = __syncthreads_or(rep) != 0;
    pdl_wait();
    pdl_trigger();
    const unsigned long long t0 = tl_start(b.tl);
    tl_stop(b.tl, 8, tw);
    if (b.evready && blockIdx.x == 0 && threadIdx.x < 4) b.evready[threadIdx.x] = 0;  // for the next update
    int dgray = 0;
    // any failed stage (status ctr[6]: 1 overflow pool, 2 mask pool, 3 full narrow-item
    // queue, 4 handoff timeout) left some verdicts uncomputed: apply nothing, so the
    // engine stays at its pre-update state (the host grows the queue and replays on 3,
    // and fails the update otherwise)
    const int status = b.ctr[6];
    // Work list: when fewer than half the cells are dirty, the dirty slices only, from
    // touch's work units (a cell's first chunk stands for the cell: {cell, 0, count,
    // mask base}); otherwise every slice, with its state loads issued before the cell
    // record's (one round trip less on the chain).
    const bool dirty_only = 2 * b.ctr[0] < s.ncells;
    const int spc = s.cell >> 5;
    const int n_work = status != 0 ? 0 : (dirty_only ? min(b.ctr[10], b.units_cap) * spc : nslices);
    // static striding over the work list (a same-address atomic per slice to take work
    // dynamically serialised at the L2: slower at c5)
    for (int wq = blockIdx.x * kWarpsPerCta + wi; wq < n_work; wq += gridDim.x * kWarpsPerCta) {
        int q = wq;
        int4 un = make_int4(0, 0, 0, 0);
        bool skip = false;
        if (dirty_only) {
            un = b.units[wq / spc];
            skip = un.y != 0;  // warp-uniform: a later chunk of a listed cell
            q = un.x * spc + wq % spc;
        }
        const int c0 = q << 5;
        skip |= c0 >= s.Np;
        const int cell = c0 / s.cell;
        const int c = c0 + lane, t = c - cell * s.cell;
        const bool valid = !skip && c < s.Np;
        // the slice's state (coalesced, cell order) is loaded together with the
        // cell record, so one memory round trip serves both
        int label = 0, oc = 0, bc = 0, id = -1;
        unsigned long long OW = 0, UW = 0;
        uint32_t cw = 0;
        if (valid) {
            id = s.orig[c];
            cw = s.cnt[c];
            if (!WIDE) {
                OW = s.over[c];
                UW = s.under[c];
            }
            label = s.state_c[c];
        }
        int4 rec = make_int4(0, 0, 0, 0);
        if (!skip) {
            if (dirty_only) {
                const int32_t* lst =
                    un.z <= s.cap ? b.cell_list + static_cast<size_t>(cell) * s.cap : b.pool + b.cell_ovf[cell];
                const unsigned long long la = reinterpret_cast<unsigned long long>(lst);
                rec = make_int4(un.z, un.w, static_cast<int>(la & 0xffffffffu), static_cast<int>(la >> 32));
            } else {
                rec = b.crec[cell];
            }
        }
        const int count = rec.x;
        oc = cw & 0xffff;
        bc = cw >> 16;
        const int label0 = label;
        const uint32_t cnt0 = cw;
        const unsigned long long OW0 = OW, UW0 = UW;
        bool hit_last = false;
        const int32_t* list = rec_list(rec);
        const int W = (count + 31) >> 5;
        for (int base = 0, w = 0; base < count; base += 32, ++w) {
            const int m = min(32, count - base);
            if (lane < m) {  // list entries are move indices; the event of move e moves obstacle ids[e]
                const int e = list[base + lane];
                som[wi][lane] = make_int2(staged ? s_ids[e] : b.ids[e], e);
            }
            uint32_t tm = 0, ro = 0, ru = 0;
            if (valid) {
                tm = b.mpool[rec.y + (0 * W + w) * s.cell + t];
                ro = b.mpool[rec.y + (1 * W + w) * s.cell + t];
                ru = b.mpool[rec.y + (2 * W + w) * s.cell + t];
            }
            __syncwarp();
            // WIDE: the old bits of this lane's touching events, all loads in flight together
            uint32_t oldO = 0, oldU = 0;
            if (WIDE && !repeats) {
                for (uint32_t x = tm; x;) {
                    int k[4];
                    unsigned long long wo[4], wu[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        k[j] = x ? __ffs(x) - 1 : -1;
                        x &= x - 1;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k[j] >= 0) {
                            const size_t idx = static_cast<size_t>(som[wi][k[j]].x >> 6) * s.Np + c;
                            wo[j] = s.over[idx];
                            wu[j] = s.under[idx];
                        }
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (k[j] >= 0) {
                            const int ob = som[wi][k[j]].x & 63;
                            oldO |= static_cast<uint32_t>((wo[j] >> ob) & 1ull) << k[j];
                            oldU |= static_cast<uint32_t>((wu[j] >> ob) & 1ull) << k[j];
                        }
                }
            }
            // a touching event changes nothing for a component that neither held its bits
            // nor is hit now: walk only the events some lane of the slice is active for, in
            // list (= move) order (with an obstacle moved twice in the batch, its second
            // move's old bits are the first one's new bits: then every touching event)
            uint32_t act = tm;
            if (!repeats) {
                if (!WIDE)
                    for (uint32_t x = tm; x; x &= x - 1) {
                        const int kk = __ffs(x) - 1;
                        const int ob = som[wi][kk].x & 63;
                        oldO |= static_cast<uint32_t>((OW >> ob) & 1ull) << kk;
                        oldU |= static_cast<uint32_t>((UW >> ob) & 1ull) << kk;
                    }
                act = tm & (ro | ru | oldO | oldU);
            }
            for (uint32_t em = __reduce_or_sync(0xffffffffu, act); em; em &= em - 1) {
                const int k = __ffs(em) - 1;
                const int before = label;
                const int2 om = som[wi][k];
                if ((act >> k) & 1u) {
                    const int o = om.x;
                    const size_t widx = static_cast<size_t>(o >> 6) * s.Np + c;
                    const unsigned long long bit = 1ull << (o & 63);
                    bool old_over, old_under;
                    unsigned long long ow = 0, uw = 0;
                    if (!WIDE) {
                        old_over = (OW & bit) != 0;
                        old_under = (UW & bit) != 0;
                    } else if (!repeats) {
                        old_over = (oldO >> k) & 1u;
                        old_under = (oldU >> k) & 1u;
                    } else {
                        ow = s.over[widx];
                        uw = s.under[widx];
                        old_over = (ow & bit) != 0;
                        old_under = (uw & bit) != 0;
                    }
                    const bool n_over = (ro >> k) & 1u, n_under = (ru >> k) & 1u;
                    if (old_over) {  // revalidate_old_intersections (engine_batch.cpp:114-143)
                        oc -= 1;
                        const int rest = bc - (old_under ? 1 : 0);
                        label = oc == 0 ? 0 : ((s.use_under && rest > 0) ? 1 : 2);
                    }
                    if (n_over) {  // over phase (engine_batch.cpp:163-177)
                        if (label == 0) label = 2;
                        oc += 1;
                    }
                    if (n_under) label = 1;  // under phase (engine_batch.cpp:181-188)
                    bc += (n_over && n_under ? 1 : 0) - (old_over && old_under ? 1 : 0);
                    if (!WIDE) {
                        OW = n_over ? (OW | bit) : (OW & ~bit);
                        UW = n_under ? (UW | bit) : (UW & ~bit);
                    } else if (!repeats) {  // each lane owns its component's words: only this bit changes
                        if (n_over != old_over)
                            n_over ? atomicOr(&s.over[widx], bit) : atomicAnd(&s.over[widx], ~bit);
                        if (n_under != old_under)
                            n_under ? atomicOr(&s.under[widx], bit) : atomicAnd(&s.under[widx], ~bit);
                    } else {
                        const unsigned long long nw = n_over ? (ow | bit) : (ow & ~bit);
                        const unsigned long long nuw = n_under ? (uw | bit) : (uw & ~bit);
                        if (nw != ow) s.over[widx] = nw;
                        if (nuw != uw) s.under[widx] = nuw;
                    }
                    if (HITS && om.y == b.n - 1) hit_last = n_over;
                }
                if (PER_MOVE && __any_sync(0xffffffffu, label != before)) {
                    const bool ch = label != before;
                    const unsigned gg = __ballot_sync(0xffffffffu, ch && label == 0);
                    const unsigned r = __ballot_sync(0xffffffffu, ch && label == 1);
                    const unsigned y = __ballot_sync(0xffffffffu, ch && label == 2);
                    const unsigned f = __ballot_sync(0xffffffffu, ch && before == 2);
                    if (lane == 0 && (gg | r | y | f)) {
                        int* mv = b.mv + 4 * om.y;
                        if (gg) atomicAdd(mv + 0, __popc(gg));
                        if (r) atomicAdd(mv + 1, __popc(r));
                        if (y) atomicAdd(mv + 2, __popc(y));
                        if (f) atomicAdd(mv + 3, __popc(f));
                    }
                }
            }
            __syncwarp();
        }
        if (valid && count > 0) {
            if (label != label0) {
                s.state[id] = static_cast<uint8_t>(label);
                s.state_c[c] = static_cast<uint8_t>(label);
                dgray += (label == 2) - (label0 == 2);
            }
            const uint32_t cwn = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
            if (cwn != cnt0) s.cnt[c] = cwn;
            if (!WIDE) {
                if (OW != OW0) s.over[c] = OW;
                if (UW != UW0) s.under[c] = UW;
            }
        }
        if (HITS && count > 0) {
            const bool h = valid && hit_last && label == 2;
            const unsigned bal = __ballot_sync(0xffffffffu, h);
            int pos = 0;
            if (lane == 0 && bal) pos = atomicAdd(&b.ctr[5], __popc(bal));
            pos = __shfl_sync(0xffffffffu, pos, 0);
            if (h) {
                const int at = pos + __popc(bal & ((1u << lane) - 1u));
                b.hits[at] = id;
                b.hits_prev[at] = static_cast<uint8_t>(label0);
            }
        }
    }
    for (int off = 16; off; off >>= 1) dgray += __shfl_down_sync(0xffffffffu, dgray, off);
    if (lane == 0 && dgray) atomicAdd(b.unknown, dgray);
    if (status == 0) commit_grid(s, b);
    tl_stop(b.tl, 4, t0);
}

// Single-move updates (n == 1: update_obstacle and every eager move): one kernel after
// the pose kernel, no binning, cell lists, work units or item queues.  CTA b tests the
// cells b, b + G, b + 2G, ... (one per thread; a move's dirty cells are neighbours in
// Morton order, so the stride spreads them over the CTAs) against the move's new and old
// union boxes, then runs every hit cell with one thread per component: touch, both
// narrow tests and the reference's transition for the one event (engine_batch.cpp:114-188).
// The per-move counters gather in shared memory; the gray over-hits are listed for the
// eager resolve.
template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(kMaxCell) single_cells_kernel(Store s, Batch b) {
    constexpr bool HITS = (FLAGS & kHits) != 0;
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    const int tid = threadIdx.x, lane = tid & 31, T = blockDim.x;
    // the first round's cell boxes are static: loaded while the pose kernel runs
    double q0[6];
    {
        const long long k = blockIdx.x + static_cast<long long>(gridDim.x) * tid;
#pragma unroll
        for (int j = 0; j < 6; ++j) q0[j] = k < s.ncells ? s.cell_aabb[6 * k + j] : 0.0;
    }
    pdl_wait();
    pdl_trigger();
    __shared__ double sbx[24];  // the event's new union, old union, box, sphere box
    __shared__ int s_mv[4], s_cells[kMaxCell], s_n;
    if (tid < 24) sbx[tid] = b.evt[tid];
    if (tid < 4) s_mv[tid] = 0;
    if (tid == 0) s_n = 0;
    if (b.evready && blockIdx.x == 0 && tid < 4) b.evready[tid] = 0;  // for the next update
    commit_grid(s, b);  // s.cur / s.cur_union: read by the next update's pose kernel only
    __syncthreads();
    const Event& ev = b.ev[0];
    const int o = ev.o;
    const unsigned long long bit = 1ull << (o & 63);
    int dgray = 0;
    for (int r0 = 0; blockIdx.x + static_cast<long long>(gridDim.x) * r0 < s.ncells; r0 += T) {
        const long long k = blockIdx.x + static_cast<long long>(gridDim.x) * (r0 + tid);
        if (k < s.ncells) {
            double q[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) q[j] = r0 == 0 ? q0[j] : s.cell_aabb[6 * k + j];
            if (rggd::overlaps(q, sbx) | rggd::overlaps(q, sbx + 6)) s_cells[atomicAdd(&s_n, 1)] = static_cast<int>(k);
        }
        __syncthreads();
        const int nh = s_n;
        for (int h = 0; h < nh; ++h) {
            const int c = s_cells[h] * s.cell + tid;
            if (c >= s.Np) continue;
            const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
            const double aabb[6] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y};
            const bool touch = rggd::overlaps(aabb, sbx) | rggd::overlaps(aabb, sbx + 6);
            if (!touch) continue;
            const bool box = rggd::overlaps(aabb, sbx + 12);
            const bool sph = s.use_under && rggd::overlaps(aabb, sbx + 18);
            const size_t widx = WIDE ? static_cast<size_t>(o >> 6) * s.Np + c : static_cast<size_t>(c);
            const int id = s.orig[c];
            const uint32_t cw = s.cnt[c];
            const int label0 = s.state_c[c];
            const unsigned long long ow = s.over[widx], uw = s.under[widx];
            const bool n_over = box && over_test<false>(s, c, ev, nullptr);
            bool n_under = false;
            if (sph) {
                const int rows = s.B * s.S;
                n_under = under_range32(s, s.row[c * rows], s.row[(c + 1) * rows], b.evs, ev);
            }
            int oc = cw & 0xffff, bc = cw >> 16, label = label0;
            const bool old_over = (ow & bit) != 0, old_under = (uw & bit) != 0;
            if (old_over) {  // revalidate_old_intersections (engine_batch.cpp:114-143)
                oc -= 1;
                const int rest = bc - (old_under ? 1 : 0);
                label = oc == 0 ? 0 : ((s.use_under && rest > 0) ? 1 : 2);
            }
            if (n_over) {  // over phase (engine_batch.cpp:163-177)
                if (label == 0) label = 2;
                oc += 1;
            }
            if (n_under) label = 1;  // under phase (engine_batch.cpp:181-188)
            bc += (n_over && n_under ? 1 : 0) - (old_over && old_under ? 1 : 0);
            const unsigned long long nw = n_over ? (ow | bit) : (ow & ~bit);
            const unsigned long long nuw = n_under ? (uw | bit) : (uw & ~bit);
            if (nw != ow) s.over[widx] = nw;
            if (nuw != uw) s.under[widx] = nuw;
            const uint32_t cwn = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
            if (cwn != cw) s.cnt[c] = cwn;
            if (label != label0) {  // finish_counts (engine_batch.cpp:41-53)
                s.state[id] = static_cast<uint8_t>(label);
                s.state_c[c] = static_cast<uint8_t>(label);
                dgray += (label == 2) - (label0 == 2);
                if (PER_MOVE) {
                    atomicAdd(&s_mv[label], 1);
                    if (label0 == 2) atomicAdd(&s_mv[3], 1);
                }
            }
            if (HITS && n_over && label == 2) {
                const int at = atomicAdd(&b.ctr[5], 1);
                b.hits[at] = id;
                b.hits_prev[at] = static_cast<uint8_t>(label0);
            }
        }
        __syncthreads();
        if (tid == 0) s_n = 0;
        __syncthreads();
    }
    for (int off = 16; off; off >>= 1) dgray += __shfl_down_sync(0xffffffffu, dgray, off);
    if (lane == 0 && dgray) atomicAdd(b.unknown, dgray);
    __syncthreads();
    if (PER_MOVE && tid < 4 && s_mv[tid]) atomicAdd(&b.mv[tid], s_mv[tid]);
}

// Synchronous host updates: the per-move counters and the status block straight
// into mapped pinned host memory (one small PDL-launched kernel after apply,
// instead of two device-to-host copies).
__global__ void host_out_kernel(Batch b) {
    pdl_wait();
    for (int t = threadIdx.x; t < 4 * b.n; t += blockDim.x) b.out_mv[t] = b.mv[t];
    for (int t = threadIdx.x; t < 24; t += blockDim.x) b.out_ctr[t] = b.ctr[t];
    // out_ctr[31]: "results stored", released to the host (it polls instead of a stream sync)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        reinterpret_cast<volatile int32_t*>(b.out_ctr)[31] = 1;
    }
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
    pdl_wait();
    pdl_trigger();
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

// host_out (synchronous host updates with the gray list): the same ids, also written into
// mapped pinned host memory, through shared memory so each tile's contiguous output range
// goes over PCIe in 16-byte stores (the host reads the list when the update returns)
__global__ void __launch_bounds__(kCompactThreads) gray_write_kernel(const uint8_t* st, int N, const int32_t* tile_cnt,
                                                                     int ntiles, int32_t* out, int32_t* gray_n,
                                                                     int32_t* host_out) {
    pdl_wait();
    pdl_trigger();
    __shared__ int ws[kCompactThreads / 32];
    __shared__ int s_base;
    __shared__ __align__(16) int32_t s_ids[kTile + 4];
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
    if (!host_out) {
        if (n) {
            const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
            for (int i = 0; i < 16; ++i)
                if (b[i] == 2) out[pos++] = base + i;
        }
        return;
    }
    // the tile's ids in shared memory at their offset from the 16-byte-aligned start of
    // its output range, then copied out as int4 (host and device)
    const int lo = s_base & ~3, head = s_base - lo;
    const int total = ws[kCompactThreads / 32 - 1];
    if (n) {
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
        int q = pos - lo;
        for (int i = 0; i < 16; ++i)
            if (b[i] == 2) s_ids[q++] = base + i;
    }
    __syncthreads();
    const int end = head + total;  // entries [head, end) of s_ids are this tile's
    for (int j = 4 * threadIdx.x; j < end; j += 4 * kCompactThreads) {
        if (j >= head && j + 4 <= end) {
            const int4 q4 = *reinterpret_cast<const int4*>(&s_ids[j]);
            *reinterpret_cast<int4*>(out + lo + j) = q4;
            *reinterpret_cast<int4*>(host_out + lo + j) = q4;
        } else {  // the partial words at either end of the range (a neighbour tile owns the rest)
            for (int u = j; u < j + 4 && u < end; ++u)
                if (u >= head) out[lo + u] = s_ids[u], host_out[lo + u] = s_ids[u];
        }
    }
    // the host reads the list once host_out_kernel raises its flag: release this CTA's
    // host stores at system scope first
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
}

__global__ void write_states_kernel(Store s, const int32_t* ids, const uint8_t* st, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    s.state[ids[i]] = st[i];
    const int c = s.rank[ids[i]];
    if (c >= 0) s.state_c[c] = st[i];
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
        h = over_test<false>(s, c, ev, nullptr);
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

// FP32 FMA issue-rate probe: 16 independent FFMA chains per thread.
__global__ void fp32_peak_kernel(float* sink, int iters) {
    float x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = 1.0f + 1e-6f * (threadIdx.x + k);
    const float a = 0.9999999f, c = 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, c);
    }
    float t = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) t += x[k];
    if (t == 12345.0f) sink[0] = t;
}

}  // namespace

// ------------------------------------------------------------------ launchers

// Launch with programmatic stream serialization (PDL): the kernel's CTAs may be
// scheduled while the previous kernel on the stream drains; they wait in
// pdl_wait() for its results.  Captured into CUDA graphs as programmatic edges.
// One shared-memory carveout for every kernel of the update: an SM whose
// L1/shared split differs from the next kernel's must drain before that
// kernel's CTAs can land on it (RGG_CARVEOUT = percent, <0 leaves the driver's
// per-kernel choice).
static void carveout(const void* fn) {
    static const int pct = [] {
        const char* e = std::getenv("RGG_CARVEOUT");
        return e ? std::atoi(e) : -1;
    }();
    if (pct < 0) return;
    static const void* done[64];
    static int ndone = 0;
    for (int i = 0; i < ndone; ++i)
        if (done[i] == fn) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    if (ndone < 64) done[ndone++] = fn;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
    static const bool off = std::getenv("RGG_NO_PDL") != nullptr;
    carveout(reinterpret_cast<const void*>(k));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

cudaError_t launch_pose(const Store& s, const Batch& b, cudaStream_t st) {
    const int warps = 4;  // moves per CTA
    carveout(reinterpret_cast<const void*>(pose_kernel));
    pose_kernel<<<(b.n + warps - 1) / warps, 32 * warps, 0, st>>>(s, b);
    return cudaGetLastError();
}

cudaError_t launch_init_obstacles(const Store& s, Event*, cudaStream_t st) {
    if (s.M == 0) return cudaSuccess;
    init_obstacles_kernel<<<(s.M + 127) / 128, 128, 0, st>>>(s);
    return cudaGetLastError();
}

cudaError_t launch_bin(const Store& s, const Batch& b, cudaStream_t st) {
    if (s.ncells == 0) return cudaSuccess;  // no components: nothing to bin
    static const bool no_small = std::getenv("RGG_NO_SMALL_BIN") != nullptr;
    if (b.n <= kBinSmallMax && !no_small)
        return launch_pdl(bin_small_kernel, dim3((s.ncells + kBinSmallWarps - 1) / kBinSmallWarps),
                          dim3(32 * kBinSmallWarps), st, s, b);
    static const int self_box = [] {  // tests: RGG_SELF_BOX_MAX=0 takes the waiting variant at every size
        const char* v = std::getenv("RGG_SELF_BOX_MAX");
        return v ? std::atoi(v) : kScatterSelfBox;
    }();
    cudaError_t e = b.n < self_box  // a CTA per event
                        ? launch_pdl(bin_scatter_kernel<true>, dim3(b.n), dim3(kScatterThreads), st, s, b)
                        : launch_pdl(bin_scatter_kernel<false>, dim3(b.n), dim3(kScatterThreads), st, s, b);
    if (e != cudaSuccess) return e;
    return launch_pdl(bin_cells_kernel, dim3((s.ncells + kCellWarps - 1) / kCellWarps), dim3(32 * kCellWarps), st, s, b);
}


cudaError_t launch_host_out(const Batch& b, cudaStream_t st) {
    return launch_pdl(host_out_kernel, dim3(1), dim3(256), st, b);
}

// Eager batches run one single-move graph per move.  Between two graphs this
// kernel saves move i-1's report terms (apply counters, resolved hits, resolve
// deltas) to its slot and stages move i into the graph's move slot 0.
__global__ void eager_step_kernel(Batch b, int32_t* ids0, double* rt0, const int32_t* st_ids, const double* st_rt,
                                  int32_t* rep, int i, int k) {
    const int t = threadIdx.x;
    if (i > 0 && t < 8) rep[8 * (i - 1) + t] = t < 4 ? b.mv[t] : (t == 4 ? b.ctr[5] : b.ctr[20 + t - 5]);
    if (i > 0 && t == 0 && b.ctr[6]) b.ctr[18] |= b.ctr[6];  // sticky status of the batch (pose resets ctr[6])
    if (i < k) {
        if (t == 0) ids0[0] = st_ids[i];
        if (t < 12) rt0[t] = st_rt[12 * static_cast<size_t>(i) + t];
    }
}

cudaError_t launch_eager_step(const Batch& b, int32_t* ids0, double* rt0, const int32_t* st_ids, const double* st_rt,
                              int32_t* rep, int i, int k, cudaStream_t st) {
    eager_step_kernel<<<1, 32, 0, st>>>(b, ids0, rt0, st_ids, st_rt, rep, i, k);
    return cudaGetLastError();
}

template <int F, bool W>
static cudaError_t apply6_t(const Store& s, const Batch& b, int grid, cudaStream_t st) {
    return launch_pdl(apply_warp_kernel<F, W>, dim3(grid), dim3(32 * kWarpsPerCta), st, s, b);
}

// persistent slice kernels: one wave (resident CTAs x SMs), fewer CTAs when the
// store has fewer slices
static int grid_slices(const Store& s, const void* fn) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    static const void* fns[16];
    static int occ[16], nfn = 0;
    int per_sm = 0;
    for (int i = 0; i < nfn; ++i)
        if (fns[i] == fn) per_sm = occ[i];
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kWarpsPerCta, 0);
        per_sm = per_sm < 1 ? 1 : per_sm;
        if (nfn < 16) fns[nfn] = fn, occ[nfn++] = per_sm;
    }
    const int need = ((s.Np + 31) / 32 + kWarpsPerCta - 1) / kWarpsPerCta;
    return need < per_sm * sms ? (need < 1 ? 1 : need) : per_sm * sms;
}

template <int F, bool W>
static cudaError_t apply_t(const Store& s, const Batch& b, cudaStream_t st) {
    return launch_pdl(apply_warp_kernel<F, W>, dim3(grid_slices(s, reinterpret_cast<const void*>(apply_warp_kernel<F, W>))),
                      dim3(32 * kWarpsPerCta), st, s, b);
}

template <int F, bool W>
static cudaError_t single_t(const Store& s, const Batch& b, cudaStream_t st) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // one round of cell tests per CTA when the cells allow, at least 2 CTAs per SM otherwise
    const int grid = std::max(std::min(s.ncells, 2 * sms), (s.ncells + s.cell - 1) / s.cell);
    return launch_pdl(single_cells_kernel<F, W>, dim3(std::max(1, grid)), dim3(s.cell), st, s, b);
}

cudaError_t launch_single(const Store& s, const Batch& b, int flags, cudaStream_t st) {
    if (s.ncells == 0) {
        commit_kernel<<<1, 128, 0, st>>>(s, b);
        return cudaGetLastError();
    }
    const bool wide = s.W > 1;
    constexpr int H = kHits, P = kPerMove;
    switch (flags & (kHits | kPerMove)) {
        case H | P: return wide ? single_t<H | P, true>(s, b, st) : single_t<H | P, false>(s, b, st);
        case H: return wide ? single_t<H, true>(s, b, st) : single_t<H, false>(s, b, st);
        case P: return wide ? single_t<P, true>(s, b, st) : single_t<P, false>(s, b, st);
        default: return wide ? single_t<0, true>(s, b, st) : single_t<0, false>(s, b, st);
    }
}

cudaError_t launch_classify(const Store& s, const Batch& b, int flags, int grid, cudaStream_t st) {
    if (s.ncells == 0) {  // no components: only the obstacles' operands move on
        if (b.n == 0 || (flags & kCensus)) return cudaSuccess;
        commit_kernel<<<(b.n + 7) / 8, 128, 0, st>>>(s, b);
        return cudaGetLastError();
    }
    if (flags & kCensus) {
        touch_warp_kernel<true><<<grid_slices(s, reinterpret_cast<const void*>(touch_warp_kernel<true>)),
                                  32 * kWarpsPerCta, 0, st>>>(s, b);
        narrow_census_kernel<<<grid, 128, 0, st>>>(s, b);
        return cudaGetLastError();
    }
    // touch: one CTA per work unit when a cell's slices fill the CTA's warps (128-component
    // cells), else (and for the published-unit handoff) one warp per (slice, unit)
    static const bool warp_touch = std::getenv("RGG_WARP_TOUCH") != nullptr;
    const bool cta = !warp_touch && !b.unit_ready && (s.cell >> 5) == kWarpsPerCta;
    cudaError_t e = cta ? launch_pdl(touch_cta_kernel, dim3(grid_slices(s, reinterpret_cast<const void*>(touch_cta_kernel))),
                                     dim3(32 * kWarpsPerCta), st, s, b)
                        : launch_pdl(touch_warp_kernel<false>,
                                     dim3(grid_slices(s, reinterpret_cast<const void*>(touch_warp_kernel<false>))),
                                     dim3(32 * kWarpsPerCta), st, s, b);
    {
        static int g_over = 0, g_over_inline = 0, g_under = 0;
        if (!g_over) {
            int sms = 148, dev = 0, n = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, narrow_over_kernel<true>, 128, 0);
            g_over = sms * std::max(1, n);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, narrow_over_kernel<false>, 128, 0);
            g_over_inline = sms * std::max(1, n);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, narrow_under_kernel, 128, 0);
            g_under = sms * std::max(1, n);
        }
        if (e == cudaSuccess)
            e = b.recheck_queue ? launch_pdl(narrow_over_kernel<true>, dim3(g_over), dim3(128), st, s, b)
                                : launch_pdl(narrow_over_kernel<false>, dim3(g_over_inline), dim3(128), st, s, b);
        if (e == cudaSuccess) e = launch_pdl(narrow_under_kernel, dim3(g_under), dim3(128), st, s, b);
    }
    if (e != cudaSuccess) return e;
    const bool wide = s.W > 1;
    switch (flags & (kPerMove | kHits)) {
        case 0:
            return wide ? apply_t<0, true>(s, b, st) : apply_t<0, false>(s, b, st);
        case kPerMove:
            return wide ? apply_t<kPerMove, true>(s, b, st) : apply_t<kPerMove, false>(s, b, st);
        case kHits:
            return wide ? apply_t<kHits, true>(s, b, st) : apply_t<kHits, false>(s, b, st);
        default:
            return wide ? apply_t<kPerMove | kHits, true>(s, b, st) : apply_t<kPerMove | kHits, false>(s, b, st);
    }
}

void filter_stats(unsigned long long* out, bool reset) {
    cudaMemcpyFromSymbol(out, g_filter_stats, sizeof(g_filter_stats));
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(g_filter_stats, z, sizeof(z));
    }
}

int classify_occupancy(int, int) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, narrow_census_kernel, 128, 0);
    return n < 1 ? 1 : n;
}

cudaError_t launch_compact(const Store& s, int32_t* out_ids, int32_t* tile_cnt, int32_t* gray_n, cudaStream_t st,
                           int32_t* host_out) {
    const int ntiles = (s.N + kTile - 1) / kTile;
    if (ntiles == 0) return cudaMemsetAsync(gray_n, 0, sizeof(int32_t), st);
    cudaError_t e = launch_pdl(gray_count_kernel, dim3(ntiles), dim3(kCompactThreads), st,
                               static_cast<const uint8_t*>(s.state), s.N, tile_cnt);
    if (e != cudaSuccess) return e;
    return launch_pdl(gray_write_kernel, dim3(ntiles), dim3(kCompactThreads), st, static_cast<const uint8_t*>(s.state),
                      s.N, static_cast<const int32_t*>(tile_cnt), ntiles, out_ids, gray_n, host_out);
}

cudaError_t launch_write_states(const Store& s, const int32_t* ids, const uint8_t* st_in, int n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    write_states_kernel<<<(n + 255) / 256, 256, 0, st>>>(s, ids, st_in, n);
    return cudaGetLastError();
}

cudaError_t launch_pair_masks(const Store& s, const int32_t* rank, int kind, const int32_t* cand, int n, int o,
                              uint8_t* mask, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    pair_masks_kernel<<<(n + 127) / 128, 128, 0, st>>>(s, rank, kind, cand, n, o, mask);
    return cudaGetLastError();
}

cudaError_t launch_fp32_peak(float* sink, int iters, int grid, int block, cudaStream_t st) {
    fp32_peak_kernel<<<grid, block, 0, st>>>(sink, iters);
    return cudaGetLastError();
}

cudaError_t launch_fp64_peak(double* sink, int iters, int grid, int block, cudaStream_t st) {
    fp64_peak_kernel<<<grid, block, 0, st>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace rggk
