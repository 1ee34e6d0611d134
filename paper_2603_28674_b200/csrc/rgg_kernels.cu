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
    const int o = mids[i];
    // prev / last links: the same obstacle moved earlier / later in this batch
    int p = -1;
    bool is_last = true;
    for (int base = 0; base < b.n; base += 32) {
        const int j = base + lane;
        const bool same = j < b.n && mids[j] == o;
        const unsigned before = __ballot_sync(0xffffffffu, same && j < i);
        const unsigned after = __ballot_sync(0xffffffffu, same && j > i);
        if (before) p = base + 31 - __clz(before);
        if (after) is_last = false;
    }
    const double he[3] = {s.ohe[3 * o], s.ohe[3 * o + 1], s.ohe[3 * o + 2]};
    const double* rt_new = mrt + 12 * static_cast<size_t>(i);
    const double* rt_old = p >= 0 ? mrt + 12 * static_cast<size_t>(p) : rt_new;
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
    // the binning boxes first: the bin kernel starts on them (Batch::evready)
    double nu6 = 0.0, ol6 = 0.0;
    if (lane < 6) {
        nu6 = lane < 3 ? fmin(bn[lane], bs[lane]) : fmax(bn[lane], bs[lane]);
        ol6 = p >= 0 ? os[lane] : s.cur_union[6 * o + lane];
        b.evbox[12 * static_cast<size_t>(i) + lane] = nu6;  // compact copy for the binning
        b.evbox[12 * static_cast<size_t>(i) + 6 + lane] = ol6;
    }
    if (b.evready) {  // release: the warp's stores (evbox, and the counter resets of warp 0), then the count
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
    if (lane < 12) ev.rt[lane] = rt_new[lane];
    if (b.src_ids) {  // the HBM copy the later kernels (and a replay) read
        if (lane == 0) const_cast<int32_t*>(b.ids)[i] = o;
        if (lane < 12) const_cast<double*>(b.rt)[12 * static_cast<size_t>(i) + lane] = rt_new[lane];
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
    if (b.unit_ready) {  // release this event's operands to the touch kernel
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(b.evready + 1, 1);
        }
    }
    tl_stop(b.tl, 0, t0);
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

// ------------------------------------------------------------------ binning
//
// One CTA per group of 16 cells (a Morton-contiguous "super-cell", union box
// precomputed), one warp per cell.  Events stream through in chunks of 512:
// each thread loads one event's new/old boxes (compact evbox array, coalesced)
// and tests them against the super-cell box; an ordered block-wide ballot
// compaction leaves the chunk's candidates in shared memory; each warp then
// tests its cell against the candidates and appends hits, in event order, to
// the cell's fixed-capacity list (overflow -> pool) with warp ballots.  Work is
// O(supercells x events + cells x candidates) instead of O(cells x events).

// The per-cell test runs on fp32 boxes rounded outward (lower corners down, upper
// corners up), a superset of the fp64 test: a listed event that touches none of
// the cell's components is dropped by touch's exact per-component test, so the
// lists only need to contain every overlapping event (the overflow pass below
// applies the same two tests, so counts and lists agree).
constexpr int kBinThreads = 512;  // 16 warps = 16 cells per CTA (one super-cell)
constexpr int kBinChunk = 512;    // events filtered per pass

__device__ __forceinline__ void box_out32(const double* d, float* f) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        f[k] = __double2float_rd(d[k]);
        f[3 + k] = __double2float_ru(d[3 + k]);
    }
}
__device__ __forceinline__ bool overlaps32(const float* a, const float* b) {
    return (a[0] <= b[3]) & (b[0] <= a[3]) & (a[1] <= b[4]) & (b[1] <= a[4]) & (a[2] <= b[5]) & (b[2] <= a[5]);
}

// The per-cell record of a listed cell (lane 0 after the warp's list stores): count,
// dirty list, mask block, touch work units, the 16-byte cell record, and the unit
// stamps of the early-touch handoff.
__device__ __forceinline__ void bin_cell_tail(const Store& s, const Batch& b, int cell, int count,
                                              const int32_t* inl, int lane) {
    __syncwarp();  // every lane's list entries precede the unit stamps below
    if (lane == 0) {
        b.cell_count[cell] = count;
        int mbase = 0, ub = 0, W = 0;
        if (count > 0) {
            b.dirty[atomicAdd(&b.ctr[0], 1)] = cell;
            // mask block of the v3 touch / narrow / apply kernels: 3 * ceil(count/32) words per component
            const long long need = 3ll * ((count + 31) >> 5) * s.cell;
            const long long base = atomicAdd(reinterpret_cast<unsigned long long*>(b.mtop),
                                             static_cast<unsigned long long>(need));
            if (base + need > b.mpool_cap) atomicExch(&b.ctr[6], 2);
            mbase = base + need > b.mpool_cap ? 0 : static_cast<int>(base);
            // one touch work unit per chunk of 32 listed events, carrying what the
            // touch kernel needs of the cell record
            W = (count + 31) >> 5;
            ub = atomicAdd(&b.ctr[10], W);
            for (int w = 0; w < W && ub + w < b.units_cap; ++w) b.units[ub + w] = make_int4(cell, w, count, mbase);
        }
        // one 16-byte record per cell: count, mask base, list address
        const int32_t* list = count <= s.cap ? inl : b.pool + b.cell_ovf[cell];
        const unsigned long long a = reinterpret_cast<unsigned long long>(list);
        b.crec[cell] = make_int4(count, mbase, static_cast<int>(a & 0xffffffffu), static_cast<int>(a >> 32));
        if (b.unit_ready && count > 0) {  // release the cell's units (record, list, mask base) to touch
            const int gen = reinterpret_cast<volatile int32_t*>(b.evready)[4];
            __threadfence();
            for (int w = 0; w < W && ub + w < b.units_cap; ++w) b.unit_ready[ub + w] = gen;
        }
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

#ifndef RGG_BIN_MINB
#define RGG_BIN_MINB 2  // two CTAs per SM (registers <= 64)
#endif
__global__ void __launch_bounds__(kBinThreads, RGG_BIN_MINB) bin_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
    if (b.evready) {
        // the pose warps publish their binning boxes first (release: fence + count);
        // the rest of the pose kernel overlaps this kernel, whose end waits for it
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
    const unsigned long long t0 = tl_start(b.tl);
    tl_stop(b.tl, 5, tw);
    __shared__ float cbox[12][kBinChunk];  // SoA: lane q reads column q, conflict-free
    __shared__ int cidx[kBinChunk];
    __shared__ int wsum[kBinThreads / 32];
    __shared__ int s_nc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * (kBinThreads / 32) + warp;
    const bool live = cell < s.ncells;
    double sb[6], cb[6];
    float cbf[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) sb[k] = s.super_aabb[6 * static_cast<size_t>(blockIdx.x) + k];
    if (live) {
        for (int k = 0; k < 6; ++k) cb[k] = s.cell_aabb[6 * static_cast<size_t>(cell) + k];
        box_out32(cb, cbf);
    }
    int count = 0;
    int32_t* inl = b.cell_list + static_cast<size_t>(cell) * s.cap;
    for (int base = 0; base < b.n; base += kBinChunk) {
        // ---- super-cell filter, ordered compaction of the chunk's candidates
        const int e = base + threadIdx.x;
        double bx[12];
        bool cand = false;
        if (threadIdx.x < kBinChunk && e < b.n) {
            const double2* p = reinterpret_cast<const double2*>(b.evbox + 12 * static_cast<size_t>(e));
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const double2 v = p[k];
                bx[2 * k] = v.x;
                bx[2 * k + 1] = v.y;
            }
            cand = rggd::overlaps(sb, bx) | rggd::overlaps(sb, bx + 6);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, cand);
        __syncthreads();
        if (lane == 0) wsum[warp] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int w = 0; w < kBinThreads / 32; ++w) {
                const int t = wsum[w];
                wsum[w] = acc;
                acc += t;
            }
            s_nc = acc;
        }
        __syncthreads();
        if (cand) {
            const int pos = wsum[warp] + __popc(bal & ((1u << lane) - 1u));
            cidx[pos] = e;
            float f[12];
            box_out32(bx, f);
            box_out32(bx + 6, f + 6);
#pragma unroll
            for (int k = 0; k < 12; ++k) cbox[k][pos] = f[k];
        }
        __syncthreads();
        const int nc = s_nc;
        if (!live) continue;
        // ---- per-cell test of the candidates, ordered ballot append
        for (int j = 0; j < nc; j += 32) {
            const int q = j + lane;
            bool hit = false;
            if (q < nc) {
                float qb[12];
#pragma unroll
                for (int k = 0; k < 12; ++k) qb[k] = cbox[k][q];
                hit = overlaps32(cbf, qb) | overlaps32(cbf, qb + 6);
            }
            const unsigned hb = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int pos = count + __popc(hb & ((1u << lane) - 1u));
                if (pos < s.cap) inl[pos] = cidx[q];
            }
            count += __popc(hb);
        }
    }
    if (!live) {
        if (b.evready) pdl_wait();  // the grid ends after the pose kernel (touch waits on this grid only)
        return;
    }
    if (count > s.cap) {
        // Overflow: the full ordered list goes to the pool (second pass over the events).
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
                if (e < b.n) {  // the same two tests as the listing pass
                    const double* bx = b.evbox + 12 * static_cast<size_t>(e);
                    float f[12];
                    box_out32(bx, f);
                    box_out32(bx + 6, f + 6);
                    hit = (rggd::overlaps(sb, bx) | rggd::overlaps(sb, bx + 6)) &&
                          (overlaps32(cbf, f) | overlaps32(cbf, f + 6));
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (hit) b.pool[pbase + at + __popc(bal & ((1u << lane) - 1u))] = e;
                at += __popc(bal);
            }
            if (lane == 0) b.cell_ovf[cell] = pbase;
        }
    }
    bin_cell_tail(s, b, cell, count, inl, lane);
    tl_stop(b.tl, 1, t0);
    bin_warp_done(b, lane);
    if (b.evready) pdl_wait();
}

// Small batches (n <= 64 moves): one warp per cell, no super-cell stage.  Lane l
// tests events l and l + 32 (exact fp64 closed-box tests of the new and old
// boxes), two ordered ballots build the list.  Small warps-per-CTA so every cell's
// warp is resident in one wave even for a million components (c4: 8400 cells).
constexpr int kBinSmallMax = 64;
constexpr int kBinSmallWarps = 8;

__global__ void __launch_bounds__(32 * kBinSmallWarps) bin_small_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
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
    const unsigned long long t0 = tl_start(b.tl);
    tl_stop(b.tl, 5, tw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cell = blockIdx.x * kBinSmallWarps + warp;
    if (cell >= s.ncells) {
        if (b.evready) pdl_wait();
        return;
    }
    double cb[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) cb[k] = s.cell_aabb[6 * static_cast<size_t>(cell) + k];
    unsigned bal[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int e = 32 * h + lane;
        bool hit = false;
        if (e < b.n) {
            const double* bx = b.evbox + 12 * static_cast<size_t>(e);
            hit = rggd::overlaps(cb, bx) | rggd::overlaps(cb, bx + 6);
        }
        bal[h] = __ballot_sync(0xffffffffu, hit);
    }
    int count = __popc(bal[0]) + __popc(bal[1]);
    int32_t* inl = b.cell_list + static_cast<size_t>(cell) * s.cap;
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
    bin_cell_tail(s, b, cell, count, inl, lane);
    tl_stop(b.tl, 1, t0);
    bin_warp_done(b, lane);
    if (b.evready) pdl_wait();
}

// ----------------------------------------------------------------- classify

// batch_over for one (component, obstacle) pair: any body intersects (engine_batch.cpp:55-74).
// filter outcome counters (tests / RGG_DEBUG_TIMING): [0] SAT filtered, [1] SAT rechecked in
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
            int f;
            if (s.dbg_flags & 512) {  // 512: the axis-form filter
                const rggd::Box32& a32 = s.sat32[i];
                f = rggd::sat_filter32(a32.c, a32, osat, ev.b32);
            } else {
                const rggd::Box32G a32 = rggd::load_box32g(s.sat32 + i), o32 = rggd::load_box32g(&ev.b32);
                f = rggd::sat_filter32g(a32, o32.c, o32);
            }
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
            if (COUNT) {
                *tests += 1;
                hit |= rggd::seg_sphere_fast(seg, ev.cen + 3 * sp, r_total);
            } else {
                const int f = rggd::seg_filter32(seg, ev.cen + 3 * sp, r_total);
                if (f == 1 || (f == 2 && seg_exact(seg, ev.cen + 3 * sp, r_total))) return true;
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
// is read only when a sphere is undecided.  Verdicts are the reference's.
__device__ __forceinline__ bool under_range32(const Store& s, int lo, int hi, const Event& ev) {
    const int nsph = ev.nsph;
    for (int j = lo; j < hi; ++j) {
        const float4 v0 = s.seg32[2 * static_cast<size_t>(j)], v1 = s.seg32[2 * static_cast<size_t>(j) + 1];
        const rggd::SegF g = rggd::segf_prep(v0, v1, ev.r);
        bool sure = false;
        uint32_t und = 0;
#pragma unroll 4
        for (int sp = 0; sp < nsph; ++sp) {
            const float cx = __double2float_rn(ev.cen[3 * sp]), cy = __double2float_rn(ev.cen[3 * sp + 1]),
                        cz = __double2float_rn(ev.cen[3 * sp + 2]);
            const int f = rggd::segf_filter(g, cx, cy, cz, (fabsf(cx) + fabsf(cy)) + fabsf(cz));
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

constexpr int kUnderLanes = 4;  // lanes per under-approximation work item
constexpr int kStageEv = 128;   // touch stages a whole batch of up to this many events per CTA

// ------------------------------------------------------- v3: touch / narrow / apply
//
// Per cell with L listed events the bin kernel reserves a mask block of
// 3 * ceil(L/32) * cell words: touch[w][t], over[w][t], under[w][t] (bit k of
// word w = the cell's event at list position 32w + k, for component t of the
// cell).  touch fills the touch words and emits one work item per (component,
// event) pair whose boxes overlap; narrow evaluates every item with the whole
// GPU and ORs the verdicts into the result words; apply replays each
// component's events in move order from the three words.

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

// the moved obstacles' operands, alone (a store without components)
__global__ void commit_kernel(Store s, Batch b) { commit_grid(s, b); }

__device__ __forceinline__ const int32_t* rec_list(int4 r) {
    return reinterpret_cast<const int32_t*>((static_cast<unsigned long long>(static_cast<uint32_t>(r.w)) << 32) |
                                            static_cast<uint32_t>(r.z));
}

// Narrow tests of a pair whose item did not fit the queue (kept out of line so
// the touch kernel's register budget stays that of an AABB filter).
__device__ __noinline__ bool over_inline(const Store& s, int c, const Event& ev) {
    return over_test<false>(s, c, ev, nullptr);
}
__device__ __noinline__ bool under_inline(const Store& s, int c, const Event& ev) {
    return under_part<false>(s, c, ev, 0, 1, nullptr);
}

__global__ void __launch_bounds__(kMaxCell) touch_kernel(Store s, Batch b) {
    __shared__ double sbox[kEvChunk][24];  // nu, old, box, sph of the chunk's events
    __shared__ int sev[kEvChunk];
    __shared__ int s_no, s_nu, s_bo, s_bu;
    __shared__ unsigned long long scen[4];
    const int cell = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    commit_grid(s, b);
    const int4 rec = b.crec[cell];
    const int count = rec.x;
    if (count == 0) return;
    const bool census = b.census_on != 0;
    if (census && tid < 4) scen[tid] = 0;
    const int32_t* list = rec_list(rec);
    const int W = (count + 31) >> 5, T = s.cell;
    const int mbase = rec.y;
    const int c = cell * T + tid;
    const bool valid = c < s.Np;
    double aabb[6];
    if (valid) {
        const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
        aabb[0] = a0.x, aabb[1] = a0.y, aabb[2] = a1.x, aabb[3] = a1.y, aabb[4] = a2.x, aabb[5] = a2.y;
    }
    bool any_box = false, any_sph = false;
    for (int w = 0; w < W; ++w) {
        const int m = min(32, count - 32 * w);
        __syncthreads();
        if (tid < m) sev[tid] = list[32 * w + tid];
        if (tid == 0) s_no = s_nu = 0;
        __syncthreads();
        for (int t = tid; t < m * 24; t += blockDim.x) {
            const int e = t / 24, k = t % 24;
            const Event& ev = b.ev[sev[e]];
            sbox[e][k] = k < 6 ? ev.nu[k] : (k < 12 ? ev.old[k - 6] : (k < 18 ? ev.box[k - 12] : ev.sph[k - 18]));
        }
        __syncthreads();
        uint32_t tm = 0, bm = 0, sm = 0;
        if (valid) {
            for (int k = 0; k < m; ++k) {
                if (rggd::overlaps(aabb, sbox[k]) || rggd::overlaps(aabb, sbox[k] + 6)) {
                    tm |= 1u << k;
                    if (rggd::overlaps(aabb, sbox[k] + 12)) bm |= 1u << k;
                    if (s.use_under && rggd::overlaps(aabb, sbox[k] + 18)) sm |= 1u << k;
                }
            }
        }
        const int wt = mbase + (0 * W + w) * T + tid, wo = mbase + (1 * W + w) * T + tid,
                  wu = mbase + (2 * W + w) * T + tid;
        b.mpool[wt] = tm;
        b.mpool[wo] = 0;
        b.mpool[wu] = 0;
        any_box |= bm != 0;
        any_sph |= sm != 0;
        // block-level reservation in the item queues: one global atomic per queue per CTA
        const int no = __popc(bm), nu = __popc(sm);
        int xo = no, xu = nu;
        for (int off = 1; off < 32; off <<= 1) {
            const int yo = __shfl_up_sync(0xffffffffu, xo, off), yu = __shfl_up_sync(0xffffffffu, xu, off);
            if (lane >= off) xo += yo, xu += yu;
        }
        int wbo = 0, wbu = 0;
        if (lane == 31) {
            wbo = atomicAdd(&s_no, xo);
            wbu = atomicAdd(&s_nu, xu);
        }
        __syncthreads();
        if (tid == 0) {
            s_bo = s_no ? atomicAdd(&b.ctr[8], s_no) : 0;
            s_bu = s_nu ? atomicAdd(&b.ctr[9], s_nu) : 0;
        }
        __syncthreads();
        wbo = __shfl_sync(0xffffffffu, wbo, 31);
        wbu = __shfl_sync(0xffffffffu, wbu, 31);
        int at = s_bo + wbo + xo - no;
        for (uint32_t x = bm; x; x &= x - 1, ++at) {
            const int k = __ffs(x) - 1;
            if (at < b.items_cap)
                b.items_over[at] = make_int4(c, sev[k], wo, 1 << k);
            else if (over_inline(s, c, b.ev[sev[k]]))
                b.mpool[wo] |= 1u << k;  // this thread owns the word until the narrow kernel
        }
        at = s_bu + wbu + xu - nu;
        const int ulo = sm ? s.row[c * s.B * s.S] : 0, uhi = sm ? s.row[(c + 1) * s.B * s.S] : 0;
        for (uint32_t x = sm; x; x &= x - 1, ++at) {
            const int k = __ffs(x) - 1;
            if (at < b.items_cap)
                b.items_under[at] = make_int4(ulo, uhi, wu, (sev[k] << 5) | k);
            else if (under_inline(s, c, b.ev[sev[k]]))
                b.mpool[wu] |= 1u << k;
        }
    }
    if (census) {
        // algorithmic-bytes census: components of dirty cells,
        // components reading SatBoxes, components reading segments, segments read
        int segs = 0;
        if (valid && any_sph) {
            const int rows = s.B * s.S;
            segs = s.row[(c + 1) * rows] - s.row[c * rows];
        }
        unsigned long long v[4] = {valid ? 1ull : 0ull, any_box ? 1ull : 0ull, any_sph ? 1ull : 0ull,
                                   static_cast<unsigned long long>(segs)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            unsigned long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&scen[k], x);
        }
        __syncthreads();
        if (tid < 4 && scen[tid]) atomicAdd(&b.census[8 + tid], scen[tid]);
    }
}

// The narrow tests of all items, GPU-wide (persistent grid).  Over items
// {component, event, result word, bit}: one thread each (15-axis SAT per body).
// Under items {first segment, end segment, result word, event << 5 | bit}: G
// lanes each.
template <bool COUNT, int G>
__global__ void __launch_bounds__(128) narrow_kernel(Store s, Batch b) {
    const unsigned long long tw = COUNT ? 0 : tl_start(b.tl);
    pdl_wait();
    pdl_trigger();
    const unsigned long long t0 = COUNT ? 0 : tl_start(b.tl);
    if (!COUNT) tl_stop(b.tl, 7, tw);
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    unsigned long long* dbgw = (!COUNT && b.dbg) ? b.dbg + 4 * static_cast<size_t>(gt >> 5) : nullptr;
    if (dbgw && lane == 0) dbgw[0] = gtimer();
    const int n_over = min(b.ctr[8], b.items_cap), n_under = min(b.ctr[9], b.items_cap);
    long long c_sat = 0, c_tests = 0, c_op = 0, c_up = 0, c_oh = 0, c_uh = 0;
    if (!COUNT && G == 1) {
        // One pass over both queues (over items first).  The next item is loaded
        // while the current one is tested, and an under item's segment records
        // are prefetched into L1 before they are walked: about one exposed memory
        // round trip per item instead of one per load.
        const int total = n_over + n_under;
        const auto item = [&](int i) {
            return i < n_over ? b.items_over[i] : b.items_under[i - n_over];
        };
        // two items ahead: the item after next is loaded and the next item's operands
        // are prefetched into L1 while the current one is tested
        int i = gt;
        int4 it = i < total ? item(i) : make_int4(0, 0, 0, 0);
        int4 nx = i + nthreads < total ? item(i + nthreads) : make_int4(0, 0, 0, 0);
        unsigned long long d_items = 0, d_segs = 0;
        while (i < total) {
            if (dbgw) d_items += 1, d_segs += i < n_over ? 0 : it.y - it.x;
            const int inext = i + nthreads, i2 = inext + nthreads;
            const int4 nn = i2 < total ? item(i2) : make_int4(0, 0, 0, 0);
            if (inext < total) {
                if (inext < n_over) {
                    prefetch_l1(s.sat32 + static_cast<size_t>(nx.x) * s.B);
                } else {
                    for (int j = nx.x; j < nx.y; j += 4) prefetch_l1(s.seg32 + 2 * static_cast<size_t>(j));
                }
            }
            if (i < n_over) {
                if (!(s.dbg_flags & 128) && over_test<false>(s, it.x, b.ev[it.y], nullptr) &&
                    !(s.dbg_flags & 1024))  // 128: ablation, no over tests; 1024: no result atomics
                    atomicOr(&b.mpool[it.z], static_cast<uint32_t>(it.w));
            } else if (s.dbg_flags & 256) {  // 256: ablation, no under tests
            } else {
                if (under_range32(s, it.x, it.y, b.ev[it.w >> 5]) && !(s.dbg_flags & 1024))
                    atomicOr(&b.mpool[it.z], 1u << (it.w & 31));
            }
            it = nx;
            nx = nn;
            i = inext;
        }
        if (dbgw) {
            // lane maxima: items, segments
            for (int off = 16; off; off >>= 1) {
                d_items = max(d_items, __shfl_xor_sync(0xffffffffu, d_items, off));
                d_segs = max(d_segs, __shfl_xor_sync(0xffffffffu, d_segs, off));
            }
        }
        if (dbgw && lane == 0) dbgw[2] = d_items, dbgw[3] = d_segs;
    }
    for (int i = gt; i < (COUNT || G > 1 ? n_over : 0); i += nthreads) {
        const int4 it = b.items_over[i];  // component, event, result word, bit
        const bool h = over_test<COUNT>(s, it.x, b.ev[it.y], &c_sat);
        if (COUNT) c_op += s.B, c_oh += h;
        if (h) atomicOr(&b.mpool[it.z], static_cast<uint32_t>(it.w));
    }
    const int g = gt % G, groups = nthreads / G;
    const unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (lane & ~(G - 1));
    for (int i = gt / G; i < (COUNT || G > 1 ? n_under : 0); i += groups) {
        const int4 it = b.items_under[i];
        bool h = under_range<COUNT>(s, it.x, it.y, b.ev[it.w >> 5], g, G, &c_tests);
#pragma unroll
        for (int off = 1; off < G; off <<= 1) {
            const bool other = __shfl_xor_sync(gmask, h, off);  // the group's lanes share i
            h = h || other;
        }
        if (COUNT) c_up += 1, c_uh += h;
        if (h && g == 0) atomicOr(&b.mpool[it.z], 1u << (it.w & 31));
    }
    if (dbgw) {
        __syncwarp();
        if (lane == 0) dbgw[1] = gtimer();
    }
    if (!COUNT) tl_stop(b.tl, 3, t0);
    if (COUNT) {
        long long v[6] = {c_op, c_sat, c_up, c_tests, c_oh, c_uh};
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&b.census[k], static_cast<unsigned long long>(x));
        }
        return;
    }
}

// Per-move transitions (engine_batch.cpp:114-188) of every component of a
// dirty cell, in list (= move) order, from the touch / over / under words.
template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(kMaxCell) apply_kernel(Store s, Batch b) {
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    constexpr bool HITS = (FLAGS & kHits) != 0;
    __shared__ int s_o[32], s_move[32];
    __shared__ int scnt[32][4];
    const int cell = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
    const int4 rec = b.crec[cell];
    const int count = rec.x;
    if (count == 0) return;
    const int32_t* list = rec_list(rec);
    const int W = (count + 31) >> 5, T = s.cell;
    const uint32_t* mb = b.mpool + rec.y;
    const int c = cell * T + tid;
    const bool valid = c < s.Np;
    int label = 0, oc = 0, bc = 0, id = -1;
    unsigned long long OW = 0, UW = 0;
    if (valid) {
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
    bool hit_last = false;
    for (int w = 0; w < W; ++w) {
        const int m = min(32, count - 32 * w);
        __syncthreads();
        if (tid < m) {
            const Event& ev = b.ev[list[32 * w + tid]];
            s_o[tid] = ev.o;
            s_move[tid] = ev.move;
        }
        if (PER_MOVE)
            for (int t = tid; t < m * 4; t += blockDim.x) scnt[t >> 2][t & 3] = 0;
        __syncthreads();
        const uint32_t tm = mb[(0 * W + w) * T + tid], ro = mb[(1 * W + w) * T + tid],
                       ru = mb[(2 * W + w) * T + tid];
        for (int k = 0; k < m; ++k) {
            const int before = label;
            if (valid && ((tm >> k) & 1u)) {
                const int o = s_o[k];
                const int wo = o >> 6;
                const unsigned long long bit = 1ull << (o & 63);
                unsigned long long ow, uw;
                if (WIDE) {
                    ow = s.over[static_cast<size_t>(wo) * s.Np + c];
                    uw = s.under[static_cast<size_t>(wo) * s.Np + c];
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
                    if (nw != ow) s.over[static_cast<size_t>(wo) * s.Np + c] = nw;
                    if (nuw != uw) s.under[static_cast<size_t>(wo) * s.Np + c] = nuw;
                } else {
                    OW = nw;
                    UW = nuw;
                }
                if (HITS && s_move[k] == b.n - 1) hit_last = n_over;
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
                if (v) atomicAdd(&b.mv[4 * s_move[t >> 2] + (t & 3)], v);
            }
        }
    }
    int dgray = 0;
    if (valid) {
        if (label != label0) {
            s.state[id] = static_cast<uint8_t>(label);
            s.state_c[c] = static_cast<uint8_t>(label);
            dgray = (label == 2) - (label0 == 2);
        }
        const uint32_t cw = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
        if (cw != cnt0) s.cnt[c] = cw;
        if (!WIDE) {
            if (OW != OW0) s.over[c] = OW;
            if (UW != UW0) s.under[c] = UW;
        }
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
        if (h) {
                const int at = pos + __popc(bal & ((1u << lane) - 1u));
                b.hits[at] = id;
                b.hits_prev[at] = static_cast<uint8_t>(label0);
            }
    }
}

// ------------------------------------------------- v4: warp-centric fused classify
//
// One warp owns a slice of 32 consecutive (cell-sorted) components and runs
// the whole per-update work of that slice warp-synchronously, with no CTA
// barrier: its operands are loaded up front, each lane builds its touch / box /
// sphere masks over the cell's event list (32 events per pass, boxes read as
// warp-broadcast L1 loads), the (component, event) pairs needing a narrow test
// become a warp-local work list that all 32 lanes drain (SATs one lane each,
// segment-sphere tests kUnderLanes lanes each), and each lane then replays its
// events in move order with the reference's transition.  Warps are persistent
// and stride over the slices, so there is no dependence on CTA scheduling.
constexpr int kWarpsPerCta = 4;
static_assert(kStageEv <= 32 * kWarpsPerCta, "the touch staging table is the warps' chunk buffers");
constexpr int kStageIds = 1024;  // apply stages the moved obstacle ids of batches up to this size

template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(32 * kWarpsPerCta) classify_warp_kernel(Store s, Batch b) {
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    constexpr bool HITS = (FLAGS & kHits) != 0;
    constexpr bool CENSUS = (FLAGS & kCensus) != 0;
    __shared__ uint16_t sitem[kWarpsPerCta][2][32 * 32];
    __shared__ uint32_t sres[kWarpsPerCta][2][32];
    __shared__ int sev[kWarpsPerCta][32];
    __shared__ double sbx[kWarpsPerCta][32][24];  // per event: nu, old, box, sph (one load wave per chunk)
    __shared__ int2 som[kWarpsPerCta][32];        // per event: obstacle id, move index
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = (s.Np + 31) >> 5;
    if (!CENSUS) commit_grid(s, b);
    long long c_sat = 0, c_tests = 0, c_op = 0, c_up = 0, c_oh = 0, c_uh = 0;
    unsigned long long c_dirty = 0, c_box = 0, c_sph = 0, c_segs = 0, c_touch = 0;
    int dgray = 0;
    // slices near an obstacle are Morton-adjacent and heavy: spread them over warps / SMs by
    // walking the slices with a prime stride (a bijection when it does not divide nslices)
    const long long stride = (nslices % 7919) ? 7919 : 1;
    for (int q0 = blockIdx.x * kWarpsPerCta + wi; q0 < nslices; q0 += gridDim.x * kWarpsPerCta) {
        const int q = static_cast<int>((q0 * stride) % nslices);
        const int c0 = q << 5;
        const int cell = c0 / s.cell;
        const int4 rec = b.crec[cell];
        const int count = rec.x;
        if (count == 0) continue;  // warp-uniform: clean cell
        const int c = c0 + lane;
        const bool valid = c < s.Np;
        const int rows = s.B * s.S;
        int seg_lo = 0, seg_hi = 0;
        double aabb[6];
        int label = 0, oc = 0, bc = 0, id = -1;
        unsigned long long OW = 0, UW = 0;
        if (valid) {
            seg_lo = s.row[c * rows];
            seg_hi = s.row[(c + 1) * rows];
            const double2 a0 = s.aabb[c], a1 = s.aabb[s.Np + c], a2 = s.aabb[2 * s.Np + c];
            aabb[0] = a0.x, aabb[1] = a0.y, aabb[2] = a1.x, aabb[3] = a1.y, aabb[4] = a2.x, aabb[5] = a2.y;
            if (!CENSUS) {
                id = s.orig[c];
                const uint32_t cw = s.cnt[c];
                oc = cw & 0xffff;
                bc = cw >> 16;
                if (!WIDE) {
                    OW = s.over[c];
                    UW = s.under[c];
                }
                label = s.state[id];
            }
        }
        const int label0 = label;
        const uint32_t cnt0 = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
        const unsigned long long OW0 = OW, UW0 = UW;
        bool hit_last = false, any_box = false, any_sph = false;
        unsigned long long* dbg = b.dbg ? b.dbg + 16 * static_cast<size_t>(q) : nullptr;
        const long long clk0 = clock64();
        if (dbg && lane == 0) dbg[0] = gtimer(), dbg[8] = count;
#define RGG_STAMP(i) if (dbg) { __syncwarp(); if (lane == 0) dbg[i] = gtimer(); }
        if (dbg && __any_sync(0xffffffffu, label == 77)) dbg[14] = 1;  // waits for the component loads
        RGG_STAMP(1)
        const int32_t* list = rec_list(rec);
        for (int base = 0; base < count; base += 32) {
            const int m = min(32, count - base);
            const int myev = lane < m ? list[base + lane] : 0;
            sev[wi][lane] = myev;
            if (lane < m) {  // lane k stages event k: one load wave for the whole chunk
                const Event& ev = b.ev[myev];
                double v[24];
#pragma unroll
                for (int j = 0; j < 6; ++j) v[j] = ev.nu[j], v[6 + j] = ev.old[j], v[12 + j] = ev.box[j], v[18 + j] = ev.sph[j];
#pragma unroll
                for (int j = 0; j < 24; ++j) sbx[wi][lane][j] = v[j];
                som[wi][lane] = make_int2(ev.o, ev.move);
            }
            __syncwarp();
            if (base == 0) {
                if (dbg && __any_sync(0xffffffffu, valid && aabb[0] == -1.25e300)) dbg[15] = 1;  // waits for the AABB
                RGG_STAMP(2)
            }
            // ---- touch / box / sphere masks
            uint32_t tm = 0, bm = 0, sm = 0;
            if (valid) {
                for (int k = 0; k < m; ++k) {
                    const double* bx = sbx[wi][k];
                    const bool touch = rggd::overlaps(aabb, bx) | rggd::overlaps(aabb, bx + 6);
                    tm |= static_cast<uint32_t>(touch) << k;
                    bm |= static_cast<uint32_t>(touch & rggd::overlaps(aabb, bx + 12)) << k;
                    sm |= static_cast<uint32_t>(touch & (s.use_under != 0) & rggd::overlaps(aabb, bx + 18)) << k;
                }
            }
            any_box |= bm != 0;
            any_sph |= sm != 0;
            if (CENSUS) c_touch += __popc(tm);
            // pull this lane's narrow operands towards the SM now: the work list is
            // drained by other lanes of the warp, which then hit in L1
            if (bm) {
                const size_t i0 = static_cast<size_t>(c) * s.B;
                prefetch_range(s.sat + i0 * 22, s.sat + (i0 + s.B) * 22, true);
                prefetch_range(s.sat32 + i0, s.sat32 + i0 + s.B, true);
            }
            if (sm) prefetch_range(s.seg + 8 * static_cast<size_t>(seg_lo), s.seg + 8 * static_cast<size_t>(seg_hi), true);
            if (base == 0) RGG_STAMP(3)
            // ---- warp-local narrow work list
            const int no = __popc(bm), nu = __popc(sm);
            int xo = no, xu = nu;
            for (int off = 1; off < 32; off <<= 1) {
                const int yo = __shfl_up_sync(0xffffffffu, xo, off), yu = __shfl_up_sync(0xffffffffu, xu, off);
                if (lane >= off) xo += yo, xu += yu;
            }
            const int tot_o = __shfl_sync(0xffffffffu, xo, 31), tot_u = __shfl_sync(0xffffffffu, xu, 31);
            {
                int po = xo - no, pu = xu - nu;
                for (uint32_t x = bm; x; x &= x - 1) sitem[wi][0][po++] = static_cast<uint16_t>((lane << 5) | (__ffs(x) - 1));
                for (uint32_t x = sm; x; x &= x - 1) sitem[wi][1][pu++] = static_cast<uint16_t>((lane << 5) | (__ffs(x) - 1));
            }
            sres[wi][0][lane] = 0;
            sres[wi][1][lane] = 0;
            __syncwarp();
            if (base == 0) RGG_STAMP(4)
            for (int i = lane; i < tot_o; i += 32) {
                const int it = sitem[wi][0][i], t = it >> 5, k = it & 31;
                if (!CENSUS && (s.dbg_flags & 1)) {  // ablation: no test
                    if ((s.dbg_flags & 2) == 0 && s.sat[(c0 + t) * 22] == 12345.0) atomicOr(&sres[wi][0][t], 1u << k);
                    continue;
                }
                const bool h = over_test<CENSUS>(s, c0 + t, b.ev[sev[wi][k]], &c_sat);
                if (CENSUS) c_op += s.B, c_oh += h;
                if (h) atomicOr(&sres[wi][0][t], 1u << k);
            }
            const int g = lane % kUnderLanes;
            for (int ub = 0; ub < tot_u; ub += 32 / kUnderLanes) {
                const int i = ub + lane / kUnderLanes;
                bool h = false;
                int t = 0, k = 0;
                if (i < tot_u && (!CENSUS || g == 0)) {  // census: one lane counts the whole item
                    const int it = sitem[wi][1][i];
                    t = it >> 5;
                    k = it & 31;
                    if (!CENSUS && (s.dbg_flags & 1))  // ablation: no test
                        h = (s.dbg_flags & 2) == 0 && s.seg[8 * static_cast<size_t>(seg_lo)] == 12345.0;
                    else
                    h = under_part<CENSUS>(s, c0 + t, b.ev[sev[wi][k]], CENSUS ? 0 : g, CENSUS ? 1 : kUnderLanes,
                                           &c_tests);
                }
                if (!CENSUS) {
#pragma unroll
                    for (int off = 1; off < kUnderLanes; off <<= 1) {
                        const bool other = __shfl_xor_sync(0xffffffffu, h, off);  // every lane shuffles
                        h = h || other;
                    }
                }
                if (i < tot_u && g == 0) {
                    if (CENSUS) c_up += 1, c_uh += h;
                    if (h) atomicOr(&sres[wi][1][t], 1u << k);
                }
            }
            __syncwarp();
            if (base == 0) RGG_STAMP(5)
            if (dbg && lane == 0 && base == 0) dbg[9] = tot_o, dbg[10] = tot_u;
            if (CENSUS) continue;
            // ---- transitions in move order (engine_batch.cpp:114-188)
            const uint32_t ro = sres[wi][0][lane], ru = sres[wi][1][lane];
            for (int k = 0; k < m; ++k) {
                const int before = label;
                const int2 om = som[wi][k];
                if ((tm >> k) & 1u) {
                    const int o = om.x;
                    const int wo = o >> 6;
                    const unsigned long long bit = 1ull << (o & 63);
                    unsigned long long ow, uw;
                    if (WIDE) {
                        ow = s.over[static_cast<size_t>(wo) * s.Np + c];
                        uw = s.under[static_cast<size_t>(wo) * s.Np + c];
                    } else {
                        ow = OW;
                        uw = UW;
                    }
                    const bool old_over = (ow & bit) != 0, old_under = (uw & bit) != 0;
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
                    const unsigned long long nw = n_over ? (ow | bit) : (ow & ~bit);
                    const unsigned long long nuw = n_under ? (uw | bit) : (uw & ~bit);
                    if (WIDE) {
                        if (nw != ow) s.over[static_cast<size_t>(wo) * s.Np + c] = nw;
                        if (nuw != uw) s.under[static_cast<size_t>(wo) * s.Np + c] = nuw;
                    } else {
                        OW = nw;
                        UW = nuw;
                    }
                    if (HITS && om.y == b.n - 1) hit_last = n_over;
                }
                if (PER_MOVE) {
                    const bool ch = label != before;
                    const unsigned gg = __ballot_sync(0xffffffffu, ch && label == 0);
                    const unsigned r = __ballot_sync(0xffffffffu, ch && label == 1);
                    const unsigned y = __ballot_sync(0xffffffffu, ch && label == 2);
                    const unsigned f = __ballot_sync(0xffffffffu, ch && before == 2);
                    if (lane == 0 && (gg | r | y | f) && !(s.dbg_flags & 4)) {  // 4: ablation, no counters
                        int* mv = b.mv + 4 * om.y;
                        if (gg) atomicAdd(mv + 0, __popc(gg));
                        if (r) atomicAdd(mv + 1, __popc(r));
                        if (y) atomicAdd(mv + 2, __popc(y));
                        if (f) atomicAdd(mv + 3, __popc(f));
                    }
                }
            }
        }
        if (dbg && !CENSUS) RGG_STAMP(6)
        if (CENSUS) {
            if (valid) {
                c_dirty += 1;
                c_box += any_box;
                c_sph += any_sph;
                if (any_sph) c_segs += seg_hi - seg_lo;
            }
            continue;
        }
        if (valid) {
            if (label != label0) {
                s.state[id] = static_cast<uint8_t>(label);
                s.state_c[c] = static_cast<uint8_t>(label);
                dgray += (label == 2) - (label0 == 2);
            }
            const uint32_t cw = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
            if (cw != cnt0) s.cnt[c] = cw;
            if (!WIDE) {
                if (OW != OW0) s.over[c] = OW;
                if (UW != UW0) s.under[c] = UW;
            }
        }
        if (HITS) {
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
        if (dbg) {
            __syncwarp();
            if (lane == 0) dbg[7] = gtimer(), dbg[11] = static_cast<unsigned long long>(clock64() - clk0);
        }
    }
    if (CENSUS) {
        long long v[11] = {c_op, c_sat, c_up, c_tests, c_oh, c_uh, 0, 0, 0, 0, 0};
        v[6] = static_cast<long long>(c_dirty);
        v[7] = static_cast<long long>(c_box);
        v[8] = static_cast<long long>(c_sph);
        v[9] = static_cast<long long>(c_segs);
        v[10] = static_cast<long long>(c_touch);
#pragma unroll
        for (int k = 0; k < 11; ++k) {
            long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&b.census[k < 6 ? k : k + 2], static_cast<unsigned long long>(x));
        }
    } else {
        // running gray count (the unknown_count of the reference)
        for (int off = 16; off; off >>= 1) dgray += __shfl_down_sync(0xffffffffu, dgray, off);
        if (lane == 0 && dgray) atomicAdd(b.unknown, dgray);
    }
}

// ------------------------------------------------- v6: warp-slice touch / GPU-wide narrow / warp-slice apply
//
// v4 split at its narrow phase.  A warp owns a 32-component slice (as in v4)
// for the touch masks and for the transitions, but the narrow tests of all
// slices are drained by one GPU-wide kernel (one (component, event) item per
// thread, 4 lanes per segment-sphere item), so a slice next to an obstacle no
// longer serialises its SAT / segment rounds on one warp.  Masks live in the
// per-cell mask blocks the bin kernel reserves (word (kind*W + w)*cell + t).

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
    // event operands: for small batches (n <= kStageEv) the whole batch is staged
    // once per CTA and the slices index it through their cell lists; otherwise
    // each warp stages its current chunk of 32 listed events
    __shared__ double sbx[kWarpsPerCta * 32][24];
    __shared__ int sev[kWarpsPerCta][32];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = (s.Np + 31) >> 5;
    const bool staged = b.n <= kStageEv && (s.dbg_flags & 64);  // 64: stage the batch in shared memory
    if (!staged) {  // the batch's operands into this SM's L1 (read per chunk below)
        const char* p = reinterpret_cast<const char*>(b.evt);
        const int lines = (b.n * 24 * 8 + 127) >> 7;
        for (int l = threadIdx.x; l < min(lines, 256); l += blockDim.x) prefetch_l1(p + (static_cast<size_t>(l) << 7));
    }
    if (staged) {  // all loads in flight at once, then the stores
        constexpr int kPer = kStageEv * 12 / (32 * kWarpsPerCta);
        const double2* src = reinterpret_cast<const double2*>(b.evt);
        double2* dst = reinterpret_cast<double2*>(&sbx[0][0]);
        const int nv = b.n * 12;
        double2 v[kPer];
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
            const int t = threadIdx.x + r * 32 * kWarpsPerCta;
            if (t < nv) v[r] = src[t];
        }
#pragma unroll
        for (int r = 0; r < kPer; ++r) {
            const int t = threadIdx.x + r * 32 * kWarpsPerCta;
            if (t < nv) dst[t] = v[r];
        }
        __syncthreads();
    }
    unsigned long long c_dirty = 0, c_box = 0, c_sph = 0, c_segs = 0, c_touch = 0;
    unsigned long long* dbgw = (!CENSUS && b.dbg) ? b.dbg + 8 * static_cast<size_t>(nslices) +
                                                        4 * static_cast<size_t>((blockIdx.x * blockDim.x + threadIdx.x) >> 5)
                                                  : nullptr;
    if (dbgw && lane == 0) dbgw[0] = gtimer();
    int dbg_slices = 0;
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
        double aabb[6];
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
            if (!staged && lane < m) {
                const double2* src = reinterpret_cast<const double2*>(b.evt + 24 * static_cast<size_t>(myev));
#pragma unroll
                for (int j = 0; j < 12; ++j) {
                    const double2 v = src[j];
                    sbx[32 * wi + lane][2 * j] = v.x;
                    sbx[32 * wi + lane][2 * j + 1] = v.y;
                }
            }
            __syncwarp();
            uint32_t tm = 0, bm = 0, sm = 0;
            if (valid) {
                for (int k = 0; k < m; ++k) {
                    const double* bx = sbx[staged ? sev[wi][k] : 32 * wi + k];
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
                const unsigned long long mine = static_cast<unsigned long long>(__popc(bm)) |
                                                (static_cast<unsigned long long>(__popc(sm)) << 32);
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
            for (uint32_t x = sm; x; x &= x - 1, ++at) {
                const int k = __ffs(x) - 1;
                if (at < b.items_cap) b.items_under[at] = make_int4(seg_lo, seg_hi, wu, (sev[wi][k] << 5) | k);
                else b.ctr[6] = 3;
            }
            __syncwarp();
        }
        if (CENSUS && valid) {
            c_dirty += 1;
            c_box += any_box;
            c_sph += any_sph;
            if (any_sph) c_segs += seg_hi - seg_lo;
        }
        ++dbg_slices;
    }
    if (dbgw) {
        __syncwarp();
        if (lane == 0) dbgw[1] = gtimer(), dbgw[2] = dbg_slices, dbgw[3] = 0;
    }
    if (!CENSUS) tl_stop(b.tl, 2, t0);
    if (flow) pdl_wait();  // the grid ends after bin's (narrow waits on this grid only)
    if (CENSUS) {
        unsigned long long v[5] = {c_dirty, c_box, c_sph, c_segs, c_touch};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
            unsigned long long x = v[k];
            for (int off = 16; off; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
            if (lane == 0 && x) atomicAdd(&b.census[8 + k], x);
        }
    }
}

template <int FLAGS, bool WIDE>
__global__ void __launch_bounds__(32 * kWarpsPerCta) apply_warp_kernel(Store s, Batch b) {
    const unsigned long long tw = tl_start(b.tl);
    pdl_wait();
    pdl_trigger();
    const unsigned long long t0 = tl_start(b.tl);
    tl_stop(b.tl, 8, tw);
    constexpr bool PER_MOVE = (FLAGS & kPerMove) != 0;
    constexpr bool HITS = (FLAGS & kHits) != 0;
    __shared__ int2 som[kWarpsPerCta][32];
    __shared__ int s_ids[kStageIds];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nslices = (s.Np + 31) >> 5;
    const bool staged = b.n <= kStageIds;
    if (b.evready && blockIdx.x == 0 && threadIdx.x < 4) b.evready[threadIdx.x] = 0;  // for the next update
    if (staged) {
        for (int t = threadIdx.x; t < b.n; t += blockDim.x) s_ids[t] = b.ids[t];
        __syncthreads();
    }
    int dgray = 0;
    // a full narrow-item queue left some verdicts uncomputed: apply nothing, so the
    // engine stays at its pre-update state and the host can grow the queue and replay
    const int full = b.ctr[6];
    // Work list: when fewer than half the cells are dirty, the dirty slices only, from
    // touch's work units (a cell's first chunk stands for the cell: {cell, 0, count,
    // mask base}); otherwise every slice, with its state loads issued before the cell
    // record's (one round trip less on the chain).  c4: -14 %; c5 would lose 2.5 %.
    // RGG_DEBUG_FLAGS 16384 forces the every-slice walk.
    const bool dirty_only = (s.dbg_flags & 16384) == 0 && 2 * b.ctr[0] < s.ncells;
    const int spc = s.cell >> 5;
    const int n_work = dirty_only ? min(b.ctr[10], b.units_cap) * spc : nslices;
    for (int wq = blockIdx.x * kWarpsPerCta + wi; wq < n_work; wq += gridDim.x * kWarpsPerCta) {
        int q = wq;
        int4 un = make_int4(0, 0, 0, 0);
        if (dirty_only) {
            un = b.units[wq / spc];
            if (un.y != 0) continue;  // warp-uniform: a later chunk of a listed cell
            q = un.x * spc + wq % spc;
        }
        const int c0 = q << 5;
        if (c0 >= s.Np) continue;
        const int cell = c0 / s.cell;
        const int c = c0 + lane, t = c - cell * s.cell;
        const bool valid = c < s.Np;
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
        int4 rec;
        if (dirty_only) {
            const int32_t* lst = un.z <= s.cap ? b.cell_list + static_cast<size_t>(cell) * s.cap : b.pool + b.cell_ovf[cell];
            const unsigned long long la = reinterpret_cast<unsigned long long>(lst);
            rec = make_int4(un.z, un.w, static_cast<int>(la & 0xffffffffu), static_cast<int>(la >> 32));
        } else {
            rec = b.crec[cell];
        }
        const int count = rec.x;
        if (full == 3) break;  // warp-uniform
        if (count == 0) continue;
        oc = cw & 0xffff;
        bc = cw >> 16;
        const int label0 = label;
        const uint32_t cnt0 = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
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
            // only the events that touch some component of the slice can change a
            // label or a counter: walk those, in list (= move) order
            for (uint32_t em = __reduce_or_sync(0xffffffffu, tm); em; em &= em - 1) {
                const int k = __ffs(em) - 1;
                const int before = label;
                const int2 om = som[wi][k];
                if ((tm >> k) & 1u) {
                    const int o = om.x;
                    const int wo = o >> 6;
                    const unsigned long long bit = 1ull << (o & 63);
                    unsigned long long ow, uw;
                    if (WIDE) {
                        ow = s.over[static_cast<size_t>(wo) * s.Np + c];
                        uw = s.under[static_cast<size_t>(wo) * s.Np + c];
                    } else {
                        ow = OW;
                        uw = UW;
                    }
                    const bool old_over = (ow & bit) != 0, old_under = (uw & bit) != 0;
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
                    const unsigned long long nw = n_over ? (ow | bit) : (ow & ~bit);
                    const unsigned long long nuw = n_under ? (uw | bit) : (uw & ~bit);
                    if (WIDE) {
                        if (nw != ow) s.over[static_cast<size_t>(wo) * s.Np + c] = nw;
                        if (nuw != uw) s.under[static_cast<size_t>(wo) * s.Np + c] = nuw;
                    } else {
                        OW = nw;
                        UW = nuw;
                    }
                    if (HITS && om.y == b.n - 1) hit_last = n_over;
                }
                if (PER_MOVE && __any_sync(0xffffffffu, label != before)) {
                    const bool ch = label != before;
                    const unsigned gg = __ballot_sync(0xffffffffu, ch && label == 0);
                    const unsigned r = __ballot_sync(0xffffffffu, ch && label == 1);
                    const unsigned y = __ballot_sync(0xffffffffu, ch && label == 2);
                    const unsigned f = __ballot_sync(0xffffffffu, ch && before == 2);
                    if (lane == 0 && (gg | r | y | f) && !(s.dbg_flags & 4)) {  // 4: ablation, no counters
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
        if (valid) {
            if (label != label0) {
                s.state[id] = static_cast<uint8_t>(label);
                s.state_c[c] = static_cast<uint8_t>(label);
                dgray += (label == 2) - (label0 == 2);
            }
            const uint32_t cw = static_cast<uint32_t>(oc) | (static_cast<uint32_t>(bc) << 16);
            if (cw != cnt0) s.cnt[c] = cw;
            if (!WIDE) {
                if (OW != OW0) s.over[c] = OW;
                if (UW != UW0) s.under[c] = UW;
            }
        }
        if (HITS) {
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
    if (full != 3 && !(s.dbg_flags & 8)) commit_grid(s, b);  // 8: ablation, no commit
    tl_stop(b.tl, 4, t0);
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

__global__ void __launch_bounds__(kCompactThreads) gray_write_kernel(const uint8_t* st, int N, const int32_t* tile_cnt,
                                                                     int ntiles, int32_t* out, int32_t* gray_n) {
    pdl_wait();
    pdl_trigger();
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
    const int cells_per = kBinThreads / 32;  // = kSuperCells
    static const bool no_small = std::getenv("RGG_NO_SMALL_BIN") != nullptr;
    if (b.n <= kBinSmallMax && !no_small)
        return launch_pdl(bin_small_kernel, dim3((s.ncells + kBinSmallWarps - 1) / kBinSmallWarps),
                          dim3(32 * kBinSmallWarps), st, s, b);
    return launch_pdl(bin_kernel, dim3((s.ncells + cells_per - 1) / cells_per), dim3(kBinThreads), st, s, b);
}

template <int F, bool W>
static cudaError_t apply_t(const Store& s, const Batch& b, cudaStream_t st) {
    apply_kernel<F, W><<<s.ncells, s.cell, 0, st>>>(s, b);
    return cudaGetLastError();
}

static int grid_warp(const Store& s) {
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, classify_warp_kernel<kPerMove, false>, 32 * kWarpsPerCta, 0);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        per_sm = per_sm < 1 ? 1 : per_sm;
    }
    const int slices = (s.Np + 31) / 32;
    const int need = (slices + kWarpsPerCta - 1) / kWarpsPerCta;
    return need < per_sm * sms ? (need < 1 ? 1 : need) : per_sm * sms;
}

template <int F, bool W>
static cudaError_t warp_t(const Store& s, const Batch& b, int grid, cudaStream_t st) {
    classify_warp_kernel<F, W><<<grid, 32 * kWarpsPerCta, 0, st>>>(s, b);
    return cudaGetLastError();
}

static int pipeline() {
    static const int p = [] {
        const char* e = std::getenv("RGG_PIPELINE");
        return e ? std::atoi(e) : 6;
    }();
    return p;
}

bool split_pipeline() { return pipeline() == 6; }

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

static int grid_slices(const Store& s, const void* fn) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kWarpsPerCta, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    per_sm = per_sm < 1 ? 1 : per_sm;
    const int need = ((s.Np + 31) / 32 + kWarpsPerCta - 1) / kWarpsPerCta;
    return need < per_sm * sms ? (need < 1 ? 1 : need) : per_sm * sms;
}

// lanes per under item (RGG_UNDER_LANES = 1, 2 or 4)
static int under_lanes() {
    static const int g = [] {
        const char* e = std::getenv("RGG_UNDER_LANES");
        const int v = e ? std::atoi(e) : 1;
        return v == 2 || v == 4 ? v : 1;
    }();
    return g;
}

static cudaError_t launch_narrow(const Store& s, const Batch& b, int grid, cudaStream_t st, bool pdl) {
    static const int forced = std::getenv("RGG_NARROW_CTAS") ? std::atoi(std::getenv("RGG_NARROW_CTAS")) : 0;
    if (forced > 0) grid = forced;
    switch (under_lanes()) {
        case 2:
            return pdl ? launch_pdl(narrow_kernel<false, 2>, dim3(grid), dim3(128), st, s, b)
                       : (narrow_kernel<false, 2><<<grid, 128, 0, st>>>(s, b), cudaGetLastError());
        case 4:
            return pdl ? launch_pdl(narrow_kernel<false, 4>, dim3(grid), dim3(128), st, s, b)
                       : (narrow_kernel<false, 4><<<grid, 128, 0, st>>>(s, b), cudaGetLastError());
        default:
            return pdl ? launch_pdl(narrow_kernel<false, 1>, dim3(grid), dim3(128), st, s, b)
                       : (narrow_kernel<false, 1><<<grid, 128, 0, st>>>(s, b), cudaGetLastError());
    }
}

cudaError_t launch_classify(const Store& s, const Batch& b, int flags, int grid, cudaStream_t st) {
    if (s.ncells == 0) {  // no components: only the obstacles' operands move on
        if (b.n == 0 || (flags & kCensus)) return cudaSuccess;
        commit_kernel<<<(b.n + 7) / 8, 128, 0, st>>>(s, b);
        return cudaGetLastError();
    }
    if (pipeline() == 6) {
        static int g_touch = 0, g_touch_c = 0, g_apply = 0;
        if (!g_touch) {
            g_touch = grid_slices(s, reinterpret_cast<const void*>(touch_warp_kernel<false>));
            g_touch_c = grid_slices(s, reinterpret_cast<const void*>(touch_warp_kernel<true>));
            g_apply = grid_slices(s, reinterpret_cast<const void*>(apply_warp_kernel<kPerMove, false>));
        }
        if (flags & kCensus) {
            touch_warp_kernel<true><<<g_touch_c, 32 * kWarpsPerCta, 0, st>>>(s, b);
            narrow_kernel<true, 1><<<grid, 128, 0, st>>>(s, b);
            return cudaGetLastError();
        }
        cudaError_t e = launch_pdl(touch_warp_kernel<false>, dim3(g_touch), dim3(32 * kWarpsPerCta), st, s, b);
        if (e == cudaSuccess) e = launch_narrow(s, b, grid, st, true);
        if (e == cudaSuccess && (s.dbg_flags & 16)) e = launch_narrow(s, b, grid, st, true);  // 16: run twice (warm)
        if (e != cudaSuccess) return e;
        const bool wide = s.W > 1;
        const int ga = g_apply;
        switch (flags & (kPerMove | kHits)) {
            case 0:
                return wide ? apply6_t<0, true>(s, b, ga, st) : apply6_t<0, false>(s, b, ga, st);
            case kPerMove:
                return wide ? apply6_t<kPerMove, true>(s, b, ga, st) : apply6_t<kPerMove, false>(s, b, ga, st);
            case kHits:
                return wide ? apply6_t<kHits, true>(s, b, ga, st) : apply6_t<kHits, false>(s, b, ga, st);
            default:
                return wide ? apply6_t<kPerMove | kHits, true>(s, b, ga, st)
                            : apply6_t<kPerMove | kHits, false>(s, b, ga, st);
        }
    }
    if (pipeline() == 4) {
        const int g = grid_warp(s);
        const bool wide = s.W > 1;
        if (flags & kCensus) return wide ? warp_t<kCensus, true>(s, b, g, st) : warp_t<kCensus, false>(s, b, g, st);
        switch (flags & (kPerMove | kHits)) {
            case 0:
                return wide ? warp_t<0, true>(s, b, g, st) : warp_t<0, false>(s, b, g, st);
            case kPerMove:
                return wide ? warp_t<kPerMove, true>(s, b, g, st) : warp_t<kPerMove, false>(s, b, g, st);
            case kHits:
                return wide ? warp_t<kHits, true>(s, b, g, st) : warp_t<kHits, false>(s, b, g, st);
            default:
                return wide ? warp_t<kPerMove | kHits, true>(s, b, g, st) : warp_t<kPerMove | kHits, false>(s, b, g, st);
        }
    }
    if (flags & kCensus) {
        narrow_kernel<true, 1><<<grid, 128, 0, st>>>(s, b);
        return cudaGetLastError();
    }
    touch_kernel<<<s.ncells, s.cell, 0, st>>>(s, b);
    launch_narrow(s, b, grid, st, false);
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, narrow_kernel<false, 1>, 128, 0);
    return n < 1 ? 1 : n;
}

cudaError_t launch_compact(const Store& s, int32_t* out_ids, int32_t* tile_cnt, int32_t* gray_n, cudaStream_t st) {
    const int ntiles = (s.N + kTile - 1) / kTile;
    if (ntiles == 0) return cudaMemsetAsync(gray_n, 0, sizeof(int32_t), st);
    cudaError_t e = launch_pdl(gray_count_kernel, dim3(ntiles), dim3(kCompactThreads), st,
                               static_cast<const uint8_t*>(s.state), s.N, tile_cnt);
    if (e != cudaSuccess) return e;
    return launch_pdl(gray_write_kernel, dim3(ntiles), dim3(kCompactThreads), st, static_cast<const uint8_t*>(s.state),
                      s.N, static_cast<const int32_t*>(tile_cnt), ntiles, out_ids, gray_n);
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

cudaError_t launch_fp64_peak(double* sink, int iters, int grid, int block, cudaStream_t st) {
    fp64_peak_kernel<<<grid, block, 0, st>>>(sink, iters);
    return cudaGetLastError();
}

}  // namespace rggk
