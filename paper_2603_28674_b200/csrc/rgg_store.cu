// rgg_store.cu — the engine's resident store built on the GPU.
//
// rgg_gpu_create receives the serialized layout (BatchLayout::serialize,
// proj/src/batch_layout.cpp:21-146, as the CSR view of include/rgg_gpu.h).  The
// engine re-orders it into cell-sorted SoA.  Here that runs on the
// device after one upload of the raw arrays:
//   1. centre bounds (block min/max, order-independent), 63-bit Morton keys of
//      the AABB centres — the same fp64 operations as the former host path;
//   2. stable radix sort of (key, id) (CUB), shard selection of interleaved cells;
//   3. gathers: AABB planes, SatBoxes (22-double records), Box32 filter operands,
//      per-row segment counts -> exclusive scan -> CSR rows, segment records
//      (+ the row's spline radius), id -> rank map, cell boxes;
//   4. the uniform grid over the cell boxes that the binning queries (build_cell_grid).
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "rgg_device.cuh"
#include "rgg_kernels.cuh"

namespace rggk {
namespace {

// monotone uint64 image of a double (total order of non-NaN values)
__device__ __forceinline__ unsigned long long ord_of(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double dbl_of(unsigned long long o) {
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double d;
    memcpy(&d, &b, 8);
    return d;
#endif
}

__device__ __forceinline__ double centre_of(const double* a, int k) {
    double x = 0.5 * (a[k] + a[3 + k]);
    return x == x ? x : 0.0;  // NaN guard (as the host path)
}

// bounds[0..2] = min (ordered), bounds[3..5] = max
__global__ void centre_bounds_kernel(const double* aabb, int n, unsigned long long* bounds) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
        for (int k = 0; k < 3; ++k) {
            const unsigned long long o = ord_of(centre_of(aabb + 6 * static_cast<size_t>(c), k));
            lo[k] = min(lo[k], o);
            hi[k] = max(hi[k], o);
        }
    for (int k = 0; k < 3; ++k)
        for (int off = 16; off; off >>= 1) {
            lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], off));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], off));
        }
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) {
            atomicMin(bounds + k, lo[k]);
            atomicMax(bounds + 3 + k, hi[k]);
        }
}

__device__ __forceinline__ unsigned long long spread3_d(unsigned long long x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

__global__ void morton_kernel(const double* aabb, int n, const unsigned long long* bounds, unsigned long long* key,
                              int32_t* val) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    unsigned long long code = 0;
    for (int k = 0; k < 3; ++k) {
        const double lo = dbl_of(bounds[k]), hi = dbl_of(bounds[3 + k]);
        const double span = hi - lo;
        const double t = span > 0 ? (centre_of(aabb + 6 * static_cast<size_t>(c), k) - lo) / span : 0.0;
        const unsigned long long q = static_cast<unsigned long long>(fmin(fmax(t, 0.0), 1.0) * 2097151.0);
        code |= spread3_d(q) << k;
    }
    key[c] = code;
    val[c] = c;
}

// owned[i] = order[global position of the i-th component of this shard's cells]
__global__ void select_kernel(const int32_t* order, int np, int cell, int shards, int rank, int32_t* owned,
                              int32_t* rankmap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const long long g = rank + static_cast<long long>(i / cell) * shards;
    const int c = order[g * cell + i % cell];
    owned[i] = c;
    rankmap[c] = i;
}

__global__ void gather_kernel(const int32_t* owned, int np, int B, int BS, const double* aabb, const double* sat21,
                              const int32_t* row_off, double2* aabb_out, double* sat_out, rggd::Box32* sat32,
                              int32_t* row_len) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const int c = owned[i];
    const double* a = aabb + 6 * static_cast<size_t>(c);
    aabb_out[i] = make_double2(a[0], a[1]);
    aabb_out[np + i] = make_double2(a[2], a[3]);
    aabb_out[2 * static_cast<size_t>(np) + i] = make_double2(a[4], a[5]);
    for (int b = 0; b < B; ++b) {
        const double* s = sat21 + (static_cast<size_t>(c) * B + b) * 21;
        double* d = sat_out + (static_cast<size_t>(i) * B + b) * 22;
        rggd::Box32 x{};
        for (int k = 0; k < 21; ++k) d[k] = s[k];
        d[21] = 0.0;
        for (int k = 0; k < 3; ++k) x.c[k] = s[k];
        rggd::box32_terms(s, x);
        sat32[static_cast<size_t>(i) * B + b] = x;
    }
    for (int r = 0; r < BS; ++r) {
        const size_t src = static_cast<size_t>(c) * BS + r;
        row_len[static_cast<size_t>(i) * BS + r] = row_off[src + 1] - row_off[src];
    }
}

// one thread per row of the sorted order: its real segments + the slot's spline radius
__global__ void segs_kernel(const int32_t* owned, long long nrows, int BS, const int32_t* row_off_src,
                            const int32_t* row_new, const double* segs7, const double* spline, double* seg8,
                            float4* seg32) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nrows) return;
    const int i = static_cast<int>(t / BS), r = static_cast<int>(t % BS);
    const size_t src = static_cast<size_t>(owned[i]) * BS + r;
    const int k0 = row_off_src[src], k1 = row_off_src[src + 1];
    double* d = seg8 + 8 * static_cast<size_t>(row_new[t]);
    float4* f = seg32 + 2 * static_cast<size_t>(row_new[t]);
    for (int k = k0; k < k1; ++k, d += 8, f += 2) {
        const double* s = segs7 + 7 * static_cast<size_t>(k);
        for (int j = 0; j < 7; ++j) d[j] = s[j];
        d[7] = spline[r];
        f[0] = make_float4(__double2float_rn(s[0]), __double2float_rn(s[1]), __double2float_rn(s[2]),
                           __double2float_rn(s[3]));
        f[1] = make_float4(__double2float_rn(s[4]), __double2float_rn(s[5]), __double2float_rn(s[6]),
                           __double2float_rn(spline[r]));
    }
}

__global__ void cell_box_kernel(const double2* aabb, int np, int cell, int ncells, double* cell_aabb) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ncells) return;
    double box[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
    for (int i = g * cell; i < min(np, (g + 1) * cell); ++i) {
        const double2 a0 = aabb[i], a1 = aabb[np + i], a2 = aabb[2 * static_cast<size_t>(np) + i];
        const double a[6] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y};
        for (int k = 0; k < 3; ++k) {
            box[k] = fmin(box[k], a[k]);
            box[3 + k] = fmax(box[3 + k], a[3 + k]);
        }
    }
    for (int k = 0; k < 6; ++k) cell_aabb[6 * static_cast<size_t>(g) + k] = box[k];
}


// scratch allocations released on every exit of build_store
struct Scratch {
    void* p[16] = {};
    int n = 0;
    ~Scratch() {
        for (int i = 0; i < n; ++i) cudaFree(p[i]);
    }
    template <class T>
    cudaError_t alloc(T** out, size_t count) {
        const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(out), (count ? count : 1) * sizeof(T));
        if (e == cudaSuccess) p[n++] = *out;
        return e;
    }
};

#define SCK(x)                                   \
    do {                                         \
        const cudaError_t e_ = (x);              \
        if (e_ != cudaSuccess) return e_;        \
    } while (0)

}  // namespace

cudaError_t build_store(const StoreIn& in, StoreOut& out, cudaStream_t st) {
    Scratch scratch;
    const int N = in.N, B = in.B, BS = in.B * in.S, np = in.np, cell = in.cell;
    const long long nrows = static_cast<long long>(np) * BS;
    const int ncells = (np + cell - 1) / cell;
    // 1. raw inputs (host arrays uploaded here, or device arrays the caller prepared:
    // rgg_gpu_create_from_components runs sat_prep / seg_prep on the device)
    double *aabb = nullptr, *sat21 = nullptr, *segs7 = nullptr;
    int32_t* row_off = nullptr;
    SCK(cudaStreamSynchronize(st));
    if (in.device) {
        aabb = const_cast<double*>(in.comp_aabb);
        sat21 = const_cast<double*>(in.edge_sat);
        row_off = const_cast<int32_t*>(in.row_off_dev);
        segs7 = const_cast<double*>(in.segs);
    } else {
        SCK(scratch.alloc(&aabb, static_cast<size_t>(N) * 6));
        SCK(scratch.alloc(&sat21, static_cast<size_t>(N) * B * 21));
        SCK(scratch.alloc(&row_off, static_cast<size_t>(N) * BS + 1));
        SCK(scratch.alloc(&segs7, static_cast<size_t>(in.T) * 7));
        // pageable sources, copied in stream order: a synchronous cudaMemcpy runs on the
        // legacy stream and may return before its DMA lands, unordered with st's kernels
        SCK(cudaMemcpyAsync(aabb, in.comp_aabb, static_cast<size_t>(N) * 6 * 8, cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(sat21, in.edge_sat, static_cast<size_t>(N) * B * 21 * 8, cudaMemcpyHostToDevice, st));
        SCK(cudaMemcpyAsync(row_off, in.row_off, (static_cast<size_t>(N) * BS + 1) * 4, cudaMemcpyHostToDevice, st));
        if (in.T) SCK(cudaMemcpyAsync(segs7, in.segs, static_cast<size_t>(in.T) * 7 * 8, cudaMemcpyHostToDevice, st));
    }
    SCK(cudaMemcpyAsync(out.spline, in.spline, static_cast<size_t>(BS) * 8, cudaMemcpyHostToDevice, st));
    // 2. Morton order
    unsigned long long *bounds = nullptr, *key = nullptr, *key2 = nullptr;
    int32_t *val = nullptr, *order = nullptr;
    SCK(scratch.alloc(&bounds, 6));
    SCK(scratch.alloc(&key, N));
    SCK(scratch.alloc(&key2, N));
    SCK(scratch.alloc(&val, N));
    SCK(scratch.alloc(&order, N));
    const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    SCK(cudaMemcpyAsync(bounds, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int T256 = 256;
    if (N > 0) {
        centre_bounds_kernel<<<std::min(1184, (N + T256 - 1) / T256), T256, 0, st>>>(aabb, N, bounds);
        morton_kernel<<<(N + T256 - 1) / T256, T256, 0, st>>>(aabb, N, bounds, key, val);
    }
    size_t tmp_bytes = 0, scan_bytes = 0;
    SCK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key2, val, order, N, 0, 63, st));
    int32_t *row_len = nullptr;
    SCK(scratch.alloc(&row_len, static_cast<size_t>(nrows) + 1));
    SCK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, row_len, out.row, nrows + 1, st));
    char* tmp = nullptr;
    SCK(scratch.alloc(&tmp, std::max(tmp_bytes, scan_bytes)));
    if (N > 0) SCK(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, val, order, N, 0, 63, st));
    // 3. shard selection, id -> rank, gathers
    SCK(cudaMemsetAsync(out.rank, 0xFF, static_cast<size_t>(N) * 4, st));
    if (np > 0) {
        select_kernel<<<(np + T256 - 1) / T256, T256, 0, st>>>(order, np, cell, in.shards, in.shard_rank, out.orig,
                                                              out.rank);
        gather_kernel<<<(np + 127) / 128, 128, 0, st>>>(out.orig, np, B, BS, aabb, sat21, row_off, out.aabb, out.sat,
                                                       out.sat32, row_len);
    }
    SCK(cudaMemsetAsync(row_len + nrows, 0, 4, st));
    SCK(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, row_len, out.row, nrows + 1, st));
    SCK(cudaMemcpyAsync(&out.total_segs, out.row + nrows, 4, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    SCK(cudaMalloc(reinterpret_cast<void**>(&out.seg), sizeof(double) * std::max<size_t>(1, static_cast<size_t>(out.total_segs) * 8)));
    SCK(cudaMalloc(reinterpret_cast<void**>(&out.seg32), sizeof(float4) * std::max<size_t>(1, static_cast<size_t>(out.total_segs) * 2)));
    if (nrows > 0)
        segs_kernel<<<static_cast<unsigned>((nrows + T256 - 1) / T256), T256, 0, st>>>(
            out.orig, nrows, BS, row_off, out.row, segs7, out.spline, out.seg, out.seg32);
    if (ncells > 0) cell_box_kernel<<<(ncells + 127) / 128, 128, 0, st>>>(out.aabb, np, cell, ncells, out.cell_aabb);
    const int nslices = (np + 31) / 32;
    if (nslices > 0) cell_box_kernel<<<(nslices + 127) / 128, 128, 0, st>>>(out.aabb, np, 32, nslices, out.slice_aabb);
    SCK(cudaGetLastError());
    SCK(cudaStreamSynchronize(st));
    return cudaSuccess;
}

// The serialize step on the device (batch_layout.cpp:55-62, 80-105, 132-146): per
// (component, body) sat_prep of the OBB corners (kernels_scalar.cpp:7-30) and the
// component AABB as the union of the bodies' corner boxes (aabb_of_obb,
// geometry.cpp:205-213); per real segment seg_prep (kernels_scalar.cpp:71-79).
__global__ void prep_boxes_kernel(const double* corners, int N, int B, double* sat21, double* aabb) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= N) return;
    double box[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int b = 0; b < B; ++b) {
        const double* p = corners + (static_cast<size_t>(c) * B + b) * 24;
        double cs[24];
        for (int k = 0; k < 24; ++k) cs[k] = p[k];
        rggd::sat_prep(cs, sat21 + (static_cast<size_t>(c) * B + b) * 21);
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < 3; ++k) {
                box[k] = fmin(box[k], cs[3 * i + k]);
                box[3 + k] = fmax(box[3 + k], cs[3 * i + k]);
            }
    }
    for (int k = 0; k < 6; ++k) aabb[6 * static_cast<size_t>(c) + k] = box[k];
}

__global__ void prep_segs_kernel(const double* pts, int T, double* segs7) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    const double* p = pts + 6 * static_cast<size_t>(t);
    double* q = segs7 + 7 * static_cast<size_t>(t);
    double d[3];
    for (int j = 0; j < 3; ++j) {
        q[j] = p[j];
        d[j] = __dsub_rn(p[3 + j], p[j]);
        q[3 + j] = d[j];
    }
    q[6] = __dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2]));
}

cudaError_t prep_components(const double* corners, int N, int B, const double* pts, int T, double* sat21,
                            double* aabb, double* segs7, cudaStream_t st) {
    if (N > 0) prep_boxes_kernel<<<(N + 127) / 128, 128, 0, st>>>(corners, N, B, sat21, aabb);
    if (T > 0) prep_segs_kernel<<<(T + 255) / 256, 256, 0, st>>>(pts, T, segs7);
    return cudaGetLastError();
}

// A uniform grid over the cell boxes (host side: a few thousand cells).  Bins are
// about half the median cell extent per axis (one bin along an axis the cells
// span almost entirely, e.g. z of an SE(2) roadmap), at most 128 per axis and 2^21
// in all; each cell is listed in every bin its closed box overlaps.  The binning's
// monotone index map floor((p - org) * inv), clamped, sends every point of a cell
// box and every point of an event box to bins inside the ranges both register, so
// two overlapping boxes always share a bin.
cudaError_t build_cell_grid(const double* d_cell_aabb, int ncells, CellGrid& g, cudaStream_t st) {
    std::vector<double> box(static_cast<size_t>(ncells) * 6);
    if (ncells) SCK(cudaMemcpyAsync(box.data(), d_cell_aabb, box.size() * 8, cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    std::vector<double> ext[3];
    for (int c = 0; c < ncells; ++c)
        for (int k = 0; k < 3; ++k) {
            if (!(box[6 * c] <= box[6 * c + 3])) continue;  // empty cell box
            lo[k] = std::min(lo[k], box[6 * c + k]);
            hi[k] = std::max(hi[k], box[6 * c + 3 + k]);
            ext[k].push_back(box[6 * c + 3 + k] - box[6 * c + k]);
        }
    long long total = 1;
    for (int k = 0; k < 3; ++k) {
        double med = 0.0;
        if (!ext[k].empty()) {
            std::nth_element(ext[k].begin(), ext[k].begin() + ext[k].size() / 2, ext[k].end());
            med = ext[k][ext[k].size() / 2];
        }
        const double span = ext[k].empty() ? 0.0 : hi[k] - lo[k];
        int d = 1;
        if (span > 0 && med < 0.75 * span)
            d = static_cast<int>(std::min(128.0, std::max(1.0, std::ceil(span / std::max(0.5 * med, span / 128.0)))));
        g.dim[k] = d;
        g.org[k] = ext[k].empty() ? 0.0 : lo[k];
        g.inv[k] = span > 0 ? d / span : 0.0;
        total *= d;
    }
    while (total > (1 << 21)) {  // coarsen the finest axis
        int k = 0;
        for (int j = 1; j < 3; ++j) k = g.dim[j] > g.dim[k] ? j : k;
        total /= g.dim[k];
        g.inv[k] *= static_cast<double>((g.dim[k] + 1) / 2) / g.dim[k];
        g.dim[k] = (g.dim[k] + 1) / 2;
        total *= g.dim[k];
    }
    const auto bin = [&](double v, int k) {
        const double f = std::floor((v - g.org[k]) * g.inv[k]);
        return f < 0 ? 0 : (f >= g.dim[k] ? g.dim[k] - 1 : static_cast<int>(f));
    };
    std::vector<int32_t> cnt(static_cast<size_t>(total) + 1, 0);
    std::vector<int2> lst;
    for (int pass = 0; pass < 2; ++pass) {
        for (int c = 0; c < ncells; ++c) {
            const double* b = &box[6 * static_cast<size_t>(c)];
            if (!(b[0] <= b[3])) continue;  // empty cell box
            int l[3], h[3];
            for (int k = 0; k < 3; ++k) l[k] = bin(b[k], k), h[k] = bin(b[3 + k], k);
            const int lo_packed = l[0] | (l[1] << 10) | (l[2] << 20);
            for (int z = l[2]; z <= h[2]; ++z)
                for (int y = l[1]; y <= h[1]; ++y)
                    for (int x = l[0]; x <= h[0]; ++x) {
                        const size_t q = (static_cast<size_t>(z) * g.dim[1] + y) * g.dim[0] + x;
                        if (pass == 0) ++cnt[q + 1];
                        else lst[cnt[q]++] = int2{c, lo_packed};
                    }
        }
        if (pass == 0) {
            for (size_t q = 0; q < static_cast<size_t>(total); ++q) cnt[q + 1] += cnt[q];
            lst.resize(std::max<size_t>(1, static_cast<size_t>(cnt[total])), int2{0, 0});
        } else {
            for (size_t q = static_cast<size_t>(total); q > 0; --q) cnt[q] = cnt[q - 1];
            cnt[0] = 0;
        }
    }
    SCK(cudaMalloc(reinterpret_cast<void**>(&g.off), cnt.size() * 4));
    SCK(cudaMalloc(reinterpret_cast<void**>(&g.cells), lst.size() * sizeof(int2)));
    SCK(cudaMemcpyAsync(g.off, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice, st));
    SCK(cudaMemcpyAsync(g.cells, lst.data(), lst.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    SCK(cudaStreamSynchronize(st));
    g.entries = cnt[total];
    return cudaSuccess;
}

}  // namespace rggk
