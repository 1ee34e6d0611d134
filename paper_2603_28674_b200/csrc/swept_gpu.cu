// swept_gpu.cu — the producer's outer approximation on the GPU.
//
// obb_from_points (proj/src/geometry.cpp:134-195) fits each component's swept
// volume box: PCA frame of the body corners at every discretized configuration
// (Jacobi), then 3 x 10 rotated candidate frames, keeping the smallest-volume
// one.  It is ~85 % of the host producer's time.  Here one thread fits one
// component, regenerating the corners from the forward-kinematics poses on
// every pass instead of storing the cloud.  Compiled with -fmad=false: every
// expression is the host producer's (producer.cpp, itself the reference's
// association), so the boxes are bit-identical; the cosines / sines of the ten
// candidate angles come from the host's libm.
#include <cuda_runtime.h>

#include "swept_gpu.h"

#include <chrono>
#include <cstdint>
#include <vector>
#include <cstdio>
#include <cstdlib>

namespace {

struct V3 {
    double x, y, z;
};
__device__ inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ inline double dotv(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ inline V3 crossv(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

// Transform::rotate / apply of a pose r[9], t[3] (vec3.hpp:72-84)
__device__ inline V3 rot(const double* r, V3 p) {
    return {r[0] * p.x + r[1] * p.y + r[2] * p.z, r[3] * p.x + r[4] * p.y + r[5] * p.z,
            r[6] * p.x + r[7] * p.y + r[8] * p.z};
}

// corner i of the body box at a pose (producer.cpp build_comp + corners_of)
__device__ inline V3 corner(const double* T, V3 he, int i) {
    const V3 c = {T[0] * 0.0 + T[1] * 0.0 + T[2] * 0.0 + T[9], T[3] * 0.0 + T[4] * 0.0 + T[5] * 0.0 + T[10],
                  T[6] * 0.0 + T[7] * 0.0 + T[8] * 0.0 + T[11]};
    const V3 e0 = rot(T, {1, 0, 0}) * he.x, e1 = rot(T, {0, 1, 0}) * he.y, e2 = rot(T, {0, 0, 1}) * he.z;
    V3 p = (i & 1) ? c + e0 : c - e0;
    p = (i & 2) ? p + e1 : p - e1;
    return (i & 4) ? p + e2 : p - e2;
}

__device__ inline double min_ref(double a, double b) { return b < a ? b : a; }
__device__ inline double max_ref(double a, double b) { return a < b ? b : a; }

__device__ double volume(const double* poses, int n, V3 he, const V3* ax, double* lo, double* hi) {
    for (int k = 0; k < 3; ++k) lo[k] = __longlong_as_double(0x7ff0000000000000ll), hi[k] = -lo[k];
    for (int q = 0; q < n; ++q)
        for (int i = 0; i < 8; ++i) {
            const V3 p = corner(poses + 12 * static_cast<size_t>(q), he, i);
            for (int k = 0; k < 3; ++k) {
                const double t = dotv(p, ax[k]);
                lo[k] = min_ref(lo[k], t);
                hi[k] = max_ref(hi[k], t);
            }
        }
    return (hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
}

__device__ void jacobi3(double m[3][3], double vals[3], V3 vecs[3]) {
    double v[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int sweep = 0; sweep < 64; ++sweep) {
        const double off = fabs(m[0][1]) + fabs(m[0][2]) + fabs(m[1][2]);
        if (off == 0.0) break;
        for (int p = 0; p < 2; ++p) {
            for (int q = p + 1; q < 3; ++q) {
                if (m[p][q] == 0.0) continue;
                const double theta = (m[q][q] - m[p][p]) / (2.0 * m[p][q]);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double s = t * c;
                for (int k = 0; k < 3; ++k) {
                    const double a = m[k][p], b = m[k][q];
                    m[k][p] = c * a - s * b;
                    m[k][q] = s * a + c * b;
                }
                for (int k = 0; k < 3; ++k) {
                    const double a = m[p][k], b = m[q][k];
                    m[p][k] = c * a - s * b;
                    m[q][k] = s * a + c * b;
                }
                for (int k = 0; k < 3; ++k) {
                    const double a = v[k][p], b = v[k][q];
                    v[k][p] = c * a - s * b;
                    v[k][q] = s * a + c * b;
                }
            }
        }
    }
    for (int i = 0; i < 3; ++i) {
        vals[i] = m[i][i];
        vecs[i] = {v[0][i], v[1][i], v[2][i]};
    }
}

// fit_box (producer.cpp) of the corners of n poses; out = centre, axes[3], half extents
// one thread per fit unit c (a (component, body) pair; body c % nb, half extents he3[body])
__global__ void fit_kernel(const double* poses, const int64_t* off, int ncomp, const double* he3, int nb,
                           const double* cs, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncomp) return;
    const int body = c % nb;
    const V3 he{he3[3 * body], he3[3 * body + 1], he3[3 * body + 2]};
    const double* P = poses + 12 * static_cast<size_t>(off[c]);
    const int n = static_cast<int>(off[c + 1] - off[c]);
    const double npts = static_cast<double>(8 * n);
    V3 mean{0, 0, 0};
    for (int q = 0; q < n; ++q)
        for (int i = 0; i < 8; ++i) mean = mean + corner(P + 12 * q, he, i);
    mean = mean * (1.0 / npts);
    double cov[3][3] = {};
    for (int q = 0; q < n; ++q)
        for (int i = 0; i < 8; ++i) {
            const V3 d = corner(P + 12 * q, he, i) - mean;
            const double dc[3] = {d.x, d.y, d.z};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) cov[a][b] += dc[a] * dc[b];
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) cov[a][b] /= npts;
    double vals[3];
    V3 axes[3];
    jacobi3(cov, vals, axes);
    int ord[3] = {0, 1, 2};
    for (int i = 1; i < 3; ++i)
        for (int j = i; j > 0 && vals[ord[j]] > vals[ord[j - 1]]; --j) {
            const int t = ord[j];
            ord[j] = ord[j - 1];
            ord[j - 1] = t;
        }
    V3 best[3] = {axes[ord[0]], axes[ord[1]], axes[ord[2]]};
    best[2] = crossv(best[0], best[1]);
    double lo[3], hi[3];
    double best_vol = volume(P, n, he, best, lo, hi);
    for (int k = 0; k < 3; ++k) {
        const V3 pivot = best[k];
        V3 win[3] = {best[0], best[1], best[2]};
        for (int step = -5; step <= 5; ++step) {
            if (step == 0) continue;
            // Transform::rotation_axis_angle (geometry.cpp:13-29) with the host's cos / sin
            const double len = sqrt(dotv(pivot, pivot));
            const double kx = pivot.x / len, ky = pivot.y / len, kz = pivot.z / len;
            const double co = cs[2 * (step + 5)], si = cs[2 * (step + 5) + 1], v = 1.0 - co;
            const double r[9] = {kx * kx * v + co, kx * ky * v - kz * si, kx * kz * v + ky * si,
                                 ky * kx * v + kz * si, ky * ky * v + co, ky * kz * v - kx * si,
                                 kz * kx * v - ky * si, kz * ky * v + kx * si, kz * kz * v + co};
            V3 cand[3];
            for (int j = 0; j < 3; ++j) cand[j] = rot(r, best[j]);
            const double vol = volume(P, n, he, cand, lo, hi);
            if (vol < best_vol) {
                best_vol = vol;
                for (int j = 0; j < 3; ++j) win[j] = cand[j];
            }
        }
        for (int j = 0; j < 3; ++j) best[j] = win[j];
    }
    volume(P, n, he, best, lo, hi);
    const V3 ctr = best[0] * ((lo[0] + hi[0]) * 0.5) + best[1] * ((lo[1] + hi[1]) * 0.5) + best[2] * ((lo[2] + hi[2]) * 0.5);
    double* o = out + 15 * static_cast<size_t>(c);
    o[0] = ctr.x, o[1] = ctr.y, o[2] = ctr.z;
    for (int k = 0; k < 3; ++k) o[3 + 3 * k] = best[k].x, o[4 + 3 * k] = best[k].y, o[5 + 3 * k] = best[k].z;
    o[12] = (hi[0] - lo[0]) * 0.5, o[13] = (hi[1] - lo[1]) * 0.5, o[14] = (hi[2] - lo[2]) * 0.5;
}

// ---- inner approximation (swept.cpp:188-228: build_inner_approx + simplify :79-92
// + cap_segments :125-162), one thread per (component, sphere), as producer.cpp

__device__ inline double point_seg_dist(V3 a, V3 b, V3 c) {
    const double s3 = b.x - a.x, s4 = b.y - a.y, s5 = b.z - a.z;
    const double s6 = (s3 * s3 + s4 * s4) + s5 * s5;
    const double px = c.x - a.x, py = c.y - a.y, pz = c.z - a.z;
    double t = 0.0;
    if (s6 > 0.0) {
        t = ((px * s3 + py * s4) + pz * s5) / s6;
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double qx = px - t * s3, qy = py - t * s4, qz = pz - t * s5;
    return sqrt((qx * qx + qy * qy) + qz * qz);
}

__device__ inline bool covers(const V3* pts, int j, int p, double radius) {
    for (int m = j + 1; m < p; ++m)
        if (!(point_seg_dist(pts[j], pts[p], pts[m]) < radius)) return false;
    return true;
}

struct InnerDev {
    int nsph, K;
    const double *centre, *radius, *step, *tol;
};

// COUNT: nspl / npts_total per (component, sphere); else write the spline sizes and points
template <bool COUNT>
__global__ void inner_kernel(const double* poses, const int64_t* off, int ncomp, InnerDev sp, V3* raw_scr,
                             int32_t* kept_scr, int32_t* nspl, int32_t* npts_total, const int64_t* spl_off,
                             const int64_t* pt_off, int32_t* spl_npts, double* pts) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= static_cast<long long>(ncomp) * sp.nsph) return;
    const int c = static_cast<int>(t / sp.nsph), si = static_cast<int>(t % sp.nsph);
    const int n = static_cast<int>(off[c + 1] - off[c]);
    int ns = 0, np = 0;
    const double rad = sp.radius[si];
    if (rad > 0.0) {
        V3* raw = raw_scr + off[c] * sp.nsph + static_cast<long long>(si) * n;
        int32_t* kept = kept_scr + off[c] * sp.nsph + static_cast<long long>(si) * n;
        const V3 sc{sp.centre[3 * si], sp.centre[3 * si + 1], sp.centre[3 * si + 2]};
        int nr = 0;
        bool step_ok = true;
        for (int q = 0; q < n; ++q) {
            const double* T = poses + 12 * static_cast<size_t>(off[c] + q);
            const V3 p{T[0] * sc.x + T[1] * sc.y + T[2] * sc.z + T[9], T[3] * sc.x + T[4] * sc.y + T[5] * sc.z + T[10],
                       T[6] * sc.x + T[7] * sc.y + T[8] * sc.z + T[11]};
            if (nr) {
                const V3 d = p - raw[nr - 1];
                if (sqrt(dotv(d, d)) > sp.step[si]) step_ok = false;
            }
            if (!nr || !(p.x == raw[nr - 1].x && p.y == raw[nr - 1].y && p.z == raw[nr - 1].z)) raw[nr++] = p;
        }
        if (step_ok) {
            const double tol = sp.tol[si];
            // simplify
            int nk = 0, j = 0;
            kept[nk++] = 0;
            while (j < nr - 1) {
                int p = j + 1;
                while (p + 1 <= nr - 1 && covers(raw, j, p + 1, tol)) ++p;
                kept[nk++] = p;
                j = p;
            }
            // cap_split
            const int q = nk - 1, K = sp.K;
            const auto emit = [&](int cnt, auto&& idx) {  // one spline of cnt points raw[idx(0..cnt)]
                if (!COUNT) {
                    spl_npts[spl_off[t] + ns] = cnt;
                    for (int k = 0; k < cnt; ++k) {
                        const V3 v = raw[idx(k)];
                        double* o = pts + 3 * (pt_off[t] + np + k);
                        o[0] = v.x, o[1] = v.y, o[2] = v.z;
                    }
                }
                ++ns;
                np += cnt;
            };
            if (q <= K) {
                emit(nk, [&](int k) { return kept[k]; });
            } else {
                bool ok = true;
                for (int i = 0; ok && i < K; ++i) {
                    const int a = kept[llround(static_cast<double>(i) * q / K)];
                    const int b = kept[llround(static_cast<double>(i + 1) * q / K)];
                    ok = covers(raw, a, b, tol);
                }
                if (ok) {
                    emit(K + 1, [&](int k) { return kept[llround(static_cast<double>(k) * q / K)]; });
                } else {
                    for (int start = 0; start < q; start += K) {
                        const int stop = min(start + K, q);
                        emit(stop - start + 1, [&](int k) { return kept[start + k]; });
                    }
                }
            }
        }
    }
    if (COUNT) {
        nspl[t] = ns;
        npts_total[t] = np;
    }
}

}  // namespace

// Streamed fit: the host produces the poses chunk by chunk into two pinned
// staging buffers; each chunk's copy runs while the next one is produced, and one
// fit kernel runs at the end over the poses resident on the device.
struct FitStream {
    int device = 0;
    cudaStream_t st = nullptr;
    double* dp = nullptr;         // all poses, device
    int64_t* doff = nullptr;
    double* dcs = nullptr;
    double* dout = nullptr;
    double* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int32_t ncomp = 0;  // fit units
    int32_t nb = 1;     // bodies: unit c fits body c % nb
    double* dhe = nullptr;
};

void rggp_fit_end(void* p) {
    FitStream* f = static_cast<FitStream*>(p);
    if (!f) return;
    cudaSetDevice(f->device);
    if (f->st) cudaStreamSynchronize(f->st);
    cudaFree(f->dp), cudaFree(f->doff), cudaFree(f->dcs), cudaFree(f->dout), cudaFree(f->dhe);
    for (int k = 0; k < 2; ++k) {
        if (f->stage[k]) cudaFreeHost(f->stage[k]);
        if (f->done[k]) cudaEventDestroy(f->done[k]);
    }
    if (f->st) cudaStreamDestroy(f->st);
    delete f;
}

// chunk_configs: capacity of each staging buffer (configurations)
void* rggp_fit_begin(const int64_t* off, int32_t ncomp, const double* he3, int32_t nbodies, const double* cos_sin,
                     int64_t chunk_configs, int32_t device) {
    FitStream* f = new FitStream();
    if (device < 0 && cudaGetDevice(&device) != cudaSuccess) device = 0;  // the caller's current device
    f->device = device;
    f->ncomp = ncomp;
    f->nb = nbodies;
    const size_t total = static_cast<size_t>(off[ncomp]);
    bool ok = cudaSetDevice(device) == cudaSuccess && cudaStreamCreateWithFlags(&f->st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMalloc(&f->dp, (total ? total : 1) * 96) == cudaSuccess &&
              cudaMalloc(&f->doff, (static_cast<size_t>(ncomp) + 1) * 8) == cudaSuccess &&
              cudaMalloc(&f->dcs, 22 * 8) == cudaSuccess &&
              cudaMalloc(&f->dhe, static_cast<size_t>(nbodies) * 24) == cudaSuccess &&
              cudaMalloc(&f->dout, (static_cast<size_t>(ncomp) + 1) * 15 * 8) == cudaSuccess;
    for (int k = 0; ok && k < 2; ++k)
        ok = cudaHostAlloc(reinterpret_cast<void**>(&f->stage[k]), static_cast<size_t>(chunk_configs) * 96, 0) == cudaSuccess &&
             cudaEventCreateWithFlags(&f->done[k], cudaEventDisableTiming) == cudaSuccess && cudaEventRecord(f->done[k], f->st) == cudaSuccess;
    ok = ok && cudaMemcpyAsync(f->doff, off, (static_cast<size_t>(ncomp) + 1) * 8, cudaMemcpyHostToDevice, f->st) == cudaSuccess &&
         cudaMemcpyAsync(f->dcs, cos_sin, 22 * 8, cudaMemcpyHostToDevice, f->st) == cudaSuccess &&
         cudaMemcpyAsync(f->dhe, he3, static_cast<size_t>(nbodies) * 24, cudaMemcpyHostToDevice, f->st) == cudaSuccess &&
         cudaStreamSynchronize(f->st) == cudaSuccess;
    if (!ok) {
        rggp_fit_end(f);
        return nullptr;
    }
    return f;
}

// the staging buffer of a slot, once its previous copy has drained
double* rggp_fit_staging(void* p, int32_t slot) {
    FitStream* f = static_cast<FitStream*>(p);
    return cudaEventSynchronize(f->done[slot]) == cudaSuccess ? f->stage[slot] : nullptr;
}

// queue the copy of a slot's nconfigs poses to configuration first_config
int rggp_fit_push(void* p, int32_t slot, int64_t first_config, int64_t nconfigs) {
    FitStream* f = static_cast<FitStream*>(p);
    cudaError_t e = cudaMemcpyAsync(f->dp + 12 * first_config, f->stage[slot], static_cast<size_t>(nconfigs) * 96,
                                    cudaMemcpyHostToDevice, f->st);
    if (e == cudaSuccess) e = cudaEventRecord(f->done[slot], f->st);
    return e;
}

// fit every component, boxes to out (ncomp x 15), release everything
int rggp_fit_finish(void* p, double* out, const InnerSpec* spec, InnerOut* inner) {
    FitStream* f = static_cast<FitStream*>(p);
    static const bool dbg = std::getenv("RGG_DEBUG_FIT") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    const auto mark = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(f->st);
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[fit] %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    };
    mark("copies");
    cudaError_t e = cudaSuccess;
    if (f->ncomp > 0) {
        fit_kernel<<<(f->ncomp + 127) / 128, 128, 0, f->st>>>(f->dp, f->doff, f->ncomp, f->dhe, f->nb, f->dcs, f->dout);
        e = cudaGetLastError();
    }
    mark("kernel");
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, f->dout, static_cast<size_t>(f->ncomp) * 15 * 8, cudaMemcpyDeviceToHost, f->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(f->st);
    mark("boxes D2H");
    if (e == cudaSuccess && spec && inner && spec->nsph > 0 && f->ncomp > 0) {
        // the splines: count, scan on the host, write
        const int nsph = spec->nsph;
        const long long nt = static_cast<long long>(f->ncomp) * nsph;
        int64_t total = 0;
        cudaMemcpyAsync(&total, f->doff + f->ncomp, 8, cudaMemcpyDeviceToHost, f->st);
        cudaStreamSynchronize(f->st);
        double* dspec = nullptr;
        V3* raw = nullptr;
        int32_t *kept = nullptr, *dns = nullptr, *dnp = nullptr, *dsn = nullptr;
        int64_t *dso = nullptr, *dpo = nullptr;
        double* dpts = nullptr;
        std::vector<double> hspec(6 * nsph);
        for (int k = 0; k < 3 * nsph; ++k) hspec[k] = spec->centre[k];
        for (int k = 0; k < nsph; ++k)
            hspec[3 * nsph + k] = spec->radius[k], hspec[4 * nsph + k] = spec->step_bound[k], hspec[5 * nsph + k] = spec->tol[k];
        auto ok = [&](cudaError_t x) { return e == cudaSuccess && (e = x) == cudaSuccess; };
        ok(cudaMalloc(&dspec, hspec.size() * 8));
        ok(cudaMalloc(&raw, static_cast<size_t>(total) * nsph * sizeof(V3) + 16));
        ok(cudaMalloc(&kept, static_cast<size_t>(total) * nsph * 4 + 16));
        ok(cudaMalloc(&dns, nt * 4));
        ok(cudaMalloc(&dnp, nt * 4));
        ok(cudaMemcpyAsync(dspec, hspec.data(), hspec.size() * 8, cudaMemcpyHostToDevice, f->st));
        const InnerDev sd{nsph, spec->K, dspec, dspec + 3 * nsph, dspec + 4 * nsph, dspec + 5 * nsph};
        const unsigned grid = static_cast<unsigned>((nt + 127) / 128);
        if (e == cudaSuccess) {
            inner_kernel<true><<<grid, 128, 0, f->st>>>(f->dp, f->doff, f->ncomp, sd, raw, kept, dns, dnp, nullptr,
                                                         nullptr, nullptr, nullptr);
            ok(cudaGetLastError());
        }
        inner->nspl.resize(nt);
        std::vector<int32_t> np(nt);
        ok(cudaMemcpyAsync(inner->nspl.data(), dns, nt * 4, cudaMemcpyDeviceToHost, f->st));
        ok(cudaMemcpyAsync(np.data(), dnp, nt * 4, cudaMemcpyDeviceToHost, f->st));
        ok(cudaStreamSynchronize(f->st));
        mark("splines count");
        std::vector<int64_t> so(nt + 1, 0), po(nt + 1, 0);
        for (long long k = 0; k < nt; ++k) so[k + 1] = so[k] + inner->nspl[k], po[k + 1] = po[k] + np[k];
        inner->npts.resize(so[nt]);
        inner->pts.resize(static_cast<size_t>(po[nt]) * 3);
        ok(cudaMalloc(&dso, (nt + 1) * 8));
        ok(cudaMalloc(&dpo, (nt + 1) * 8));
        ok(cudaMalloc(&dsn, so[nt] * 4 + 4));
        ok(cudaMalloc(&dpts, po[nt] * 24 + 8));
        ok(cudaMemcpyAsync(dso, so.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, f->st));
        ok(cudaMemcpyAsync(dpo, po.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, f->st));
        if (e == cudaSuccess) {
            inner_kernel<false><<<grid, 128, 0, f->st>>>(f->dp, f->doff, f->ncomp, sd, raw, kept, nullptr, nullptr, dso,
                                                          dpo, dsn, dpts);
            ok(cudaGetLastError());
        }
        ok(cudaMemcpyAsync(inner->npts.data(), dsn, so[nt] * 4, cudaMemcpyDeviceToHost, f->st));
        ok(cudaMemcpyAsync(inner->pts.data(), dpts, po[nt] * 24, cudaMemcpyDeviceToHost, f->st));
        ok(cudaStreamSynchronize(f->st));
        mark("splines write");
        for (void* q : {static_cast<void*>(dspec), static_cast<void*>(raw), static_cast<void*>(kept),
                        static_cast<void*>(dns), static_cast<void*>(dnp), static_cast<void*>(dso),
                        static_cast<void*>(dpo), static_cast<void*>(dsn), static_cast<void*>(dpts)})
            cudaFree(q);
    }
    rggp_fit_end(f);
    return e;
}

extern "C" int rgg_build_gpu_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        (void)cudaGetLastError();
        return 0;
    }
    return n;
}
