// rgg_device.cuh — fp64-exact device predicates of the SerRGG hot path (sm_100a).
//
// Every expression is written with explicit round-to-nearest intrinsics
// (__dadd_rn / __dsub_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn), which nvcc
// never contracts into DFMA, in the operation order of the reference's scalar
// backend (proj/src/kernels_scalar.cpp, built with -ffp-contract=off,
// proj/CMakeLists.txt:12-14).  That is what makes every predicate bit-identical
// to the reference on every input (proj/include/rgg/kernels.hpp:8-13 states the
// same contract for its AVX2 backend).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>

#include <cstdint>

namespace rggd {

__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
// x / len for a positive len (sat_prep's unit axes): a zero numerator returns x itself,
// which is the IEEE quotient (a zero with x's sign); __ddiv_rn sends a zero numerator to
// its out-of-line slow path (~100 instructions), and axis-aligned boxes have many
__device__ __forceinline__ double div_pos(double x, double len) { return x == 0.0 ? x : __ddiv_rn(x, len); }

// dot3 of kernels_scalar.cpp:35: (x0 y0 + x1 y1) + x2 y2
__device__ __forceinline__ double dot3(const double* x, const double* y) {
    return add(add(mul(x[0], y[0]), mul(x[1], y[1])), mul(x[2], y[2]));
}

// Vec3 dot (vec3.hpp:39) has the same association.
__device__ __forceinline__ double dot3v(double x0, double x1, double x2, double y0, double y1, double y2) {
    return add(add(mul(x0, y0), mul(x1, y1)), mul(x2, y2));
}

// SatBox as 21 doubles: center[0..2], e[k][j] at 3+3k+j, u[k][j] at 12+3k+j
// (proj/include/rgg/kernels.hpp:18-22).

// separated_on, proj/src/kernels_scalar.cpp:37-42.  a = edge box, b = obstacle.
__device__ __forceinline__ bool separated_on(const double* a, const double* b, const double* d, const double* ax) {
    const double ra = add(add(fabs(dot3(a + 3, ax)), fabs(dot3(a + 6, ax))), fabs(dot3(a + 9, ax)));
    const double rb = add(add(fabs(dot3(b + 3, ax)), fabs(dot3(b + 6, ax))), fabs(dot3(b + 9, ax)));
    const double s = fabs(dot3(d, ax));
    return s > add(ra, rb);
}

// sat_boxes, proj/src/kernels_scalar.cpp:48-69.  The verdict is "no tested
// axis separates"; the set of tested axes (face axes always, cross axes iff
// n2 >= 1e-12) is the reference's, so the boolean is identical whatever the
// evaluation order.  COUNT accumulates SATCOST_ref in
// reference order when non-null.
template <bool COUNT>
__device__ __forceinline__ bool sat_boxes(const double* a, const double* b, long long* cost) {
    double d[3];
    d[0] = sub(b[0], a[0]);
    d[1] = sub(b[1], a[1]);
    d[2] = sub(b[2], a[2]);
    int flops = 3;
    bool sep = false;
#pragma unroll
    for (int k = 0; k < 3 && !sep; ++k) {
        flops += 40;
        sep = separated_on(a, b, d, a + 12 + 3 * k);
    }
#pragma unroll
    for (int k = 0; k < 3 && !sep; ++k) {
        flops += 40;
        sep = separated_on(a, b, d, b + 12 + 3 * k);
    }
#pragma unroll
    for (int i = 0; i < 3 && !sep; ++i) {
        const double* x = a + 12 + 3 * i;
#pragma unroll
        for (int j = 0; j < 3 && !sep; ++j) {
            const double* y = b + 12 + 3 * j;
            double axis[3];
            axis[0] = sub(mul(x[1], y[2]), mul(x[2], y[1]));
            axis[1] = sub(mul(x[2], y[0]), mul(x[0], y[2]));
            axis[2] = sub(mul(x[0], y[1]), mul(x[1], y[0]));
            const double n2 = dot3(axis, axis);
            flops += 14;
            if (n2 >= 1e-12) {
                flops += 40;
                sep = separated_on(a, b, d, axis);
            }
        }
    }
    if (COUNT) *cost += flops;
    return !sep;
}

// One lane's share of sat_boxes: the axes {g, g+G, ...} of the reference's
// 15 (a.u[0..2], b.u[0..2], then a.u[i] x b.u[j] row-major).  The pair is
// separated iff some lane finds a separating tested axis, so OR-ing the
// lanes' results gives exactly !sat_boxes(a, b).  a/b stay in memory (global,
// L1-cached / shared) so the axis index can be dynamic.
__device__ __forceinline__ bool sat_separated_part(const double* a, const double* b, int g, int G) {
    double d[3];
    d[0] = sub(b[0], a[0]);
    d[1] = sub(b[1], a[1]);
    d[2] = sub(b[2], a[2]);
    for (int ax = g; ax < 15; ax += G) {
        double axis[3];
        if (ax < 6) {
            const double* u = ax < 3 ? a + 12 + 3 * ax : b + 12 + 3 * (ax - 3);
            axis[0] = u[0];
            axis[1] = u[1];
            axis[2] = u[2];
        } else {
            const double* x = a + 12 + 3 * ((ax - 6) / 3);
            const double* y = b + 12 + 3 * ((ax - 6) % 3);
            axis[0] = sub(mul(x[1], y[2]), mul(x[2], y[1]));
            axis[1] = sub(mul(x[2], y[0]), mul(x[0], y[2]));
            axis[2] = sub(mul(x[0], y[1]), mul(x[1], y[0]));
            if (!(dot3(axis, axis) >= 1e-12)) continue;
        }
        if (separated_on(a, b, d, axis)) return true;
    }
    return false;
}

// seg_point_dist + seg_sphere, proj/src/kernels_scalar.cpp:81-96.
// s = SegPrep (a[3], d[3], dd).  Closed predicate.
__device__ __forceinline__ bool seg_sphere(const double* s, const double* c, double r_total) {
    const double px = sub(c[0], s[0]);
    const double py = sub(c[1], s[1]);
    const double pz = sub(c[2], s[2]);
    double t = 0.0;
    if (s[6] > 0.0) {
        t = __ddiv_rn(add(add(mul(px, s[3]), mul(py, s[4])), mul(pz, s[5])), s[6]);
        t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    }
    const double qx = sub(px, mul(t, s[3]));
    const double qy = sub(py, mul(t, s[4]));
    const double qz = sub(pz, mul(t, s[5]));
    return __dsqrt_rn(add(add(mul(qx, qx), mul(qy, qy)), mul(qz, qz))) <= r_total;
}

// seg_sphere with an exact fast path.  Returns the same verdict as seg_sphere
// on every input: the clamp cases t = 0 (num <= 0) and t = 1 (num >= dd)
// produce the reference's q without the division (num/dd lands on the clamp
// value), and sqrt_rn(x) <= r is decided from x against r*r outside a 2^-40
// relative band (sqrt_rn is monotone and within half an ulp), so the fp64
// division and square root run only for interior projections and for the
// band (SURVEY.md §7 "fp32-fast + recheck" done entirely in fp64).
__device__ __forceinline__ bool seg_sphere_fast(const double* s, const double* c, double r_total) {
    if (!(r_total >= 0.0)) return false;  // sqrt_rn(x) >= 0 > r_total (or NaN)
    const double px = sub(c[0], s[0]);
    const double py = sub(c[1], s[1]);
    const double pz = sub(c[2], s[2]);
    double qx = px, qy = py, qz = pz;
    if (s[6] > 0.0) {
        const double num = add(add(mul(px, s[3]), mul(py, s[4])), mul(pz, s[5]));
        if (!(num == num)) return false;  // NaN propagates to the reference's distance
        if (num >= s[6]) {  // t = 1 (num/dd >= 1 is clamped, or is 1.0)
            qx = sub(px, s[3]);
            qy = sub(py, s[4]);
            qz = sub(pz, s[5]);
        } else if (num > 0.0) {  // 0 < t <= 1
            double t = __ddiv_rn(num, s[6]);
            t = t > 1.0 ? 1.0 : t;
            qx = sub(px, mul(t, s[3]));
            qy = sub(py, mul(t, s[4]));
            qz = sub(pz, mul(t, s[5]));
        }  // num <= 0: t = +-0 and q == p in value
    }
    const double x = add(add(mul(qx, qx), mul(qy, qy)), mul(qz, qz));
    const double r2 = r_total * r_total;
    if (x < r2 * (1.0 - 0x1p-40)) return true;
    if (x > r2 * (1.0 + 0x1p-40)) return false;
    return __dsqrt_rn(x) <= r_total;
}

// ---------------------------------------------------------------- fp32 filters
//
// fp32 versions of the two predicates that return 0 (false for sure), 1 (true
// for sure) or 2 (undecided).  Each carries a rigorous bound on the distance
// between its fp32 result and the exact-arithmetic value, and only calls a
// decision when the margin clears that bound plus the reference's own fp64
// rounding (which is ~1e-16 relative, far below it).  Undecided pairs are
// re-evaluated with the exact fp64 sequence, so the verdicts are still the
// reference's bit for bit.  u = 2^-24 (fp32 unit roundoff).
//
// Box32 (filter operand of a SatBox, one 128-byte line): the fp64 centre (d is
// formed in fp64), e[9], u[9] rounded to nearest, L = sum of |e_k|_1 rounded up.
// The filter reads only this line; the 176-byte fp64 SatBox is read only for the
// rare undecided pair.
// The first 80 bytes are what sat_filter32g reads (five 16-byte loads, Box32G).
struct __align__(16) Box32 {
    double c[3];
    float u[9];
    float h[3];      // |e_k|_2 rounded to nearest: the half extents (sat_filter32g)
    float Lh;        // h_0 + h_1 + h_2 rounded up
    uint32_t degen;  // some unit axis is zero (zero-extent box): the filters defer to fp64
    float L;         // sum_k |e_k|_1 rounded up (sat_filter32)
    float e[9];
    float pad[2];
};
static_assert(sizeof(Box32) == 128, "Box32 is one cache line");

struct __align__(16) Box32G {
    double c[3];
    float u[9];
    float h[3];
    float Lh;
    uint32_t degen;
};
static_assert(sizeof(Box32G) == 80 && offsetof(Box32, L) == 80, "Box32G is the head of Box32");

// the head of a Box32 in five vector loads
__device__ __forceinline__ Box32G load_box32g(const Box32* p) {
    Box32G x;
    const float4* q = reinterpret_cast<const float4*>(p);
    float4* d = reinterpret_cast<float4*>(&x);
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] = q[k];
    return x;
}

__device__ __forceinline__ float dot3f(const float* x, const float* y) {
    return fmaf(x[2], y[2], fmaf(x[1], y[1], x[0] * y[0]));
}

// margin |d.ax| - (ra + rb) of one axis in fp32
__device__ __forceinline__ float margin32(const float* d, const Box32& a, const Box32& b, const float* ax) {
    const float ra = fabsf(dot3f(a.e, ax)) + fabsf(dot3f(a.e + 3, ax)) + fabsf(dot3f(a.e + 6, ax));
    const float rb = fabsf(dot3f(b.e, ax)) + fabsf(dot3f(b.e + 3, ax)) + fabsf(dot3f(b.e + 6, ax));
    return fabsf(dot3f(d, ax)) - (ra + rb);
}

// sat_boxes filter.  Error model per axis (|axis_i| <= A): |m32 - m| <= 10 u S A
// for face axes (inputs rounded, one rounding per FMA / add, S = |d|_1 + La + Lb);
// cross axes add the axis' own error E_i <= 4u(|x1 y2| + |x2 y1|): |dm| <= S max E.
// Margins below twice those bounds are undecided; so are cross axes whose
// n2 >= 1e-12 decision (kernels_scalar.cpp:64-65) is within its error.
__device__ __forceinline__ int sat_filter32(const double* ca, const Box32& a, const double* cb, const Box32& b) {
    constexpr float u = 5.9604645e-8f;  // 2^-24
    float d[3];
    d[0] = __double2float_rn(__dsub_rn(cb[0], ca[0]));
    d[1] = __double2float_rn(__dsub_rn(cb[1], ca[1]));
    d[2] = __double2float_rn(__dsub_rn(cb[2], ca[2]));
    const float S = (fabsf(d[0]) + fabsf(d[1]) + fabsf(d[2]) + a.L + b.L) * (1.0f + 16.0f * u);
    if (!(S < 3.0e37f)) return 2;  // non-finite or huge operands: let fp64 decide
    const float tol_face = 20.0f * u * S;
    bool sep = false, undecided = false;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const float* ax = k < 3 ? a.u + 3 * k : b.u + 3 * (k - 3);
        const float m = margin32(d, a, b, ax);
        sep |= m > tol_face;
        undecided |= fabsf(m) <= tol_face;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float* x = a.u + 3 * i;
            const float* y = b.u + 3 * j;
            float ax[3], er[3];
            ax[0] = fmaf(x[1], y[2], -x[2] * y[1]);
            ax[1] = fmaf(x[2], y[0], -x[0] * y[2]);
            ax[2] = fmaf(x[0], y[1], -x[1] * y[0]);
            er[0] = 8.0f * u * (fabsf(x[1] * y[2]) + fabsf(x[2] * y[1]));
            er[1] = 8.0f * u * (fabsf(x[2] * y[0]) + fabsf(x[0] * y[2]));
            er[2] = 8.0f * u * (fabsf(x[0] * y[1]) + fabsf(x[1] * y[0]));
            const float n2 = dot3f(ax, ax);
            const float n2err = (2.0f * fabsf(ax[0]) + 2.0f * er[0]) * er[0] + (2.0f * fabsf(ax[1]) + 2.0f * er[1]) * er[1] +
                                (2.0f * fabsf(ax[2]) + 2.0f * er[2]) * er[2] + 8.0f * u * n2 + 1e-18f;
            const bool tested = n2 - n2err >= 1e-12f * (1.0f + 1e-6f);
            const bool maybe = !tested && n2 + n2err >= 1e-12f * (1.0f - 1e-6f);
            const float A = fmaxf(fabsf(ax[0]), fmaxf(fabsf(ax[1]), fabsf(ax[2])));
            const float E = fmaxf(er[0], fmaxf(er[1], er[2]));
            const float tol = 2.0f * S * (E + 10.0f * u * A);
            const float m = margin32(d, a, b, ax);
            sep |= tested & (m > tol);
            undecided |= (tested & (fabsf(m) <= tol)) | (maybe & (m > -tol));
        }
    }
    if (sep) return 0;           // a tested axis separates for sure
    return undecided ? 2 : 1;    // every tested axis overlaps for sure -> intersect
}

// The Box32 terms of one SatBox (fp64 e[9], u[9] at sat + 3, sat + 12).
__host__ __device__ inline void box32_terms(const double* sat, Box32& x) {
    double l1 = 0.0, hd[3];
    bool degen = false;
    for (int k = 0; k < 3; ++k) {
        double n2 = 0.0, u2 = 0.0;
        for (int j = 0; j < 3; ++j) {
            const double e = sat[3 + 3 * k + j], uu = sat[12 + 3 * k + j];
            x.e[3 * k + j] = static_cast<float>(e);
            x.u[3 * k + j] = static_cast<float>(uu);
            l1 += e < 0 ? -e : e;
            n2 += e * e;
            u2 += uu * uu;
        }
        hd[k] = sqrt(n2);
        x.h[k] = static_cast<float>(hd[k]);
        degen |= !(u2 > 0.5);
    }
    // sat_filter32g's margins equal the reference's for orthonormal frames with e_k = |e_k| u_k
    // (what sat_prep produces, kernels_scalar.cpp:18-28): a caller's SatBox outside that
    // (|u_i.u_j|, ||u_k|^2 - 1| or the e/u misalignment above 1e-9) is decided in fp64
    for (int i = 0; i < 3 && !degen; ++i) {
        const double* ui = sat + 12 + 3 * i;
        const double* ei = sat + 3 + 3 * i;
        const double uu = ui[0] * ui[0] + ui[1] * ui[1] + ui[2] * ui[2];
        degen |= !(fabs(uu - 1.0) <= 1e-9);
        const double h = hd[i];
        for (int k = 0; k < 3; ++k) degen |= !(fabs(ei[k] - h * ui[k]) <= 1e-9 * (h + 1e-300));
        for (int j = i + 1; j < 3; ++j) {
            const double* uj = sat + 12 + 3 * j;
            degen |= !(fabs(ui[0] * uj[0] + ui[1] * uj[1] + ui[2] * uj[2]) <= 1e-9);
        }
    }
    x.degen = degen ? 1u : 0u;
    // rounded up: nextafter of the nearest float of a value inflated by 1e-15
    const float lf = static_cast<float>(l1 * (1.0 + 1e-15));
    const float hf = static_cast<float>((static_cast<double>(x.h[0]) + x.h[1] + x.h[2]) * (1.0 + 1e-15));
#ifdef __CUDA_ARCH__
    x.L = nextafterf(lf, __int_as_float(0x7f800000));
    x.Lh = nextafterf(hf, __int_as_float(0x7f800000));
#else
    x.L = std::nextafter(lf, std::numeric_limits<float>::infinity());
    x.Lh = std::nextafter(hf, std::numeric_limits<float>::infinity());
#endif
}

// sat_boxes filter in the frame of box a (the classic OBB form): with
// R_ij = a.u_i . b.u_j, t = d in a's frame, t' = d in b's frame and half
// extents h = |e_k|, the reference's 15 margins (kernels_scalar.cpp:37-69) are
//   a.u_i:        |t_i|  - (ha_i + sum_j hb_j |R_ij|)
//   b.u_j:        |t'_j| - (sum_i ha_i |R_ij| + hb_j)
//   a.u_i x b.u_j: |t_i2 R_i1j - t_i1 R_i2j| - (ha_i1 |R_i2j| + ha_i2 |R_i1j| + hb_j1 |R_ij2| + hb_j2 |R_ij1|)
// up to the frames' orthogonality (~1e-14 of S for the reference's boxes),
// for either handedness.  fp32 error (inputs rounded once, dot products by
// FMA): faces <= 10 u S, crosses <= 26 u S with S = |d|_1 + Lh_a + Lh_b; the
// tolerances are 16 u S and 32 u S.  The cross axis is skipped by the
// reference when |u_i x v_j|^2 < 1e-12: |R_ij| <= 1 - 2^-10 is tested for
// sure; nearer-parallel pairs classify n2 from the explicit cross product as
// sat_filter32 does (exact zeros stay exact).  Same return as sat_filter32.
__device__ __forceinline__ int sat_filter32g(const Box32G& a, const double* cb, const Box32G& b) {
    constexpr float u = 5.9604645e-8f;  // 2^-24
    if (a.degen | b.degen) return 2;
    float d[3];
    d[0] = __double2float_rn(__dsub_rn(cb[0], a.c[0]));
    d[1] = __double2float_rn(__dsub_rn(cb[1], a.c[1]));
    d[2] = __double2float_rn(__dsub_rn(cb[2], a.c[2]));
    const float S = (fabsf(d[0]) + fabsf(d[1]) + fabsf(d[2]) + a.Lh + b.Lh) * (1.0f + 16.0f * u);
    if (!(S < 3.0e37f)) return 2;
    float R[3][3], AR[3][3], t[3], tb[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        t[i] = dot3f(d, a.u + 3 * i);
        tb[i] = dot3f(d, b.u + 3 * i);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            R[i][j] = dot3f(a.u + 3 * i, b.u + 3 * j);
            AR[i][j] = fabsf(R[i][j]);
        }
    }
    const float tol_f = 16.0f * u * S, tol_c = 32.0f * u * S;
    bool sep = false, undecided = false;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float ma = fabsf(t[i]) - (a.h[i] + fmaf(b.h[2], AR[i][2], fmaf(b.h[1], AR[i][1], b.h[0] * AR[i][0])));
        const float mb = fabsf(tb[i]) - (fmaf(a.h[2], AR[2][i], fmaf(a.h[1], AR[1][i], a.h[0] * AR[0][i])) + b.h[i]);
        sep |= (ma > tol_f) | (mb > tol_f);
        undecided |= (fabsf(ma) <= tol_f) | (fabsf(mb) <= tol_f);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const int i1 = i == 2 ? 0 : i + 1, i2 = i == 0 ? 2 : i - 1;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const int j1 = j == 2 ? 0 : j + 1, j2 = j == 0 ? 2 : j - 1;
            const float m = fabsf(fmaf(t[i2], R[i1][j], -t[i1] * R[i2][j])) -
                            (fmaf(a.h[i1], AR[i2][j], a.h[i2] * AR[i1][j]) + fmaf(b.h[j1], AR[i][j2], b.h[j2] * AR[i][j1]));
            bool tested = true, maybe = false;
            if (AR[i][j] > 1.0f - 9.765625e-4f) {  // near-parallel edges: n2 from the explicit cross product
                const float* x = a.u + 3 * i;
                const float* y = b.u + 3 * j;
                float ax[3], er[3];
                ax[0] = fmaf(x[1], y[2], -x[2] * y[1]);
                ax[1] = fmaf(x[2], y[0], -x[0] * y[2]);
                ax[2] = fmaf(x[0], y[1], -x[1] * y[0]);
                er[0] = 8.0f * u * (fabsf(x[1] * y[2]) + fabsf(x[2] * y[1]));
                er[1] = 8.0f * u * (fabsf(x[2] * y[0]) + fabsf(x[0] * y[2]));
                er[2] = 8.0f * u * (fabsf(x[0] * y[1]) + fabsf(x[1] * y[0]));
                const float n2 = dot3f(ax, ax);
                const float n2err = (2.0f * fabsf(ax[0]) + 2.0f * er[0]) * er[0] + (2.0f * fabsf(ax[1]) + 2.0f * er[1]) * er[1] +
                                    (2.0f * fabsf(ax[2]) + 2.0f * er[2]) * er[2] + 8.0f * u * n2 + 1e-18f;
                tested = n2 - n2err >= 1e-12f * (1.0f + 1e-6f);
                maybe = !tested && n2 + n2err >= 1e-12f * (1.0f - 1e-6f);
            }
            sep |= tested & (m > tol_c);
            undecided |= (tested & (fabsf(m) <= tol_c)) | (maybe & (m > -tol_c));
        }
    }
    if (sep) return 0;
    return undecided ? 2 : 1;
}

// seg_sphere filter.  p and d come from the fp64 operands; t uses a fast
// reciprocal.  |x32 - |p - t* d|^2| <= 32 u (|p| + |d|)^2 covers the roundings
// and the t error (quadratic at an interior optimum, exact at the clamps, and
// a near-clamp flip moves x by <= 2 t |p.d| with t at rounding level); the
// reference's x is within 1e-15 of the same value and its sqrt(x) <= r is
// x <= r^2 up to half an ulp.
__device__ __forceinline__ int seg_filter32(const double* s, const double* c, double r_total) {
    constexpr float u = 5.9604645e-8f;
    if (!(r_total >= 0.0)) return 0;
    const float px = __double2float_rn(__dsub_rn(c[0], s[0]));
    const float py = __double2float_rn(__dsub_rn(c[1], s[1]));
    const float pz = __double2float_rn(__dsub_rn(c[2], s[2]));
    const float dx = __double2float_rn(s[3]), dy = __double2float_rn(s[4]), dz = __double2float_rn(s[5]);
    const float dd = __double2float_rn(s[6]);
    float t = 0.0f;
    if (dd > 0.0f) {
        const float num = fmaf(pz, dz, fmaf(py, dy, px * dx));
        t = fminf(fmaxf(num * __frcp_rn(dd), 0.0f), 1.0f);
    }
    const float qx = fmaf(-t, dx, px), qy = fmaf(-t, dy, py), qz = fmaf(-t, dz, pz);
    const float x = fmaf(qz, qz, fmaf(qy, qy, qx * qx));
    const float P = fabsf(px) + fabsf(py) + fabsf(pz) + fabsf(dx) + fabsf(dy) + fabsf(dz);
    const float err = 64.0f * u * P * P + 1e-30f;
    const float r = static_cast<float>(r_total);
    const float r2 = r * r;
    const float r2err = 8.0f * u * r2;
    if (!(x == x) || !(P < 3.0e18f)) return 2;  // non-finite inputs: let fp64 decide
    if (x + err < r2 - r2err) return 1;
    if (x - err > r2 + r2err) return 0;
    return 2;
}

// seg_filter32 with the segment-only terms hoisted: one Seg32 per (segment,
// r_total), then one branch-free call per sphere.  Same error model (P summed in
// another order: the 64u P^2 bound keeps a factor-2 margin over the 32u needed).
struct Seg32 {
    float dx, dy, dz, inv_dd, dabs, r2, r2err;
    bool dd_pos, r_ok;
};

__device__ __forceinline__ Seg32 seg32_prep(const double* s, double r_total) {
    constexpr float u = 5.9604645e-8f;
    Seg32 g;
    g.r_ok = r_total >= 0.0;
    g.dx = __double2float_rn(s[3]);
    g.dy = __double2float_rn(s[4]);
    g.dz = __double2float_rn(s[5]);
    const float dd = __double2float_rn(s[6]);
    g.dd_pos = dd > 0.0f;
    g.inv_dd = g.dd_pos ? __frcp_rn(dd) : 0.0f;
    g.dabs = fabsf(g.dx) + fabsf(g.dy) + fabsf(g.dz);
    const float r = static_cast<float>(r_total);
    g.r2 = r * r;
    g.r2err = 8.0f * u * g.r2;
    return g;
}

__device__ __forceinline__ int seg_filter32_pre(const double* s, const Seg32& g, const double* c) {
    constexpr float u = 5.9604645e-8f;
    const float px = __double2float_rn(__dsub_rn(c[0], s[0]));
    const float py = __double2float_rn(__dsub_rn(c[1], s[1]));
    const float pz = __double2float_rn(__dsub_rn(c[2], s[2]));
    float t = 0.0f;
    if (g.dd_pos) {
        const float num = fmaf(pz, g.dz, fmaf(py, g.dy, px * g.dx));
        t = fminf(fmaxf(num * g.inv_dd, 0.0f), 1.0f);
    }
    const float qx = fmaf(-t, g.dx, px), qy = fmaf(-t, g.dy, py), qz = fmaf(-t, g.dz, pz);
    const float x = fmaf(qz, qz, fmaf(qy, qy, qx * qx));
    const float P = ((fabsf(px) + fabsf(py)) + fabsf(pz)) + g.dabs;
    const float err = 64.0f * u * P * P + 1e-30f;
    const int f = !(x == x) || !(P < 3.0e18f) ? 2 : (x + err < g.r2 - g.r2err ? 1 : (x - err > g.r2 + g.r2err ? 0 : 2));
    return g.r_ok ? f : 0;
}

// The same filter over a compact fp32 copy of the segment record (32 bytes:
// a[3], d[3], dd, spline radius, each rounded to nearest; rgg_store.cu segs_kernel),
// so the narrow kernel streams half the bytes and reads the fp64 record only for
// an undecided pair.  With a and the sphere centre c rounded before the
// subtraction, p32 = fl(c32 - a32) carries an absolute error of at most
// E = u(|c|_1 + |a|_1) beyond the one rounding the 64u P^2 model covers; the
// distance to a segment is 1-Lipschitz in p, so sqrt(x) moves by at most E and x
// by at most 2 sqrt(x) E + E^2 <= 2 P E + E^2 (P >= |q|_1 >= sqrt(x)), both
// charged with 10 % margin.  r = fl(fl(o_r) + spline32) is within 3u r of the
// fp64 r_total, so r^2 within 7u; the band uses 16u.  A non-positive or tiny r
// (never in a valid layout) is left to fp64, which applies the reference's sign rule.
struct SegF {
    float ax, ay, az, dx, dy, dz, inv_dd, dabs, aabs, r2, r2err;
    bool dd_pos, r_fast;
};

__device__ __forceinline__ SegF segf_prep(float4 v0, float4 v1, float ro) {
    constexpr float u = 5.9604645e-8f;
    SegF g;
    g.ax = v0.x, g.ay = v0.y, g.az = v0.z;
    g.dx = v0.w, g.dy = v1.x, g.dz = v1.y;
    g.dd_pos = v1.z > 0.0f;
    g.inv_dd = g.dd_pos ? __frcp_rn(v1.z) : 0.0f;
    g.dabs = fabsf(g.dx) + fabsf(g.dy) + fabsf(g.dz);
    g.aabs = fabsf(g.ax) + fabsf(g.ay) + fabsf(g.az);
    const float r = ro + v1.w;  // ro = fl(o_minus_r)
    g.r_fast = r > 16.0f * u * (fabsf(ro) + fabsf(v1.w)) && r < 1.0e18f;
    g.r2 = r * r;
    g.r2err = 16.0f * u * g.r2;
    return g;
}

// c32: the sphere centre rounded to nearest; cabs = |c32|_1 (>= |c|_1 (1 - u), the
// 10 % margin covers the difference).  1 = hit, 0 = miss, 2 = undecided.
__device__ __forceinline__ int segf_filter(const SegF& g, float cx, float cy, float cz, float cabs) {
    constexpr float u = 5.9604645e-8f;
    if (!g.r_fast) return 2;
    const float px = cx - g.ax, py = cy - g.ay, pz = cz - g.az;
    float t = 0.0f;
    if (g.dd_pos) {
        const float num = fmaf(pz, g.dz, fmaf(py, g.dy, px * g.dx));
        t = fminf(fmaxf(num * g.inv_dd, 0.0f), 1.0f);
    }
    const float qx = fmaf(-t, g.dx, px), qy = fmaf(-t, g.dy, py), qz = fmaf(-t, g.dz, pz);
    const float x = fmaf(qz, qz, fmaf(qy, qy, qx * qx));
    const float P = ((fabsf(px) + fabsf(py)) + fabsf(pz)) + g.dabs;
    const float E = 1.1f * u * (cabs + g.aabs);
    const float err = 64.0f * u * P * P + 2.2f * P * E + 1.1f * E * E + 1e-30f;
    return !(x == x) || !(P < 3.0e18f) || !(cabs < 1.0e18f) ? 2
                                                          : (x + err < g.r2 - g.r2err ? 1 : (x - err > g.r2 + g.r2err ? 0 : 2));
}

// sat_prep, proj/src/kernels_scalar.cpp:7-30.
__device__ __forceinline__ void sat_prep(const double* c, double* s) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int hi = (1 << k) * 3;
#pragma unroll
        for (int j = 0; j < 3; ++j) s[3 + 3 * k + j] = mul(0.5, sub(c[hi + j], c[j]));
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) s[j] = add(add(add(c[j], s[3 + j]), s[6 + j]), s[9 + j]);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double* ek = s + 3 + 3 * k;
        const double n2 = add(add(mul(ek[0], ek[0]), mul(ek[1], ek[1])), mul(ek[2], ek[2]));
        if (n2 > 0.0) {
            const double len = __dsqrt_rn(n2);
#pragma unroll
            for (int j = 0; j < 3; ++j) s[12 + 3 * k + j] = div_pos(ek[j], len);
        } else {
            s[12 + 3 * k + 0] = s[12 + 3 * k + 1] = s[12 + 3 * k + 2] = 0.0;
        }
    }
}

// Transform::apply, proj/include/rgg/vec3.hpp:72-76: ((r0 x + r1 y) + r2 z) + t.
__device__ __forceinline__ void tf_apply(const double* rt, double x, double y, double z, double* out) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        out[i] = add(add(add(mul(rt[3 * i], x), mul(rt[3 * i + 1], y)), mul(rt[3 * i + 2], z)), rt[9 + i]);
}

// Aabb::overlaps, proj/include/rgg/vec3.hpp:126-129 (closed).  Evaluated
// without short-circuit so all twelve operands load in parallel.
__device__ __forceinline__ bool overlaps(const double* a, const double* b) {
    const double b0 = b[0], b1 = b[1], b2 = b[2], b3 = b[3], b4 = b[4], b5 = b[5];
    return (a[0] <= b3) & (b0 <= a[3]) & (a[1] <= b4) & (b1 <= a[4]) & (a[2] <= b5) & (b2 <= a[5]);
}

// sat_boxes with every tested axis evaluated (no early exit) from register
// operands: the 15 axis tests are independent, so their latency overlaps and
// the critical path is one axis deep.  A degenerate cross axis (n2 < 1e-12,
// or NaN) is masked out exactly where the reference skips it, so the verdict
// -- "no tested axis separates" -- is bit-for-bit sat_boxes (kernels_scalar.cpp:48-69).
__device__ __forceinline__ bool sat_boxes_flat(const double* A, const double* Bx) {
    double a[21], b[21];
#pragma unroll
    for (int k = 0; k < 21; ++k) {
        a[k] = A[k];
        b[k] = Bx[k];
    }
    double d[3];
    d[0] = sub(b[0], a[0]);
    d[1] = sub(b[1], a[1]);
    d[2] = sub(b[2], a[2]);
    bool sep = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) sep |= separated_on(a, b, d, a + 12 + 3 * k);
#pragma unroll
    for (int k = 0; k < 3; ++k) sep |= separated_on(a, b, d, b + 12 + 3 * k);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double* x = a + 12 + 3 * i;
            const double* y = b + 12 + 3 * j;
            double axis[3];
            axis[0] = sub(mul(x[1], y[2]), mul(x[2], y[1]));
            axis[1] = sub(mul(x[2], y[0]), mul(x[0], y[2]));
            axis[2] = sub(mul(x[0], y[1]), mul(x[1], y[0]));
            const bool tested = dot3(axis, axis) >= 1e-12;
            sep |= tested & separated_on(a, b, d, axis);
        }
    }
    return !sep;
}

}  // namespace rggd
