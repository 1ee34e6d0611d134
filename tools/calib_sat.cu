// Per-warp cost of one round of SAT / segment-sphere tests with operands in L1
// (profiling helper, not product code).  Uses the product's device predicates.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2603_28674_b200/csrc/rgg_device.cuh"

__global__ void filt_k(const double* boxes, const rggd::Box32* b32, const double* obst, int rounds,
                       unsigned long long* cyc, int* sink) {
    const int lane = threadIdx.x & 31;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) % 4096;
    int acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) acc += rggd::sat_filter32(boxes + 22 * i, b32[i], obst + 22 * (r & 7), b32[r & 7]);
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) sink[0] = acc;
}

__global__ void segf_k(const double* segs, const double* cen, int rounds, unsigned long long* cyc, int* sink) {
    const int lane = threadIdx.x & 31;
    const double* s = segs + 8 * ((blockIdx.x * blockDim.x + threadIdx.x) % 4096);
    int acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r)
        for (int sp = 0; sp < 5; ++sp) acc += rggd::seg_filter32(s, cen + 3 * ((r + sp) & 7), 0.6);
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) sink[0] = acc;
}

template <int MODE>
__global__ void sat_k(const double* boxes, const double* obst, int rounds, unsigned long long* cyc, int* sink) {
    const int lane = threadIdx.x & 31;
    const double* a = boxes + 22 * ((blockIdx.x * blockDim.x + threadIdx.x) % 4096);
    int acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
        bool h;
        if (MODE == 0) h = rggd::sat_boxes_flat(a, obst + 21 * (r & 7));
        else h = rggd::sat_boxes<false>(a, obst + 21 * (r & 7), nullptr);
        acc += h;
    }
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) sink[0] = acc;
}

__global__ void seg_k(const double* segs, const double* cen, int rounds, unsigned long long* cyc, int* sink) {
    const int lane = threadIdx.x & 31;
    const double* s = segs + 8 * ((blockIdx.x * blockDim.x + threadIdx.x) % 4096);
    int acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r)
        for (int sp = 0; sp < 5; ++sp) acc += rggd::seg_sphere_fast(s, cen + 3 * ((r + sp) & 7), 0.6);
    const long long t1 = clock64();
    if (lane == 0) atomicAdd(cyc, (unsigned long long)(t1 - t0));
    if (acc == 12345) sink[0] = acc;
}

int main() {
    // random boxes near contact
    const int nb = 4096;
    double* hb = new double[nb * 22];
    srand(1);
    auto U = [] { return rand() / double(RAND_MAX) * 2 - 1; };
    for (int i = 0; i < nb; ++i) {
        double* b = hb + 22 * i;
        for (int j = 0; j < 3; ++j) b[j] = U();
        for (int k = 0; k < 3; ++k) {
            double v[3] = {U(), U(), U()}, n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            for (int j = 0; j < 3; ++j) b[12 + 3 * k + j] = v[j] / n, b[3 + 3 * k + j] = v[j] / n * 0.6;
        }
    }
    double *db, *dobst, *dseg, *dcen;
    cudaMalloc(&db, nb * 22 * 8);
    cudaMemcpy(db, hb, nb * 22 * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&dobst, 8 * 21 * 8);
    cudaMemcpy(dobst, hb, 8 * 21 * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&dseg, nb * 8 * 8);
    for (int i = 0; i < nb; ++i) { double* s = hb + 8 * i; for (int j = 0; j < 6; ++j) s[j] = U(); s[6] = s[3]*s[3]+s[4]*s[4]+s[5]*s[5]; }
    cudaMemcpy(dseg, hb, nb * 8 * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&dcen, 8 * 3 * 8);
    cudaMemcpy(dcen, hb, 24 * 8, cudaMemcpyHostToDevice);
    rggd::Box32* b32h = new rggd::Box32[nb];
    for (int i = 0; i < nb; ++i) { double l = 0; for (int k = 0; k < 9; ++k) { b32h[i].e[k] = hb[22*i+3+k]; b32h[i].u[k] = hb[22*i+12+k]; l += fabs(hb[22*i+3+k]); } b32h[i].L = l * 1.0001; }
    rggd::Box32* db32; cudaMalloc(&db32, nb * sizeof(rggd::Box32)); cudaMemcpy(db32, b32h, nb * sizeof(rggd::Box32), cudaMemcpyHostToDevice);
    unsigned long long* cyc; int* sink;
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 4);
    for (int warps_per_sm : {1, 4, 16, 32}) {
        for (int mode = 0; mode < 5; ++mode) {
            cudaMemset(cyc, 0, 8);
            const int rounds = 64;
            const int block = 128, grid = 148 * warps_per_sm / 4 > 0 ? 148 * warps_per_sm / 4 : 148;
            const int g = warps_per_sm == 1 ? 148 : grid;
            const int bs = warps_per_sm == 1 ? 32 : block;
            if (mode == 0) sat_k<0><<<g, bs>>>(db, dobst, rounds, cyc, sink);
            if (mode == 1) sat_k<1><<<g, bs>>>(db, dobst, rounds, cyc, sink);
            if (mode == 2) seg_k<<<g, bs>>>(dseg, dcen, rounds, cyc, sink);
            if (mode == 3) filt_k<<<g, bs>>>(db, db32, db, rounds, cyc, sink);
            if (mode == 4) segf_k<<<g, bs>>>(dseg, dcen, rounds, cyc, sink);
            cudaDeviceSynchronize();
            unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double warps = double(g) * bs / 32;
            printf("warps/SM %2d %-14s cycles per warp-round %8.0f\n", warps_per_sm,
                   mode == 0 ? "sat flat" : mode == 1 ? "sat early-exit" : mode == 2 ? "seg x5 spheres" : mode == 3 ? "sat filter32" : "seg filter32 x5", c / warps / rounds);
        }
    }
    return 0;
}
