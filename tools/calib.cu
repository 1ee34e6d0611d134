// Calibration microbenchmarks (profiling helper, not product code).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_k() {}
__global__ void aabb_k(const double2* __restrict__ a, int n, const double* __restrict__ boxes, int nb, unsigned char* out) {
    __shared__ double sb[64 * 6];
    for (int t = threadIdx.x; t < nb * 6; t += blockDim.x) sb[t] = boxes[t];
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double2 p0 = a[c], p1 = a[n + c], p2 = a[2 * n + c];
    unsigned m = 0;
    for (int k = 0; k < nb; ++k) {
        const double* b = sb + 6 * k;
        m |= ((p0.x <= b[3]) & (b[0] <= p1.y) & (p0.y <= b[4]) & (b[1] <= p2.x) & (p1.x <= b[5]) & (b[2] <= p2.y)) << (k & 31);
    }
    out[c] = m & 0xff;
}
__global__ void atomic_k(int* ctr, int per) {
    for (int i = 0; i < per; ++i) if ((threadIdx.x & 31) == 0) atomicAdd(ctr, 1);
}
__global__ void chain_k(double* out, int iters) {  // dependent fp64 chain per thread
    double x = threadIdx.x * 1e-3;
    for (int i = 0; i < iters; ++i) x = __dadd_rn(__dmul_rn(x, 0.999), 1e-3);
    if (x == 1234.5) out[0] = x;
}
int main() {
    const int n = 124080, nb = 4;
    double2* a; double* boxes; unsigned char* out; int* ctr; double* o;
    cudaMalloc(&a, 3 * n * sizeof(double2)); cudaMemset(a, 0, 3 * n * sizeof(double2));
    cudaMalloc(&boxes, 64 * 6 * 8); cudaMemset(boxes, 0, 64 * 48);
    cudaMalloc(&out, n); cudaMalloc(&ctr, 4); cudaMalloc(&o, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    auto time = [&](const char* name, auto f) {
        f(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 20; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
        printf("%-40s %8.2f us\n", name, best * 1e3);
    };
    time("empty kernel <<<1,32>>>", [&] { empty_k<<<1, 32>>>(); });
    time("empty kernel <<<970,128>>>", [&] { empty_k<<<970, 128>>>(); });
    time("aabb 124k comps x 4 boxes (128 thr)", [&] { aabb_k<<<(n + 127) / 128, 128>>>(a, n, boxes, nb, out); });
    time("aabb 124k comps x 64 boxes (128 thr)", [&] { aabb_k<<<(n + 127) / 128, 128>>>(a, n, boxes, 64, out); });
    time("atomics: 3880 warps x 1 same addr", [&] { atomic_k<<<970, 128>>>(ctr, 1); });
    time("atomics: 3880 warps x 8 same addr", [&] { atomic_k<<<970, 128>>>(ctr, 8); });
    time("fp64 chain 1000 dep ops, 1 warp", [&] { chain_k<<<1, 32>>>(o, 500); });
    time("fp64 chain 1000 dep ops, 148x4 warps", [&] { chain_k<<<148, 128>>>(o, 500); });
    time("fp64 chain 1000 dep ops, 148x64 warps", [&] { chain_k<<<148 * 8, 256>>>(o, 500); });
    return 0;
}
