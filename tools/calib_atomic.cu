// Same-address atomic throughput on the GPU (diagnostic): `ctas` CTAs, thread 0 of each
// does `per` atomicAdds on one address (result used), timed with events.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_same(int* ctr, int per, int* sink) {
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i < per; ++i) acc += atomicAdd(ctr, 1);
        if (acc == -1) sink[0] = acc;
    }
}
__global__ void k_spread(int* ctr, int per, int* sink) {
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i < per; ++i) acc += atomicAdd(ctr + (blockIdx.x & 1023) * 32, 1);
        if (acc == -1) sink[0] = acc;
    }
}
int main() {
    int *ctr, *sink;
    cudaMalloc(&ctr, 1 << 20);
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int ctas : {1024, 8400, 34000})
        for (int which = 0; which < 2; ++which) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (which == 0) k_same<<<ctas, 128>>>(ctr, 2, sink);
                else k_spread<<<ctas, 128>>>(ctr, 2, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep == 2) printf("%s ctas %d x 2 atomics: %.1f us (%.2f ns per atomic)\n", which ? "spread" : "same  ", ctas, ms * 1e3, ms * 1e6 / (ctas * 2));
            }
        }
    return 0;
}
