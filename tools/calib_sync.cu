// Cost of a grid-wide barrier (cooperative launch) vs a kernel boundary (profiling helper).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void syncs_k(int n, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < n; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = n;
}
__global__ void one_k(int* sink) { if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1; }
int main() {
    int* sink; cudaMalloc(&sink, 4);
    int dev = 0, sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int per : {1, 4}) {
        for (int n : {0, 10, 100}) {
            void* args[] = {&n, &sink};
            float best = 1e9, ms;
            for (int r = 0; r < 10; ++r) {
                cudaEventRecord(a);
                cudaLaunchCooperativeKernel((void*)syncs_k, dim3(sms * per), dim3(128), args, 0, 0);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
            }
            printf("cooperative grid %d x 128: %3d grid.sync() -> %.2f us\n", sms * per, n, best * 1e3);
        }
    }
    // back-to-back kernels in one graph
    for (int n : {1, 10, 100}) {
        cudaStream_t st; cudaStreamCreate(&st);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < n; ++i) one_k<<<592, 128, 0, st>>>(sink);
        cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
        float best = 1e9, ms;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(a, st); cudaGraphLaunch(ge, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
        }
        printf("graph of %3d kernels <<<592,128>>> -> %.2f us\n", n, best * 1e3);
    }
    return 0;
}
