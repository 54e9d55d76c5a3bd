// Microbenchmark: fp64 global reductions (REDG.ADD.F64) on B200, to size the
// reaction-force scatter of Newton-3 kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbred tools/microbench_red.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void red_random(double* a, int n, int per_thread, unsigned seed) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    for (int k = 0; k < per_thread; ++k) {
        s = s * 1664525u + 1013904223u;
        atomicAdd(a + (s % (unsigned)n), 1.0);
    }
}

// lanes of a warp hit 32 consecutive doubles (one 256-B span); warps random
__global__ void red_coalesced(double* a, int n, int per_thread, unsigned seed) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    for (int k = 0; k < per_thread; ++k) {
        s = s * 1664525u + 1013904223u;
        unsigned base = (s % (unsigned)(n / 32)) * 32;
        atomicAdd(a + base + (threadIdx.x & 31), 1.0);
    }
}

__global__ void ld_random(const double* a, int n, int per_thread, unsigned seed, double* out) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    double acc = 0;
    for (int k = 0; k < per_thread; ++k) {
        s = s * 1664525u + 1013904223u;
        acc += __ldg(a + (s % (unsigned)n));
    }
    if (acc == -1.0) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 5 * 1024 * 1024;   // 40 MB: L2-resident like the force arrays
    double* a;
    cudaMalloc(&a, n * sizeof(double));
    cudaMemset(a, 0, n * sizeof(double));
    int blocks = sms * 8, threads = 256, per = 256;
    double ops = (double)blocks * threads * per;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        printf("%-28s %8.3f ms  %8.1f G ops/s  %6.3f ops/clk/SM @1.965GHz\n", name, best,
               ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) / (sms * 1.965e9));
    };
    run("RED.F64 random (40 MB)", [&] { red_random<<<blocks, threads>>>(a, n, per, 1); });
    run("RED.F64 warp-coalesced", [&] { red_coalesced<<<blocks, threads>>>(a, n, per, 2); });
    run("LDG.F64 random (40 MB)", [&] { ld_random<<<blocks, threads>>>(a, n, per, 3, a); });
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
