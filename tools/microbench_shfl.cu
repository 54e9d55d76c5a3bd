// Do warp shuffles compete with shared-memory loads for the L1TEX/LSU data
// pipe?  (Design question for a walk that moves part of its j-data through
// SHFL instead of random LDS.)  Kernels: random LDS.64 x3 per iteration;
// SHFL.IDX x6 (three doubles) per iteration; both together.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mbshfl tools/microbench_shfl.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned nxt(unsigned& s) {
    s = s * 1664525u + 1013904223u;
    unsigned x = s;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
constexpr int W = 2048;

template <bool LDS, bool SHFL>
__global__ void k(int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W], z[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; z[i] = 3 * i; }
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double a = threadIdx.x, b = 2.0 * threadIdx.x, c = 3.0 * threadIdx.x;
    double acc = 0;
    int lane = threadIdx.x & 31;
    for (int it = 0; it < per; ++it) {
        unsigned r = nxt(l);
        if (LDS) {
            unsigned j = r % W;
            acc += x[j] * y[j] + z[j];
        }
        if (SHFL) {
            int src = (lane + (r & 31)) & 31;
            double p = __shfl_sync(0xffffffffu, a, src), q = __shfl_sync(0xffffffffu, b, src),
                   s = __shfl_sync(0xffffffffu, c, src);
            acc += p * q + s;
            a += 1.0;
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    int threads = 512, per = 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        int b = 4 * sms;
        launch(b);
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch(b);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double warp_iters = (double)b * threads / 32 * per;
        printf("%-36s %8.3f ms  %6.3f warp-iterations per clk per SM\n", name, best,
               warp_iters / (best * 1e-3) / (sms * 1.965e9));
    };
    run("3 LDS.64 random", [=](int b) { k<true, false><<<b, threads>>>(per, 7, out); });
    run("6 SHFL.IDX (3 doubles)", [=](int b) { k<false, true><<<b, threads>>>(per, 7, out); });
    run("3 LDS.64 + 6 SHFL.IDX", [=](int b) { k<true, true><<<b, threads>>>(per, 7, out); });
    return 0;
}
