// Random-gather throughput on B200: LSU (LDG) vs TEX (tex1Dfetch) vs both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mbgather tools/microbench_gather.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned nxt(unsigned& s) { s = s * 1664525u + 1013904223u; return s; }

__global__ void g_lsu(const int4* a, int n, int per, unsigned seed, int* out) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    int acc = 0;
    for (int k = 0; k < per; ++k) { int4 v = __ldg(a + nxt(s) % (unsigned)n); acc += v.x ^ v.w; }
    if (acc == 123456789) out[0] = acc;
}
__global__ void g_tex(cudaTextureObject_t t, int n, int per, unsigned seed, int* out) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    int acc = 0;
    for (int k = 0; k < per; ++k) { int4 v = tex1Dfetch<int4>(t, nxt(s) % (unsigned)n); acc += v.x ^ v.w; }
    if (acc == 123456789) out[0] = acc;
}
__global__ void g_mix(const int4* a, cudaTextureObject_t t, int n, int per, unsigned seed, int* out) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
    int acc = 0;
    for (int k = 0; k < per; k += 2) {
        int4 v = __ldg(a + nxt(s) % (unsigned)n);
        int4 w = tex1Dfetch<int4>(t, nxt(s) % (unsigned)n);
        acc += (v.x ^ v.w) + (w.y ^ w.z);
    }
    if (acc == 123456789) out[0] = acc;
}
// lanes of a warp gather within a 2 KB window (neighbour-list-like locality)
__global__ void g_local(const int4* a, int n, int per, unsigned seed, int* out) {
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    int acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned base = nxt(s) % (unsigned)(n - 128);
        int4 v = __ldg(a + base + (nxt(l) & 127));
        acc += v.x ^ v.w;
    }
    if (acc == 123456789) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n = 2 * 1024 * 1024;   // 32 MB of int4 (16-B records), L2-resident
    int4* a; int* out;
    cudaMalloc(&a, n * sizeof(int4)); cudaMalloc(&out, 4);
    cudaMemset(a, 1, n * sizeof(int4));
    cudaResourceDesc rd = {}; rd.resType = cudaResourceTypeLinear; rd.res.linear.devPtr = a;
    rd.res.linear.desc = cudaCreateChannelDesc<int4>(); rd.res.linear.sizeInBytes = n * sizeof(int4);
    cudaTextureDesc td = {}; td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t; cudaCreateTextureObject(&t, &rd, &td, nullptr);
    int blocks = sms * 8, threads = 256, per = 256;
    double ops = (double)blocks * threads * per;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        launch(); cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        printf("%-34s %8.3f ms %8.1f G gathers/s %6.3f per clk per SM\n", name, best,
               ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) / (sms * 1.965e9));
    };
    run("LDG.128 random", [&] { g_lsu<<<blocks, threads>>>(a, n, per, 1, out); });
    run("TEX int4 random", [&] { g_tex<<<blocks, threads>>>(t, n, per, 2, out); });
    run("LDG + TEX interleaved", [&] { g_mix<<<blocks, threads>>>(a, t, n, per, 3, out); });
    run("LDG.128 warp within 2 KB", [&] { g_local<<<blocks, threads>>>(a, n, per, 4, out); });
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
