// Can the texture path add gather bandwidth next to shared memory?  The tiled
// Verlet walk is bound by L1TEX *LSU* data-pipe wavefronts (three random
// LDS.64 per list entry, ~5.3 wavefronts each).  Texture fetches travel the
// TEX data pipe; if that pipe is independent, moving one of the three
// coordinate gathers to tex1Dfetch (from an L1-resident global copy) could
// raise the walk's ceiling.  Each kernel: per iteration one random 24-byte
// record (x, y, z as doubles) per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mbtex tools/microbench_tex.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned nxt(unsigned& s) {
    s = s * 1664525u + 1013904223u;
    unsigned x = s;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

constexpr int W = 2048;   // window rows (the walk's 2,048-row windows)

// baseline: x, y, z from shared memory (3 random LDS.64)
__global__ void k_smem3(int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W], z[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; z[i] = 3 * i; }
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = nxt(l) % W;
        acc += x[j] * y[j] + z[j];
    }
    if (acc == 1.2345) out[0] = acc;
}

// x, y from shared memory, z through the texture path (per-CTA slice of a
// global array, L1-resident)
__global__ void k_smem2_tex1(cudaTextureObject_t tz, int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; }
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    const int base = (blockIdx.x % 64) * W;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = nxt(l) % W;
        int2 v = tex1Dfetch<int2>(tz, base + j);
        acc += x[j] * y[j] + __hiloint2double(v.y, v.x);
    }
    if (acc == 1.2345) out[0] = acc;
}

// x from shared memory, y and z through the texture path
__global__ void k_smem1_tex2(cudaTextureObject_t t4, int per, unsigned seed, double* out) {
    __shared__ double x[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) x[i] = i;
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    const int base = (blockIdx.x % 64) * W;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = nxt(l) % W;
        int4 v = tex1Dfetch<int4>(t4, base + j);   // {y, z} as one 16-byte texel
        acc += x[j] * __hiloint2double(v.y, v.x) + __hiloint2double(v.w, v.z);
    }
    if (acc == 1.2345) out[0] = acc;
}

// z through LDG (LSU path, L1-cached) instead of texture: the control
__global__ void k_smem2_ldg1(const double* gz, int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; }
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    const double* zb = gz + (blockIdx.x % 64) * W;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = nxt(l) % W;
        acc += x[j] * y[j] + __ldg(zb + j);
    }
    if (acc == 1.2345) out[0] = acc;
}

// all three through the texture path
__global__ void k_tex3(cudaTextureObject_t tz, cudaTextureObject_t t4, int per, unsigned seed, double* out) {
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    const int base = (blockIdx.x % 64) * W;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = nxt(l) % W;
        int2 a = tex1Dfetch<int2>(tz, base + j);
        int4 v = tex1Dfetch<int4>(t4, base + j);
        acc += __hiloint2double(a.y, a.x) * __hiloint2double(v.y, v.x) + __hiloint2double(v.w, v.z);
    }
    if (acc == 1.2345) out[0] = acc;
}

static cudaTextureObject_t make_tex(void* p, size_t bytes, cudaChannelFormatDesc d) {
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = p;
    rd.res.linear.desc = d;
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    cudaCreateTextureObject(&t, &rd, &td, nullptr);
    return t;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int n = 64 * W;
    double* gz;
    double2* g4;
    cudaMalloc(&gz, n * sizeof(double));
    cudaMalloc(&g4, n * sizeof(double2));
    cudaMemset(gz, 0, n * sizeof(double));
    cudaMemset(g4, 0, n * sizeof(double2));
    cudaTextureObject_t tz = make_tex(gz, n * sizeof(double), cudaCreateChannelDesc<int2>());
    cudaTextureObject_t t4 = make_tex(g4, n * sizeof(double2), cudaCreateChannelDesc<int4>());
    int threads = 512, per = 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* name, int blocks, auto launch) {
        launch(blocks);
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            launch(blocks);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double ops = (double)blocks * threads * per;
        printf("%-44s %8.3f ms %6.3f records per clk per SM  (%s)\n", name, best,
               ops / (best * 1e-3) / (sms * 1.965e9), cudaGetErrorString(cudaGetLastError()));
    };
    int b = 4 * sms;
    run("smem x,y,z (3 LDS.64)", b, [=](int bl) { k_smem3<<<bl, threads>>>(per, 7, out); });
    run("smem x,y + tex z", b, [=](int bl) { k_smem2_tex1<<<bl, threads>>>(tz, per, 7, out); });
    run("smem x + tex {y,z} (16-B texel)", b, [=](int bl) { k_smem1_tex2<<<bl, threads>>>(t4, per, 7, out); });
    run("smem x,y + LDG z (control)", b, [=](int bl) { k_smem2_ldg1<<<bl, threads>>>(gz, per, 7, out); });
    run("tex x + tex {y,z}", b, [=](int bl) { k_tex3<<<bl, threads>>>(tz, t4, per, 7, out); });
    return 0;
}
