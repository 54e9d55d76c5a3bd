// Shared-memory building blocks for a Newton-3 Verlet walk on B200:
// random 32-B record gathers from shared memory and fp64 shared atomics.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/mbsmem tools/microbench_smem.cu
#include <cstdio>
#include <cuda_runtime.h>

// LCG step + finaliser: the raw LCG's low bits form a per-lane permutation
// modulo 16 (bank-conflict-free by accident), so hash before use
__device__ __forceinline__ unsigned nxt(unsigned& s) {
    s = s * 1664525u + 1013904223u;
    unsigned x = s;
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

constexpr int W = 768;    // records per CTA window (static smem <= 48 KB: 24 KB positions + 18 KB forces)

// lanes pick independent random records in the window (local = within 128)
template <bool LOCAL>
__device__ __forceinline__ unsigned pick(unsigned& s, unsigned& l) {
    if (LOCAL) return (nxt(s) % (W - 128)) + (nxt(l) & 127);
    return nxt(l) % W;
}

template <bool LOCAL>
__global__ void s_gather(int per, unsigned seed, double* out) {
    __shared__ double4 p[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) p[i] = make_double4(i, 2 * i, 3 * i, 0);
    __syncthreads();
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        double4 v = p[pick<LOCAL>(s, l)];
        acc += v.x + v.y + v.z;
    }
    if (acc == 1.2345) out[0] = acc;
}

template <bool LOCAL>
__global__ void s_gather_soa(int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W], z[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; z[i] = 3 * i; }
    __syncthreads();
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = pick<LOCAL>(s, l);
        acc += x[j] + y[j] + z[j];
    }
    if (acc == 1.2345) out[0] = acc;
}

// {x,y} as one 16-B record + z as an 8-B one: 2 loads per gather instead of 3
template <bool LOCAL>
__global__ void s_gather_xy(int per, unsigned seed, double* out) {
    __shared__ double2 xy[W];
    __shared__ double z[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { xy[i] = make_double2(i, 2 * i); z[i] = 3 * i; }
    __syncthreads();
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = pick<LOCAL>(s, l);
        double2 v = xy[j];
        acc += v.x + v.y + z[j];
    }
    if (acc == 1.2345) out[0] = acc;
}

// MODE 0: random rows; 1: bank class of row = (lane + k) mod 16 (conflict-free
// per half-warp); 2: class (lane + k/4 + drift) mod 16 with a random per-lane
// drift of 0..3 steps -- what a list sorted by (class - lane) mod 16 gives
template <int MODE>
__global__ void s_gather_cls(int per, unsigned seed, double* out) {
    __shared__ double x[W], y[W], z[W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { x[i] = i; y[i] = 2 * i; z[i] = 3 * i; }
    __syncthreads();
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    int lane = threadIdx.x & 31;
    int drift = nxt(l) & 3;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned r = nxt(l) % (W / 16);
        unsigned cls = MODE == 0 ? (nxt(l) & 15) : MODE == 1 ? ((lane + k) & 15) : ((lane + (k + drift) / 4) & 15);
        unsigned j = r * 16 + cls;
        acc += x[j] + y[j] + z[j];
    }
    if (acc == 1.2345) out[0] = acc;
}

template <bool LOCAL>
__global__ void s_atomic(int per, unsigned seed, double* out) {
    __shared__ double f[3 * W];
    for (int i = threadIdx.x; i < 3 * W; i += blockDim.x) f[i] = 0;
    __syncthreads();
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    for (int k = 0; k < per; ++k) {
        unsigned j = pick<LOCAL>(s, l);
        atomicAdd(&f[3 * j], 1.0);
        atomicAdd(&f[3 * j + 1], 2.0);
        atomicAdd(&f[3 * j + 2], 3.0);
    }
    __syncthreads();
    if (f[threadIdx.x] == 1.2345) out[0] = 1;
}

// the N3L pattern: gather j + three atomics into j
template <bool LOCAL>
__global__ void s_n3l(int per, unsigned seed, double* out) {
    __shared__ double4 p[W];
    __shared__ double f[3 * W];
    for (int i = threadIdx.x; i < W; i += blockDim.x) { p[i] = make_double4(i, 2 * i, 3 * i, 0); }
    for (int i = threadIdx.x; i < 3 * W; i += blockDim.x) f[i] = 0;
    __syncthreads();
    unsigned s = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) / 32 * 2654435761u;
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        unsigned j = pick<LOCAL>(s, l);
        double4 v = p[j];
        acc += v.x;
        atomicAdd(&f[3 * j], v.x);
        atomicAdd(&f[3 * j + 1], v.y);
        atomicAdd(&f[3 * j + 2], v.z);
    }
    __syncthreads();
    if (f[threadIdx.x] == 1.2345 || acc == 1.2345) out[0] = 1;
}

// global random 32-B gathers over an L2-resident array, for comparison
__global__ void g_gather(const double4* a, int n, int per, unsigned seed, double* out) {
    unsigned l = seed ^ (blockIdx.x * blockDim.x + threadIdx.x) * 747796405u;
    double acc = 0;
    for (int k = 0; k < per; ++k) {
        const double4* q = a + nxt(l) % (unsigned)n;
        double4 v;
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(q));
        acc += v.x + v.y + v.z;
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int n = 1 << 20;
    double4* a;
    cudaMalloc(&a, n * sizeof(double4));
    cudaMemset(a, 0, n * sizeof(double4));
    int threads = 512, per = 512;
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
        printf("%-36s %8.3f ms %8.1f G ops/s %6.3f per clk per SM  (%s)\n", name, best,
               ops / (best * 1e-3) / 1e9, ops / (best * 1e-3) / (sms * 1.965e9),
               cudaGetErrorString(cudaGetLastError()));
    };
    // one window per CTA; 1 CTA/SM for the 140 KB kernels, 2 for the small ones
    auto big = [&](auto k) { return [=](int b) { k<<<b, threads>>>(per, 7, out); }; };
    int b1 = 4 * sms, b2 = 4 * sms;
    run("smem gather double4 random", b2, big(s_gather<false>));
    run("smem gather double4 local-128", b2, big(s_gather<true>));
    run("smem gather 3x double random", b2, big(s_gather_soa<false>));
    run("smem gather 3x double local-128", b2, big(s_gather_soa<true>));
    run("smem gather double2 xy + double z random", b2, big(s_gather_xy<false>));
    run("smem gather double2 xy + double z local", b2, big(s_gather_xy<true>));
    run("smem 3x double, random class", b2, big(s_gather_cls<0>));
    run("smem 3x double, rotated class", b2, big(s_gather_cls<1>));
    run("smem 3x double, rotated+drift", b2, big(s_gather_cls<2>));
    run("smem 3x atomicAdd f64 random", b2, big(s_atomic<false>));
    run("smem 3x atomicAdd f64 local-128", b2, big(s_atomic<true>));
    run("smem gather + 3 atomics random", b1, big(s_n3l<false>));
    run("smem gather + 3 atomics local-128", b1, big(s_n3l<true>));
    run("global LDG double4 random (32 MB)", 4 * sms, [=](int b) { g_gather<<<b, threads>>>(a, n, per, 9, out); });
    return 0;
}
