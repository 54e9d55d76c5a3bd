// Shared-memory tiled Verlet-list walk (VL-List_Iter-NoN3L-{AoS,SoA} force).
//
// Reference: vl_force_aos/_soa (kernels.py:730-818) over the lists of
// VerletListState (containers.py:343-375); the pair sets and counts are those
// of vl.cu's row-space lists, which this file only re-indexes.
//
// Why: the row-space walk (vl.cu) gathers every neighbour position from
// global memory, one random 32-byte sector per lane and entry; on B200 that
// saturates the L1TEX wavefront rate at ~1 record / clock / SM
// (profiles/round1_ncu_vl_force_bench.txt, tools/microbench_smem.cu).  Random
// 8-byte reads from shared memory sustain ~1.8 records / clock / SM.  So:
//
//  * Tiles.  Owned cells are cut into 2 x 2 cell columns x a z-run of TZ
//    cells (TZ from the mean density so the window fits).  The window of a
//    tile -- the 4 x 4 columns around it over z0-1 .. z1, i.e. 16 contiguous
//    row ranges of the cell-sorted row space -- holds every neighbour of
//    every tile row (CSF-1 grid, 26-cell stencil).
//  * Lists.  At rebuild, each tile row's list is rewritten as uint16
//    window-local indices in 4-entry groups (8 bytes per lane and group,
//    a warp's group loads are 256 contiguous bytes), streamed evict-first.
//  * Walk.  Persistent CTAs take tiles from an atomic counter, stage the
//    window's unwrapped positions (x, y, z component arrays, types) in
//    shared memory with coalesced loads, and walk the lists one thread per
//    row with the batched fast reciprocal of vl.cu.
//  * Overflow.  Tiles whose window exceeds the shared-memory budget
//    (clustered inputs) are walked by vl.cu's global-gather kernel, selected
//    row by row through a mask.
#include <cstdio>
#include <vector>

#include "device.cuh"

namespace mdg {

constexpr int kTX = 2, kTY = 2;
constexpr int kRanges = (kTX + 2) * (kTY + 2);
constexpr int kSegs = kTX * kTY;
constexpr int kWinRows = 2048;        // 48 KB of positions (+ 2 KB types) per CTA

struct TileDesc {
    int x0, y0, z0, z1;
    int ni, wrows, big, pad0;
    int wstart[kRanges];
    int woff[kRanges + 1];
    int istart[kSegs];
    int ioff[kSegs + 1];
    int pad1[2];
};
static_assert(sizeof(TileDesc) % 16 == 0, "TileDesc is copied as int4");
constexpr int kDescInts = sizeof(TileDesc) / 4;

struct TilePlan {
    int ngx, ngy, nzt, tz;
};

__global__ void vlt_desc_kernel(GridView gv, TilePlan tp, int ntiles, int cap4, int budget,
                                TileDesc* __restrict__ desc, int* __restrict__ tsize,
                                int* __restrict__ nbig) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    int gz = t % tp.nzt, g2 = t / tp.nzt;
    int gy = g2 % tp.ngy, gx = g2 / tp.ngy;
    TileDesc d;
    d.x0 = gv.H0 + gx * kTX;
    d.y0 = gv.H1 + gy * kTY;
    d.z0 = gv.H2 + gz * tp.tz;
    d.z1 = min(d.z0 + tp.tz, gv.H2 + gv.S2);
    int tx = min(kTX, gv.H0 + gv.S0 - d.x0), ty = min(kTY, gv.H1 + gv.S1 - d.y0);
    int za = max(d.z0 - 1, 0), zb = min(d.z1, gv.D2 - 1);
    int off = 0;
    for (int a = 0; a < kTX + 2; ++a)
        for (int b = 0; b < kTY + 2; ++b) {
            int R = a * (kTY + 2) + b, x = d.x0 - 1 + a, y = d.y0 - 1 + b;
            bool in = a <= tx + 1 && b <= ty + 1 && x >= 0 && x < gv.D0 && y >= 0 && y < gv.D1;
            // rounded out to multiples of 4 rows: every component range is
            // then a 32-byte aligned 1-D bulk copy (the extra rows are never
            // referenced by a list)
            int ws = in ? gv.start[gv.flat(x, y, za)] & ~3 : 0;
            int we = in ? (gv.start[gv.flat(x, y, zb) + 1] + 3) & ~3 : 0;
            d.wstart[R] = ws;
            d.woff[R] = off;
            off += we - ws;
        }
    d.woff[kRanges] = off;
    int io = 0;
    for (int a = 0; a < kTX; ++a)
        for (int b = 0; b < kTY; ++b) {
            int C = a * kTY + b;
            bool in = a < tx && b < ty;
            int x = d.x0 + a, y = d.y0 + b;
            int is = in ? gv.start[gv.flat(x, y, d.z0)] : 0;
            int ie = in ? gv.start[gv.flat(x, y, d.z1 - 1) + 1] : 0;
            d.istart[C] = is;
            d.ioff[C] = io;
            io += ie - is;
        }
    d.ioff[kSegs] = io;
    d.ni = io;
    d.wrows = off;
    d.big = off > budget || off > 65536;
    d.pad0 = 0;
    d.pad1[0] = d.pad1[1] = 0;
    desc[t] = d;
    tsize[t] = d.big ? 0 : (io + 31) / 32 * 32;   // list slots (rows padded to 32); x cap4 entries
    if (d.big) atomicAdd(nbig, 1);
}

__device__ __forceinline__ void load_desc(const TileDesc* __restrict__ desc, int t, TileDesc& d) {
    const int4* src = reinterpret_cast<const int4*>(desc + t);
    int4* dst = reinterpret_cast<int4*>(&d);
    for (int k = threadIdx.x; k < kDescInts / 4; k += blockDim.x) dst[k] = src[k];
}

// tile-local row q -> (row, window index of the row).  Branch-free: a
// data-dependent loop here splits the warp (lanes in different segments leave
// it on different trips and never reconverge before the list walk, which then
// runs once per lane group).
__device__ __forceinline__ int tile_row(const TileDesc& d, int q, int& li) {
    int C = 0;
#pragma unroll
    for (int k = 1; k < kSegs; ++k) C += q >= d.ioff[k];
    int r = d.istart[C] + (q - d.ioff[C]);
    int R = (C / kTY + 1) * (kTY + 2) + (C % kTY + 1);
    li = d.woff[R] + (r - d.wstart[R]);
    return r;
}

// Tiled list build (rebuild time).  One CTA per tile stages the window's fp32
// build positions in shared memory; each thread scans its row's nine window
// z-runs (cells cz-1 .. cz+1 of the 3 x 3 neighbouring columns, i.e. the
// 26-cell stencil + own cell, in ascending row order like vl.cu) and writes
// uint16 window indices straight into the tile list, four at a time (a
// 64-bit register collects a group, one 8-byte store flushes it; the last
// group's unused slots stay zero, which is the padding the walk expects).
// Membership is the reference's r^2 <= ell^2 on the fp64 build positions
// (kernels.py:848), decided in fp32 where the rounding bound of vl.cu's build
// proves it and in fp64 otherwise.  Lanes of rows in one cell scan the same
// candidates, so the shared-memory reads are broadcasts.
// packed fp32 pairs (FADD2 / FMUL2 / FFMA2, sm_100a)
__device__ __forceinline__ unsigned long long pack2(float x) {
    unsigned u = __float_as_uint(x);
    return (unsigned long long)u << 32 | u;
}
__device__ __forceinline__ unsigned long long f2sub(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2mul(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}

constexpr int kBuildThreadsT = 256;
constexpr int kMaxTZ = 48;

template <int NT>
__global__ void __launch_bounds__(NT) vlt_build_kernel(
    GridView gv, const TileDesc* __restrict__ desc, const int* __restrict__ tbase,
    const float4* __restrict__ b32, const double4* __restrict__ bpos,
    const unsigned* __restrict__ maxabs_bits, double ell2, int cap, int cap4,
    uint16_t* __restrict__ tl, int* __restrict__ tcnt, int* __restrict__ maxcnt, int zsorted) {
    __shared__ __align__(16) TileDesc d;
    __shared__ int cs[kRanges][kMaxTZ + 4];
    // the window's fp32 build positions as row pairs (2k, 2k+1): {x, x', y, y'}
    // and {z, z'}, so one FADD2 / FMUL2 / FFMA2 tests two candidates; +64
    // rows: the 32-wide scan starts at an even row and reads past a run's end
    __shared__ ulonglong2 wxy[(kWinRows + 64) / 2];
    __shared__ unsigned long long wz[(kWinRows + 64) / 2];
    load_desc(desc, blockIdx.x, d);
    __syncthreads();
    if (d.big) return;
    const int za = max(d.z0 - 1, 0), zb = min(d.z1, gv.D2 - 1), nz = zb - za + 1;
    const int tx = min(kTX, gv.H0 + gv.S0 - d.x0), ty = min(kTY, gv.H1 + gv.S1 - d.y0);
    // cs[R][k]: window index of the first row of cell za + k in range R
    for (int idx = threadIdx.x; idx < kRanges * (nz + 1); idx += blockDim.x) {
        int R = idx / (nz + 1), k = idx % (nz + 1);
        int a = R / (kTY + 2), b = R % (kTY + 2), x = d.x0 - 1 + a, y = d.y0 - 1 + b;
        bool in = a <= tx + 1 && b <= ty + 1 && x >= 0 && x < gv.D0 && y >= 0 && y < gv.D1;
        cs[R][k] = in ? gv.start[gv.flat(x, y, za) + k] - d.wstart[R] + d.woff[R] : 0;
    }
    int wrows = d.woff[kRanges];
    float* fxy = reinterpret_cast<float*>(wxy);
    float* fz = reinterpret_cast<float*>(wz);
    for (int w = threadIdx.x; w < wrows + 64; w += blockDim.x) {
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        if (w < wrows) {
            int lo = 0;
#pragma unroll
            for (int R = 1; R < kRanges; ++R) lo += d.woff[R] <= w;
            p = b32[d.wstart[lo] + (w - d.woff[lo])];
        }
        fxy[4 * (w >> 1) + (w & 1)] = p.x;
        fxy[4 * (w >> 1) + 2 + (w & 1)] = p.y;
        fz[2 * (w >> 1) + (w & 1)] = p.z;
    }
    __syncthreads();
    const double u = 5.9604644775390625e-08;   // 2^-24
    double X = (double)__uint_as_float(*maxabs_bits) * (1.0 + 4.0 * u);
    double ell = sqrt(ell2);
    double eta = 2.0 * u * X + 2.0 * u * ell;
    double B = 3.4641016151377544 * eta * ell + 3.0 * eta * eta + 3.0 * u * ell2;
    const float flo = __double2float_rd(ell2 - 2.0 * B), fhi = __double2float_ru(ell2 + 2.0 * B);
    // r2 <= f  <=>  bits(r2) - bits(f) - 1 < 0 (both non-negative floats)
    const int flo_i = __float_as_int(flo) + 1, fhi_i = __float_as_int(fhi) + 1;
    // z-window: rows of a column run are z-ordered (z-sorted cells, the VL
    // grid's sort_by_z), so the candidates within ell in z are a contiguous
    // sub-run; fp32 coordinates are within u|x| of fp64, hence the 2 eta pad
    const double zpad = ell + 2.0 * eta;
    // tbase counts list slots (padded rows): 32-bit even when the entries
    // (slots x cap4, BASELINE config 5: ~5.4 G) are not
    const int slot0 = tbase[blockIdx.x];
    const size_t base = (size_t)slot0 * cap4;
    for (int q = threadIdx.x; q < d.ni; q += blockDim.x) {
        int C = 0;
#pragma unroll
        for (int k = 1; k < kSegs; ++k) C += q >= d.ioff[k];
        int r = d.istart[C] + (q - d.ioff[C]);
        int a = C / kTY, b = C % kTY;
        int Rown = (a + 1) * (kTY + 2) + (b + 1);
        int li = d.woff[Rown] + (r - d.wstart[Rown]);
        int cx, cy, cz;
        gv.decode(gv.row_cell[r], cx, cy, cz);
        int k0 = max(cz - 1 - za, 0), k1 = min(cz + 2 - za, nz);
        const float qx = fxy[4 * (li >> 1) + (li & 1)], qy = fxy[4 * (li >> 1) + 2 + (li & 1)],
                    qz = fz[2 * (li >> 1) + (li & 1)];
        const unsigned long long qx2 = pack2(qx), qy2 = pack2(qy), qz2 = pack2(qz);
        const float zlo = __double2float_rd((double)qz - zpad), zhi = __double2float_ru((double)qz + zpad);
        // groups of 4 uint16 entries per lane, 32 lanes of a 32-row block side
        // by side; (glo, ghi) holds the last 4 entries, newest in the top 16
        // bits (two byte permutes per entry), and every 4th entry stores it
        uint2* op = reinterpret_cast<uint2*>(tl + base + (size_t)(q >> 5) * 32 * cap4 + (q & 31) * 4);
        unsigned glo = 0, ghi = 0;
        int c = 0;
        for (int dx = 0; dx < 3; ++dx)
            for (int dy = 0; dy < 3; ++dy) {
                int R = (a + dx) * (kTY + 2) + (b + dy);
                int s0 = cs[R][k0], e0 = cs[R][k1];
                int gR = d.wstart[R] - d.woff[R];   // global row of window index l: gR + l
                if (zsorted) {
                    int lo = s0, hi = e0;
                    while (lo < hi) {   // first row with z >= zlo
                        int mid = (lo + hi) >> 1;
                        if (fz[2 * (mid >> 1) + (mid & 1)] < zlo) lo = mid + 1; else hi = mid;
                    }
                    int s1 = lo;
                    hi = e0;
                    while (lo < hi) {   // first row with z > zhi
                        int mid = (lo + hi) >> 1;
                        if (fz[2 * (mid >> 1) + (mid & 1)] <= zhi) lo = mid + 1; else hi = mid;
                    }
                    s0 = s1;
                    e0 = lo;
                }
                for (int l0 = s0 & ~1; l0 < e0; l0 += 32) {
                    // 32 candidates (from an even row) -> two bit masks
                    // (certainly in / maybe in), built first candidate
                    // highest: r2 <= f is the sign of r2 - f - 1 on the bits
                    // of non-negative floats, shifted in by a funnel shift
                    unsigned a_in = 0, a_mb = 0;
                    const int span = min(32, e0 - l0);
                    const int nb = (span + 7) >> 3;
#pragma unroll 1
                    for (int t0 = 0; t0 < 8 * nb; t0 += 8) {   // 8-candidate batches up to the run's end
#pragma unroll
                        for (int t = 0; t < 8; t += 2) {
                            const int h = (l0 + t0 + t) >> 1;
                            ulonglong2 pxy = wxy[h];
                            unsigned long long ex = f2sub(qx2, pxy.x), ey = f2sub(qy2, pxy.y),
                                               ez = f2sub(qz2, wz[h]);
                            unsigned long long r2 = f2fma(ez, ez, f2fma(ey, ey, f2mul(ex, ex)));
                            int r0 = (int)(unsigned)r2, r1 = (int)(unsigned)(r2 >> 32);
                            a_in = __funnelshift_l((unsigned)(r0 - flo_i), a_in, 1);
                            a_mb = __funnelshift_l((unsigned)(r0 - fhi_i), a_mb, 1);
                            a_in = __funnelshift_l((unsigned)(r1 - flo_i), a_in, 1);
                            a_mb = __funnelshift_l((unsigned)(r1 - fhi_i), a_mb, 1);
                        }
                    }
                    unsigned m_in = __brev(a_in) >> (32 - 8 * nb), m_mb = __brev(a_mb) >> (32 - 8 * nb);
                    unsigned valid = span >= 32 ? 0xffffffffu : (1u << span) - 1u;
                    if (l0 < s0) valid &= ~1u;   // the even row before an odd run start
                    unsigned self = (li >= l0 && li < l0 + 32) ? 1u << (li - l0) : 0u;
                    valid &= ~self;
                    m_in &= valid;
                    unsigned m_bd = m_mb & valid & ~m_in;   // borderline: exact fp64 test
                    if (m_bd) {
                        double4 pi = ldg256(bpos + r);
                        while (m_bd) {
                            int t = __ffs(m_bd) - 1;
                            m_bd &= m_bd - 1;
                            double4 pj = ldg256(bpos + gR + l0 + t);
                            double ex = pi.x - pj.x, ey = pi.y - pj.y, ez = pi.z - pj.z;
                            if (ex * ex + ey * ey + ez * ez <= ell2) m_in |= 1u << t;
                        }
                    }
                    while (m_in) {   // ascending, like the scan order
                        int t = __ffs(m_in) - 1;
                        m_in &= m_in - 1;
                        MDG_DCHECK(l0 + t >= 0 && l0 + t < wrows && l0 + t != li);
                        glo = __byte_perm(glo, ghi, 0x5432);
                        ghi = __byte_perm(ghi, (unsigned)(l0 + t), 0x5432);
                        ++c;
                        if ((c & 3) == 0 && c <= cap4) op[(size_t)((c >> 2) - 1) * 32] = make_uint2(glo, ghi);
                    }
                }
            }
        if ((c & 3) && c < cap4) {   // the last group, its unused slots zero (the walk's padding)
            unsigned long long g = ((unsigned long long)ghi << 32 | glo) >> (16 * (4 - (c & 3)));
            op[(size_t)(c >> 2) * 32] = make_uint2((unsigned)g, (unsigned)(g >> 32));
        }
        tcnt[slot0 + q] = min(c, cap);
        if (c > cap) atomicMax(maxcnt, c);
    }
    // the tile's padding slots (its last 32-row block): empty lists, written
    // here instead of by a memset of every slot before the build
    for (int q = d.ni + threadIdx.x; q < ((d.ni + 31) & ~31); q += blockDim.x) tcnt[slot0 + q] = 0;
}

// Warp-converged tiled build (MDG_VLT_BUILD=2; measured slower than the
// lane-per-row scan above, 0.725 against 0.475 ms on config 2, and kept as
// the measured alternative).  The lane-per-row scan diverges: the lanes of a
// warp scan z-windows of different lengths and extract different numbers of
// entries, so most of its instructions run with a fraction of the lanes
// (426 M warp instructions per config-2 build, issue-bound,
// profiles/round1_ncu_vlt_build.txt).  Here a warp takes 32 rows of ONE
// column segment of the tile -- they share the nine neighbour column runs --
// and scans the union of their z-windows: every lane tests the same candidate
// (a shared-memory broadcast) against its own row, so the scan never
// diverges; only the per-lane extraction does.  The union window is about
// twice a row's own window; the membership test decides, so the lists are
// those of the lane-per-row scan entry for entry.
__global__ void __launch_bounds__(kBuildThreadsT) vlt_build_warp_kernel(
    GridView gv, const TileDesc* __restrict__ desc, const int* __restrict__ tbase,
    const float4* __restrict__ b32, const double4* __restrict__ bpos,
    const unsigned* __restrict__ maxabs_bits, double ell2, int cap, int cap4,
    uint16_t* __restrict__ tl, int* __restrict__ tcnt, int* __restrict__ maxcnt, int zsorted) {
    __shared__ __align__(16) TileDesc d;
    __shared__ int cs[kRanges][kMaxTZ + 4];
    __shared__ float4 w32[kWinRows + 32];
    load_desc(desc, blockIdx.x, d);
    __syncthreads();
    if (d.big) return;
    const int za = max(d.z0 - 1, 0), zb = min(d.z1, gv.D2 - 1), nz = zb - za + 1;
    const int tx = min(kTX, gv.H0 + gv.S0 - d.x0), ty = min(kTY, gv.H1 + gv.S1 - d.y0);
    for (int idx = threadIdx.x; idx < kRanges * (nz + 1); idx += blockDim.x) {
        int R = idx / (nz + 1), k = idx % (nz + 1);
        int a = R / (kTY + 2), b = R % (kTY + 2), x = d.x0 - 1 + a, y = d.y0 - 1 + b;
        bool in = a <= tx + 1 && b <= ty + 1 && x >= 0 && x < gv.D0 && y >= 0 && y < gv.D1;
        cs[R][k] = in ? gv.start[gv.flat(x, y, za) + k] - d.wstart[R] + d.woff[R] : 0;
    }
    int wrows = d.woff[kRanges];
    for (int w = threadIdx.x; w < wrows + 32; w += blockDim.x) {
        if (w >= wrows) {
            w32[w] = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
        }
        int lo = 0;
#pragma unroll
        for (int R = 1; R < kRanges; ++R) lo += d.woff[R] <= w;
        w32[w] = b32[d.wstart[lo] + (w - d.woff[lo])];
    }
    __syncthreads();
    // the fp32 membership bounds of vlt_build_kernel
    const double u = 5.9604644775390625e-08;   // 2^-24
    double X = (double)__uint_as_float(*maxabs_bits) * (1.0 + 4.0 * u);
    double ell = sqrt(ell2);
    double eta = 2.0 * u * X + 2.0 * u * ell;
    double B = 3.4641016151377544 * eta * ell + 3.0 * eta * eta + 3.0 * u * ell2;
    const float flo = __double2float_rd(ell2 - 2.0 * B), fhi = __double2float_ru(ell2 + 2.0 * B);
    const double zpad = ell + 2.0 * eta;
    const int slot0 = tbase[blockIdx.x];
    const size_t base = (size_t)slot0 * cap4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int tstart[kSegs + 1];
    tstart[0] = 0;
#pragma unroll
    for (int C = 0; C < kSegs; ++C) tstart[C + 1] = tstart[C] + (d.ioff[C + 1] - d.ioff[C] + 31) / 32;
    for (int task = warp; task < tstart[kSegs]; task += kBuildThreadsT / 32) {
        int C = 0;
#pragma unroll
        for (int k = 1; k < kSegs; ++k) C += task >= tstart[k];
        const int q = d.ioff[C] + (task - tstart[C]) * 32 + lane;
        const bool valid = q < d.ioff[C + 1];
        const int a = C / kTY, b = C % kTY;
        const int Rown = (a + 1) * (kTY + 2) + (b + 1);
        int r = 0, li = -64, cz = 0;
        float4 qi = make_float4(0.f, 0.f, 0.f, 0.f);
        float zlo = 3.0e38f, zhi = -3.0e38f;
        int czlo = 1 << 30, czhi = -(1 << 30);
        if (valid) {
            r = d.istart[C] + (q - d.ioff[C]);
            li = d.woff[Rown] + (r - d.wstart[Rown]);
            int cx, cy;
            gv.decode(gv.row_cell[r], cx, cy, cz);
            qi = w32[li];
            czlo = czhi = cz;
            zlo = __double2float_rd((double)qi.z - zpad);
            zhi = __double2float_ru((double)qi.z + zpad);
        }
        // the warp's union: cells and z-window
        czlo = __reduce_min_sync(0xffffffffu, czlo);
        czhi = __reduce_max_sync(0xffffffffu, czhi);
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            zlo = fminf(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
            zhi = fmaxf(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
        }
        const int k0 = max(czlo - 1 - za, 0), k1 = min(czhi + 2 - za, nz);
        // groups of 4 uint16 entries per lane, 32 lanes of a 32-row block side
        // by side; (glo, ghi) holds the last 4 entries, newest in the top 16
        // bits (two byte permutes per entry), and every 4th entry stores it
        uint2* op = reinterpret_cast<uint2*>(tl + base + (size_t)(q >> 5) * 32 * cap4 + (q & 31) * 4);
        unsigned glo = 0, ghi = 0;
        int c = 0;
        double4 pi;
        bool have_pi = false;
        for (int dx = 0; dx < 3; ++dx)
            for (int dy = 0; dy < 3; ++dy) {
                int R = (a + dx) * (kTY + 2) + (b + dy);
                int s0 = cs[R][k0], e0 = cs[R][k1];
                int gR = d.wstart[R] - d.woff[R];
                if (zsorted) {   // uniform binary searches (broadcast loads)
                    int lo = s0, hi = e0;
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (w32[mid].z < zlo) lo = mid + 1; else hi = mid;
                    }
                    int s1 = lo;
                    hi = e0;
                    while (lo < hi) {
                        int mid = (lo + hi) >> 1;
                        if (w32[mid].z <= zhi) lo = mid + 1; else hi = mid;
                    }
                    s0 = s1;
                    e0 = lo;
                }
                for (int l0 = s0; l0 < e0; l0 += 32) {
                    unsigned m_in = 0, m_mb = 0;
                    const int span = min(32, e0 - l0);
#pragma unroll 1
                    for (int t0 = 0; t0 < span; t0 += 8) {
                        unsigned b_in = 0, b_mb = 0;
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            float4 p = w32[l0 + t0 + t];
                            float fx = qi.x - p.x, fy = qi.y - p.y, fz = qi.z - p.z;
                            float r2 = fx * fx + fy * fy + fz * fz;
                            b_in |= r2 <= flo ? 1u << t : 0u;
                            b_mb |= r2 <= fhi ? 1u << t : 0u;
                        }
                        m_in |= b_in << t0;
                        m_mb |= b_mb << t0;
                    }
                    unsigned vmask = span >= 32 ? 0xffffffffu : (1u << span) - 1u;
                    unsigned self = (li >= l0 && li < l0 + 32) ? 1u << (li - l0) : 0u;
                    vmask &= valid ? ~self : 0u;
                    m_in &= vmask;
                    unsigned m_bd = m_mb & vmask & ~m_in;   // borderline: exact fp64 test
                    if (m_bd) {
                        if (!have_pi) {
                            pi = ldg256(bpos + r);
                            have_pi = true;
                        }
                        while (m_bd) {
                            int t = __ffs(m_bd) - 1;
                            m_bd &= m_bd - 1;
                            double4 pj = ldg256(bpos + gR + l0 + t);
                            double ex = pi.x - pj.x, ey = pi.y - pj.y, ez = pi.z - pj.z;
                            if (ex * ex + ey * ey + ez * ez <= ell2) m_in |= 1u << t;
                        }
                    }
                    while (m_in) {   // ascending, like the scan order
                        int t = __ffs(m_in) - 1;
                        m_in &= m_in - 1;
                        MDG_DCHECK(l0 + t >= 0 && l0 + t < wrows && l0 + t != li);
                        glo = __byte_perm(glo, ghi, 0x5432);
                        ghi = __byte_perm(ghi, (unsigned)(l0 + t), 0x5432);
                        ++c;
                        if ((c & 3) == 0 && c <= cap4) op[(size_t)((c >> 2) - 1) * 32] = make_uint2(glo, ghi);
                    }
                }
            }
        if (valid) {
            if ((c & 3) && c < cap4) {
                unsigned long long g = ((unsigned long long)ghi << 32 | glo) >> (16 * (4 - (c & 3)));
                op[(size_t)(c >> 2) * 32] = make_uint2((unsigned)g, (unsigned)(g >> 32));
            }
            tcnt[slot0 + q] = min(c, cap);
            if (c > cap) atomicMax(maxcnt, c);
        }
    }
}

// Bank-aware order of each row's list (rebuild time).  The walk gathers x, y,
// z of its k-th entry with one LDS.64 each; lanes whose entries fall into the
// same 8-byte bank pair (window index mod 16 -- every window array starts at a
// multiple of 128 bytes) serialise, ~6 wavefronts per random warp load against
// 2 when the 16 lanes of a half-warp hit distinct pairs
// (tools/microbench_smem.cu: 1.7 -> 2.9-4.2 records / clock / SM).  The order
// of a row's entries is free (it only changes the summation order), so lane l
// emits its entries by class starting at class l mod 16:
//   ORDER 1: sorted by (class - l) mod 16;
//   ORDER 2: round robin over classes l, l+1, ..., one entry per class per
//            round, which keeps the lanes of a half-warp on distinct classes
//            until classes run dry.
// One warp per 32-row block; the row's entries are bucketed in shared memory.
template <int ORDER>
__global__ void vlt_order_kernel(int64_t nblocks, int cap4, uint16_t* __restrict__ tl,
                                 const int* __restrict__ tcnt) {
    extern __shared__ int osm[];
    const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int* off = osm + warp * (2 * 16 * 32);            // [16][32] bucket starts
    int* cnt = off + 16 * 32;                          // [16][32] bucket fill
    uint16_t* bk = reinterpret_cast<uint16_t*>(osm + warps * 2 * 16 * 32) + (size_t)warp * 32 * cap4;
    int64_t B = (int64_t)blockIdx.x * warps + warp;
    if (B >= nblocks) return;
    uint16_t* base = tl + B * 32 * cap4 + lane * 4;
    int c = tcnt[B * 32 + lane];
    int rot = lane & 15;
    for (int k = 0; k < 16; ++k) cnt[k * 32 + lane] = 0;
    for (int k = 0; k < c; ++k) {
        int e = base[(size_t)(k >> 2) * 128 + (k & 3)];
        ++cnt[((e - rot) & 15) * 32 + lane];
    }
    int acc = 0, mx = 0;
    for (int k = 0; k < 16; ++k) {
        int n = cnt[k * 32 + lane];
        off[k * 32 + lane] = acc;
        acc += n;
        mx = max(mx, n);
        cnt[k * 32 + lane] = 0;
    }
    uint16_t* mine = bk + lane;   // bucket slots strided by 32 (bank = lane)
    for (int k = 0; k < c; ++k) {
        int e = base[(size_t)(k >> 2) * 128 + (k & 3)];
        int key = (e - rot) & 15;
        int p = off[key * 32 + lane] + cnt[key * 32 + lane]++;
        mine[(size_t)p * 32] = (uint16_t)e;
    }
    int q = 0;
    if (ORDER == 1) {
        for (; q < c; ++q) base[(size_t)(q >> 2) * 128 + (q & 3)] = mine[(size_t)q * 32];
    } else {
        for (int r = 0; r < mx; ++r)
            for (int key = 0; key < 16; ++key)
                if (r < cnt[key * 32 + lane]) {
                    base[(size_t)(q >> 2) * 128 + (q & 3)] = mine[(size_t)(off[key * 32 + lane] + r) * 32];
                    ++q;
                }
    }
}

// Measured (config 2): shared-memory wavefronts 38.8M -> 30.2M and the walk
// 191.6 -> 184.7 us with ORDER 2, but the pass costs 0.3-0.4 ms per rebuild,
// more than it saves over a rebuild interval of 11 steps: opt-in.
static int vlt_env_order() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_ORDER");
        v = e ? atoi(e) : 0;
    }
    return v;
}

__global__ void vlt_mark_big_kernel(const TileDesc* __restrict__ desc, uint8_t* __restrict__ big_row) {
    __shared__ __align__(16) TileDesc d;
    load_desc(desc, blockIdx.x, d);
    __syncthreads();
    if (!d.big) return;
    for (int q = threadIdx.x; q < d.ni; q += blockDim.x) {
        int li;
        big_row[tile_row(d, q, li)] = 1;
    }
}

// ---- mbarrier / 1-D bulk-copy (TMA) primitives
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity) : "memory");
}
// L2 prefetch of a 16-byte aligned range (whole multiple of 16 bytes)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

constexpr int kConsumerWarps = 13;
constexpr int kTileThreads = (kConsumerWarps + 1) * 32;

template <bool MT>
struct WinLayout {
    // doubles per buffer of `rows` window rows: x, y, z, then int32 types (MT)
    __host__ __device__ static int doubles(int rows) { return 3 * rows + (MT ? rows / 2 : 0); }
    // per buffer: x, y, z (doubles) then types (int32) for MT
};

// One tile row's list walk (the consumers' body).  WR: the walk reads the full
// lists and writes the row's inner list (the entries within rp, in list
// order, 4 to a group like the outer list) and zeroes the row's path length.
//
// Pair arithmetic (kernels.py:36-52 up to rounding): y = 1/r^2 by MUFU.RCP64H
// plus one cubically convergent correction y (1 + e + e^2) (full double
// precision; a single Newton step leaves ~1e-14, which the cancellation of
// 2 a6 - 1 at the LJ minimum turns into a 1.5e-12 force there, above the
// reference's own 1e-12 bar, tests/test_containers.py:74-80), then
//   fs = eps24 s6 y^4 (2 s6 y^3 - 1)   with s6 = sig2^3,
// i.e. y^2, y^3 = y^2 y, y^4 = y^2 y^2, one DFMA and one DMUL per pair.  For a
// single type (MT = false) the constant eps24 s6 is factored out of the row's
// sum (the caller multiplies the three totals once), so a within-cutoff pair
// costs 18 FP64 instructions: 3 DADD + 3 (r^2) + DSETP + 3 (reciprocal) + 5 + 3
// accumulating DFMAs, with no branch (the accumulation is predicated).  MT:
// per-pair sig2 / eps24 lookups (forces.py:12-22).
template <bool MT>
__device__ __forceinline__ double lj_fs_walk(double r2, double c1, double& c0) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
    double e = fma(-r2, y, 1.0);
    y = fma(y, fma(e, e, e), y);
    double y2 = y * y;
    double y3 = y2 * y, y4 = y2 * y2;
    return y4 * fma(c1, y3, -1.0);
}

template <bool MT, int PF, bool WR>
__device__ __forceinline__ void vlt_walk_row(const double* wx, const double* wy, const double* wz,
                                             const int* wt, int li, int c, const uint2* lp,
                                             uint2* op, const uint2* sel, const LJTab& tab, double rp2,
                                             double c1s, double& fx, double& fy, double& fz,
                                             unsigned& hits, int& pc, int wrows_tile, int cap) {
    MDG_DCHECK(li >= 0 && li < wrows_tile && c >= 0 && c <= cap);
    double xi = wx[li], yi = wy[li], zi = wz[li];
    int ti = MT ? wt[li] : 0;
    // the first two entry groups are independent loads: issue them together
    // (every row owns >= 2 groups, cap4 >= 8), then keep the list stream
    // ahead of the walk
    // D list groups in flight (a register ring): the group loads come from
    // L2 (the producer prefetched the tile's lists) and their latency is the
    // walk's main stall otherwise
    constexpr int D = (PF == 2 || PF == 4) ? 2 : PF == 5 ? 3 : PF == 6 ? 4 : 1;
    uint2 g[D];
#pragma unroll
    for (int q = 0; q < D; ++q) g[q] = (q == 0 || 4 * q < c) ? __ldcs(lp + (size_t)q * 32) : make_uint2(0u, 0u);
    unsigned long long pk = 0;   // the inner group being filled (pc & 3 entries)
    const int rp2_hi = __double2hiint(rp2);
    const double rc2 = tab.rc2;
    pc = 0;
    for (int k0 = 0; k0 < c; k0 += 4) {
        uint2 cur = g[0];
#pragma unroll
        for (int q = 0; q + 1 < D; ++q) g[q] = g[q + 1];
        if (k0 + 4 * D < c) g[D - 1] = __ldcs(lp + (size_t)(k0 / 4 + D) * 32);
        int jj[4] = {(int)(cur.x & 0xffffu), (int)(cur.x >> 16), (int)(cur.y & 0xffffu),
                     (int)(cur.y >> 16)};
        unsigned keep = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            int j = jj[u];
            MDG_DCHECK(j < wrows_tile);
            double dx = xi - wx[j];
            double dy = yi - wy[j];
            double dz = zi - wz[j];
            double r2 = dx * dx + dy * dy + dz * dz;
            bool live = k0 + u < c;
            bool ok = live && r2 < rc2;
            // r^2 < rp^2 on the high words (non-negative doubles order like
            // their bits; equal high words keep the entry, a harmless superset)
            if (WR) keep |= (live && __double2hiint(r2) <= rp2_hi) ? 1u << u : 0u;
            double c0 = 1.0, c1 = c1s;
            if (MT) {
                int tj = wt[j];
                double s2 = tab.sig2[ti * tab.T + tj];
                double s6 = s2 * s2 * s2;
                c1 = 2.0 * s6;
                c0 = tab.eps24[ti * tab.T + tj] * s6;
            }
            double fs = lj_fs_walk<MT>(r2, c1, c0);
            if (MT) fs *= c0;
            // straight-line: a rejected (or padding, possibly r^2 = 0) entry
            // selects 0 before it reaches the sums
            fs = ok ? fs : 0.0;
            fx = fma(fs, dx, fx);
            fy = fma(fs, dy, fy);
            fz = fma(fs, dz, fz);
            hits += ok ? 1u : 0u;
        }
        if (WR && keep) {
            // the kept entries of this group, compacted (byte permutes from
            // the 16-entry selector table), appended to the inner list; a
            // completed group is one 8-byte store
            uint2 sl = sel[keep];
            int cnt = __popc(keep);
            unsigned long long nv = ((unsigned long long)__byte_perm(cur.x, cur.y, sl.y) << 32) |
                                    __byte_perm(cur.x, cur.y, sl.x);
            if (cnt < 4) nv &= (1ull << (16 * cnt)) - 1ull;
            int s = 16 * (pc & 3);
            pk |= nv << s;
            if ((pc & 3) + cnt >= 4) {
                op[(size_t)(pc >> 2) * 32] = make_uint2((unsigned)pk, (unsigned)(pk >> 32));
                pk = s ? nv >> (64 - s) : 0ull;
            }
            pc += cnt;
        }
    }
    // the last group's unused slots are zero, the padding the walk expects
    if (WR && (pc & 3)) op[(size_t)(pc >> 2) * 32] = make_uint2((unsigned)pk, (unsigned)(pk >> 32));
}

// Persistent, warp-specialised walk.  The last warp is the producer: it takes
// the next tile from the global counter, copies its descriptor and issues the
// window's 1-D bulk copies (one per range and component) into one of two
// buffers, completing on that buffer's `full` mbarrier.  The other warps
// consume: they take 32-row chunks of the tile dynamically, walk them, and
// arrive on the buffer's `empty` mbarrier when no chunk is left, so the
// producer refills it while they already work on the other buffer.  No
// CTA-wide barrier after the prologue.
//
// PRUNE (dynamic pruning): pst[0], raised by the refresh just
// before (or by the rebuild), picks the lists of the whole launch.  1: the
// full lists (tl / tcnt), and every row's inner list (the entries with
// r^2 < rp2 now, or a few more) is written to tl_in / tcnt_in; 0: the inner
// lists.  The pair sets within rc are the same (the
// refresh only lets the inner lists run while no owned row has moved
// (rp - rc) / 2 since they were written), so forces and counts are those of
// the full walk up to the grouping of the batched reciprocal.
template <int PLAYOUT, bool MT, int PF, bool KICK, int STAGES, bool PRUNE, bool WRITE>
__global__ void __launch_bounds__(kTileThreads, 2) vlt_force_kernel(
    const TileDesc* __restrict__ desc, const int* __restrict__ tbase, int ntiles, int wrows,
    int* __restrict__ next, int ms, int64_t n, int cap4, const double* __restrict__ s3,
    const int* __restrict__ row_tid, const int* __restrict__ tcnt_out, const uint2* __restrict__ tl_out,
    const int* __restrict__ row_src, double* __restrict__ force, LJTab tab,
    unsigned long long* counter, KickArgs kick, int* pst, uint2* tl_in,
    int* tcnt_in, float* __restrict__ disp, double rp2, int* __restrict__ bmax, int64_t nblk,
    int64_t n_force) {
    extern __shared__ __align__(128) double win[];
    __shared__ __align__(16) TileDesc d[STAGES];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    __shared__ int rowctr[STAGES], tile_of[STAGES];
    __shared__ int s_mode;
    __shared__ uint2 s_sel[16];   // byte-permute selectors: compact the kept entries of a group
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (PRUNE) {
        if (threadIdx.x == 0) s_mode = *(volatile const int*)pst;
        if (threadIdx.x < 16) {
            unsigned m = threadIdx.x, sl[2] = {0u, 0u};
            int h = 0;
            for (int e = 0; e < 4; ++e)
                if (m >> e & 1) {
                    sl[h >> 1] |= (unsigned)((2 * e) | (2 * e + 1) << 4) << (8 * (h & 1));
                    ++h;
                }
            s_sel[m] = make_uint2(sl[0], sl[1]);
        }
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < STAGES; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // the lists this launch walks (every CTA has read the mode before its
    // producer's first tile fetch; the fetch that sees the counter's final
    // value, ntiles + gridDim.x - 1, is the last one, so it may clear the mode)
    const bool whole = !PRUNE || s_mode != 0;
    // with pruning, two launches per walk: the inner-list walk (WRITE = 0)
    // and then the prune walk (WRITE = 1); the one whose mode is off returns
    // here, so neither carries the other's registers
    if (PRUNE && WRITE != whole) return;
    const uint2* tl = whole ? tl_out : tl_in;
    const int* tcnt = whole ? tcnt_out : tcnt_in;
    const int* bm = whole ? bmax : bmax + nblk;
    // single type: the window stride is the compile-time kWinRows, so the
    // y / z gathers use immediate offsets from the x address
    if (!MT) wrows = kWinRows;
    const int kBuf = WinLayout<MT>::doubles(wrows);
    // single-type constants of the pair arithmetic (vlt_walk_row): fs =
    // c0 y^4 (c1 y^3 - 1), c1 = 2 sig2^3, c0 = eps24 sig2^3
    const double s6 = tab.sig2[0] * tab.sig2[0] * tab.sig2[0];
    const double c1s = 2.0 * s6, c0s = tab.eps24[0] * s6;
    if (warp == kConsumerWarps) {
        // ---------------- producer
        for (int it = 0;; ++it) {
            int b = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[b], (it / STAGES - 1) & 1);
            // tiles with no walk work here -- no rows (vacuum: BASELINE
            // config 3 is 80% empty space) or overflow tiles (the row-space
            // kernel walks them) -- are skipped, not handed through the
            // window ring; a dense system pays nothing extra (its descriptor
            // load is the one the tile needs anyway)
            int t = 0;
            for (;;) {
                if (lane == 0) t = atomicAdd(next, 1);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= ntiles) break;
                if (lane < kDescInts / 4)
                    reinterpret_cast<int4*>(&d[b])[lane] = reinterpret_cast<const int4*>(desc + t)[lane];
                __syncwarp();
                if (d[b].ni > 0 && !d[b].big) break;
            }
            if (t >= ntiles) {
                if (PRUNE && WRITE && lane == 0 && t == ntiles + (int)gridDim.x - 1) {
                    pst[0] = 0;   // the inner lists are fresh
                    ++pst[1];
                }
                if (lane == 0) {
                    tile_of[b] = -1;
                    mbar_arrive(&full[b]);
                }
                break;
            }
            const TileDesc& D = d[b];
            if (D.big) {
                if (lane == 0) {
                    tile_of[b] = t;
                    mbar_arrive(&full[b]);
                }
                continue;
            }
            double* wx = win + b * kBuf;
            double* wy = wx + wrows;
            double* wz = wy + wrows;
            int* wt = reinterpret_cast<int*>(wz + wrows);
            if (lane == 0) {
                tile_of[b] = t;
                rowctr[b] = 0;
                mbar_arrive_tx(&full[b], (unsigned)D.wrows * (MT ? 28u : 24u));
            }
            __syncwarp();
            if (lane < kRanges) {
                int R = lane, o = D.woff[R], rows = D.woff[R + 1] - o, g = D.wstart[R];
                MDG_DCHECK(o >= 0 && rows >= 0 && o + rows <= wrows && (o & 3) == 0);
                if (rows > 0) {
                    bulk_g2s(wx + o, s3 + g, rows * 8u, &full[b]);
                    bulk_g2s(wy + o, s3 + (size_t)ms + g, rows * 8u, &full[b]);
                    bulk_g2s(wz + o, s3 + 2 * (size_t)ms + g, rows * 8u, &full[b]);
                    if (MT) bulk_g2s(wt + o, row_tid + g, rows * 4u, &full[b]);
                }
            } else if (PF >= 3) {
                // the tile's list stream (and counts) into L2 while the window
                // lands: the consumers' list loads then hit L2 instead of HBM
                // per 32-row block only the groups its longest row uses
                // (bmax), not the padded capacity cap4
                const int blk0 = tbase[t] >> 5, nb = (D.ni + 31) >> 5;
                const char* lb = reinterpret_cast<const char*>(tl) + (size_t)tbase[t] * cap4 * 2;
                for (int b = lane - kRanges; b < nb; b += 32 - kRanges) {
                    unsigned bytes = (unsigned)((bm[blk0 + b] + 3) & ~3) * 64u;
                    if (bytes) bulk_prefetch_l2(lb + (size_t)b * cap4 * 64, bytes);
                }
                if (lane == kRanges) {
                    size_t cb = ((size_t)(D.ni + 3) / 4) * 16;   // tcnt slots, whole 16-byte units
                    const char* cp = reinterpret_cast<const char*>(tcnt + tbase[t]);
                    size_t a0 = (size_t)cp & 15;                 // round the start down to 16 bytes
                    bulk_prefetch_l2(cp - a0, (unsigned)(cb + 16));
                }
            }
        }
        return;
    }
    // ---------------- consumers
    unsigned hits = 0;
    for (int it = 0;; ++it) {
        int b = it % STAGES;
        mbar_wait(&full[b], (it / STAGES) & 1);
        int t = tile_of[b];
        if (t < 0) break;
        const TileDesc& D = d[b];
        if (!D.big) {
            const double* wx = win + b * kBuf;
            const double* wy = wx + wrows;
            const double* wz = wy + wrows;
            const int* wt = reinterpret_cast<const int*>(wz + wrows);
            int slot0 = tbase[t];
            size_t base = (size_t)slot0 * cap4;
            int ni = D.ni;
            for (;;) {
                int q0 = 0;
                if (lane == 0) q0 = atomicAdd(&rowctr[b], 32);
                q0 = __shfl_sync(0xffffffffu, q0, 0);
                if (q0 >= ni) break;
                int q = q0 + lane;
                int cmax = 0;
                if (q < ni) {
                    int li;
                    int r = tile_row(D, q, li);
                    size_t go = ((size_t)base + (size_t)(q >> 5) * 32 * cap4) / 4 + (q & 31);
                    int c = tcnt[slot0 + q];
                    int i = row_src[r];
                    if (i >= n_force) c = 0;   // a ghost row of the decomposition: no force work
                    double fx = 0.0, fy = 0.0, fz = 0.0;
                    int pc;
                    if (PRUNE && WRITE) {
                        vlt_walk_row<MT, PF, true>(wx, wy, wz, wt, li, c, tl + go, tl_in + go, s_sel, tab, rp2,
                                                   c1s, fx, fy, fz, hits, pc, D.wrows, cap4);
                        tcnt_in[slot0 + q] = pc;
                        disp[r] = 0.f;
                    } else {
                        vlt_walk_row<MT, PF, false>(wx, wy, wz, wt, li, c, tl + go, nullptr, s_sel, tab, rp2,
                                                    c1s, fx, fy, fz, hits, pc, D.wrows, cap4);
                    }
                    if (!MT) {
                        fx *= c0s;
                        fy *= c0s;
                        fz *= c0s;
                    }
                    if (KICK) {
                        // apply_gravity + finish_kick (integrator.py:40-51), the
                        // arithmetic of finish_kick_kernel, on this particle
                        double mi = kick.mass[kick.tid ? kick.tid[i] : 0];
                        if (kick.has_gravity) fz = __dadd_rn(fz, __dmul_rn(mi, kick.gravity));
                        double cf = __ddiv_rn(__dmul_rn(0.5, kick.dt), mi);
                        size_t a0 = pidx<PLAYOUT>(i, 0, n), a1 = pidx<PLAYOUT>(i, 1, n),
                               a2 = pidx<PLAYOUT>(i, 2, n);
                        kick.vel[a0] = __dadd_rn(kick.vel[a0], __dmul_rn(__dadd_rn(fx, kick.old_force[a0]), cf));
                        kick.vel[a1] = __dadd_rn(kick.vel[a1], __dmul_rn(__dadd_rn(fy, kick.old_force[a1]), cf));
                        kick.vel[a2] = __dadd_rn(kick.vel[a2], __dmul_rn(__dadd_rn(fz, kick.old_force[a2]), cf));
                    }
                    force[pidx<PLAYOUT>(i, 0, n)] = fx;
                    force[pidx<PLAYOUT>(i, 1, n)] = fy;
                    force[pidx<PLAYOUT>(i, 2, n)] = fz;
                    if (PRUNE && WRITE) cmax = pc;
                }
                if (PRUNE && WRITE) {   // the inner lists' block extent (producer prefetch)
                    cmax = __reduce_max_sync(0xffffffffu, cmax);
                    if (lane == 0) bmax[nblk + ((slot0 + q0) >> 5)] = cmax;
                }
                __syncwarp();
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
    }
    warp_count(counter, hits);
}

static bool vlt_env_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VL_TILED");
        v = e ? atoi(e) : 1;
    }
    return v != 0;
}

static int vlt_env_tz() {
    static int v = -2;
    if (v == -2) {
        const char* e = getenv("MDG_VLT_TZ");
        v = e ? atoi(e) : -1;
    }
    return v;
}

static int vlt_env_budget();

// per 32-row block of the list slots: the longest row (vlt_force_kernel's
// producer prefetches ceil4(max) groups of every row of the block)
__global__ void vlt_bmax_kernel(const int* __restrict__ tcnt, int64_t nblk, int* __restrict__ bmax,
                                int* __restrict__ pst, const unsigned long long* __restrict__ scal,
                                unsigned long long* __restrict__ h_build) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (pst) {   // pruning state: the next walk prunes
            pst[0] = 1;
            pst[1] = pst[2] = pst[3] = 0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 7)   // the build's scalars [1..7] to the mapped pinned mirror
        h_build[threadIdx.x] = scal[1 + threadIdx.x];
    int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nblk) return;
    int c = tcnt[w * 32 + (threadIdx.x & 31)];
    c = __reduce_max_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) bmax[w] = c;
}

// MDG_VLT_BUILD: 2 = the warp-converged scan, otherwise the lane-per-row scan
// (measured faster: 0.475 against 0.725 ms, config 2)
static int vlt_env_build() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_BUILD");
        v = e ? atoi(e) : 1;
    }
    return v;
}
static int vlt_prune_setup(Context& c, size_t list_entries, size_t slots);

// threads per tile-build CTA (MDG_VLT_BT: 256, 384 (default), 512)
static int vlt_env_bt() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_BT");
        v = e ? atoi(e) : 384;
    }
    return v;
}

// One pass of the tiled build for the plan in v.plan: descriptors, list
// bases, the build kernel; the host check's inputs are copied to the pinned
// v.h_build.  0 = launched, 1 = tiling not applicable, -1 = error.
static int vlt_pass(Context& c, bool retry) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    const TilePlan tp{v.plan[0], v.plan[1], v.plan[2], v.plan[3]};
    const int budget = v.plan[4], ntiles = tp.ngx * tp.ngy * tp.nzt;
    GridView gv = make_view(gr);
    TileDesc* desc = reinterpret_cast<TileDesc*>(v.tdesc.p);
    int* nbig = (int*)(c.scal.p + 7);
    int* maxcnt = (int*)(c.scal.p + 3);
    const unsigned* maxabs = (const unsigned*)(c.scal.p + 5);
    double ell2 = gr.g.ell * gr.g.ell;
    v.cap4 = std::max(8, (v.cap + 3) & ~3);   // >= 2 groups per row (walk prefetch)
    // [3] longest list and [7] overflow tiles were zeroed by the rebuild's
    // binning (bin_count_kernel); a capacity retry zeroes them here
    if (retry) {
        MDG_CUDA(cudaMemsetAsync(nbig, 0, sizeof(int), c.stream));
        MDG_CUDA(cudaMemsetAsync(maxcnt, 0, sizeof(int), c.stream));
    }
    vlt_desc_kernel<<<blocks_for(ntiles, 128), 128, 0, c.stream>>>(gv, tp, ntiles, v.cap4, budget,
                                                                   desc, v.tsize.p, nbig), note_launch();
    exclusive_scan_i32(c, v.tsize.p, v.tbase.p, ntiles, c.scal.p + 1);
    // the lists get an upper-bound allocation (every tile's rows padded to
    // whole 32-row blocks), so their exact size is not needed on the host
    // before the build; slots (rows padded per tile) fit 32 bits, entries
    // (slots x cap4) are 64-bit -- BASELINE config 5 (67 M particles) needs ~5.4 G
    long long slots = (long long)c.n + 32ll * ntiles;
    if (slots > (1ll << 31) - 64) return 1;   // keep the row-space walk
    long long bound = slots * v.cap4;
    v.tl.ensure((size_t)bound + 8);
    v.tcnt.ensure((size_t)slots + 32);
    if (!v.tl.p || !v.tcnt.p) {
        set_error("out of device memory (VL tile lists)");
        return -1;
    }
    // (every slot of every tile is written by the build: no memset)
    if (vlt_env_build() == 2) MDG_CUDA(cudaMemsetAsync(v.tcnt.p, 0, ((size_t)slots + 32) * sizeof(int), c.stream));
    if (vlt_env_build() != 2) {
        // threads per tile CTA: a config-2 tile has ~283 rows, so 256 threads
        // leave one warp for a second pass (measured 423 us at 256, 385 at 384,
        // 467 at 512, config 2)
#define MDG_VLTB(NT)                                                                                \
    vlt_build_kernel<NT><<<ntiles, NT, 0, c.stream>>>(gv, desc, v.tbase.p, v.b32.p, gr.spos4.p,      \
                                                      maxabs, ell2, v.cap, v.cap4, v.tl.p, v.tcnt.p, \
                                                      maxcnt, gr.sort_by_z), note_launch()
        switch (vlt_env_bt()) {
            case 256: MDG_VLTB(256); break;
            case 512: MDG_VLTB(512); break;
            default: MDG_VLTB(384); break;
        }
#undef MDG_VLTB
    } else
        vlt_build_warp_kernel<<<ntiles, kBuildThreadsT, 0, c.stream>>>(
            gv, desc, v.tbase.p, v.b32.p, gr.spos4.p, maxabs, ell2, v.cap, v.cap4, v.tl.p, v.tcnt.p,
            maxcnt, gr.sort_by_z), note_launch();
    v.nblk = slots / 32;
    v.bmax.ensure(2 * (size_t)v.nblk + 2);
    if (!v.bmax.p) {
        set_error("out of device memory (VL list blocks)");
        return -1;
    }
    vlt_bmax_kernel<<<blocks_for(v.nblk * 32, 256), 256, 0, c.stream>>>(v.tcnt.p, v.nblk, v.bmax.p,
                                                                      v.prune_ready ? v.pst.p : nullptr, c.scal.p,
                                                                      v.d_h_build), note_launch();
    // (vlt_bmax_kernel wrote h_build[0] = [1] list slots, [2] = [3] longest list,
    // [6] = [7] overflow tiles into the mapped pinned mirror: no copy-engine bubble)
    return 0;
}

// Tiled build (called by vl_rebuild after the fp32 copy): 0 = tile lists
// launched (checked by vlt_finish at their first use), 1 = tiling not
// applicable (row-space lists instead), -1 = error.
int vlt_build(Context& c) {
    Verlet& v = c.vl;
    Grid& gr = v.grid;
    v.tiled = false;
    v.prune = false;
    v.build_pending = false;
    v.ntiles = v.nbig = 0;
    if (!vlt_env_enabled() || c.n == 0 || gr.pruned.n != 26) return 1;
    const Geom& g = gr.g;
    // TZ: the window (4 x 4 columns x TZ+2 cells) at 90% of the budget, at
    // the occupancy the average row sees: sum occ^2 / sum occ over the cells
    // (BASELINE config 3's slab in 80% vacuum: 18 rows per cell against a
    // mean of 4.3, whose tiles all overflowed the window before)
    double rho = (double)c.n / ((double)g.S[0] * g.S[1] * g.S[2]);
    if (gr.occ2 > 0.0 && gr.m > 0) rho = std::max(rho, gr.occ2 / (double)gr.m);
    int tz = vlt_env_tz();
    int budget = vlt_env_budget();
    if (tz < 1) tz = (int)floor(0.9 * budget / ((kTX + 2) * (kTY + 2) * std::max(rho, 1e-9))) - 2;
    tz = std::max(1, std::min(std::min(tz, g.S[2]), kMaxTZ));
    TilePlan tp{(g.S[0] + kTX - 1) / kTX, (g.S[1] + kTY - 1) / kTY, (g.S[2] + tz - 1) / tz, tz};
    int ntiles = tp.ngx * tp.ngy * tp.nzt;
    v.plan[0] = tp.ngx; v.plan[1] = tp.ngy; v.plan[2] = tp.nzt; v.plan[3] = tz; v.plan[4] = budget;
    v.tdesc.ensure((size_t)ntiles * kDescInts);
    v.tsize.ensure(ntiles + 1);
    v.tbase.ensure(ntiles + 1);
    v.big_row.ensure((size_t)gr.m + 1);
    if (!v.tdesc.p || !v.tsize.p || !v.tbase.p || !v.big_row.p) {
        set_error("out of device memory (VL tiles)");
        return -1;
    }
    if (!v.h_build && (cudaHostAlloc((void**)&v.h_build, 8 * sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess ||
                       cudaHostGetDevicePointer((void**)&v.d_h_build, v.h_build, 0) != cudaSuccess)) {
        v.h_build = nullptr;
        set_error("pinned allocation failed (VL tiles)");
        return -1;
    }
    if (!v.ev_build && cudaEventCreateWithFlags(&v.ev_build, cudaEventDisableTiming) != cudaSuccess) {
        v.ev_build = nullptr;
        set_error("event creation failed (VL tiles)");
        return -1;
    }
    if (int e = vlt_pass(c, false)) return e;
    MDG_CUDA(cudaEventRecord(v.ev_build, c.stream));
    v.ntiles = ntiles;
    v.win_rows = budget;
    v.tiled = true;
    v.build_pending = true;
    return 0;
}

int vlt_finish(Context& c) {
    Verlet& v = c.vl;
    if (!v.build_pending) return 0;
    v.build_pending = false;
    MDG_CUDA(cudaEventSynchronize(v.ev_build));
    for (int attempt = 1; (int)(v.h_build[2] & 0xffffffffu) > v.cap; ++attempt) {
        int hmax = (int)(v.h_build[2] & 0xffffffffu);
        if (attempt >= 3) {
            set_error("VL tile lists: capacity retries exhausted");
            v.tiled = false;
            return -1;
        }
        v.cap = (hmax + hmax / 8 + 7) / 8 * 8;
        if (int e = vlt_pass(c, true)) {
            v.tiled = false;
            return e < 0 ? -1 : (vl_build_rows(c, nullptr) ? -1 : 0);
        }
        MDG_CUDA(cudaStreamSynchronize(c.stream));
    }
    const int ntiles = v.ntiles;
    const int big = (int)(v.h_build[6] & 0xffffffffu);
    Grid& gr = v.grid;
    int m = (int)gr.m;
    TileDesc* desc = reinterpret_cast<TileDesc*>(v.tdesc.p);
    if (int order = vlt_env_order()) {
        long long total = (long long)v.h_build[0];   // list slots
        int64_t nblocks = total / 32;
        int warps = (int)std::max<size_t>(1, std::min<size_t>(8, (200u << 10) / (32 * (size_t)v.cap4 * 2 + 16 * 32 * 8)));
        size_t smem = (size_t)warps * (2 * 16 * 32 * sizeof(int) + 32 * (size_t)v.cap4 * sizeof(uint16_t));
        static size_t attr = 0;
        if (smem > attr) {
            cudaFuncSetAttribute(vlt_order_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(vlt_order_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = smem;
        }
        if (nblocks > 0) {
            int grid = (int)((nblocks + warps - 1) / warps);
            if (order == 1)
                vlt_order_kernel<1><<<grid, warps * 32, smem, c.stream>>>(nblocks, v.cap4, v.tl.p, v.tcnt.p), note_launch();
            else
                vlt_order_kernel<2><<<grid, warps * 32, smem, c.stream>>>(nblocks, v.cap4, v.tl.p, v.tcnt.p), note_launch();
        }
    }
    if (big) {
        // tiles whose window does not fit: row-space lists for their rows
        MDG_CUDA(cudaMemsetAsync(v.big_row.p, 0, m, c.stream));
        vlt_mark_big_kernel<<<ntiles, 128, 0, c.stream>>>(desc, v.big_row.p), note_launch();
        if (vl_build_rows(c, v.big_row.p)) return -1;
    }
    v.nbig = big;
    {
        long long slots = (long long)c.n + 32ll * ntiles;
        if (vlt_prune_setup(c, (size_t)(slots * v.cap4) + 8, (size_t)slots + 32)) return -1;
    }
    if (getenv("MDG_VLT_DEBUG"))
        fprintf(stderr, "vlt: tz=%d tiles=%d big=%d cap=%d cap4=%d\n", v.plan[3], ntiles, big, v.cap, v.cap4);
    return 0;
}

// MDG_VLT_SPECULATE: 1 (default) the first walk after a build is queued before
// the build's host check (vlt_speculate / vl_compute), 0 after it
static int vlt_env_speculate() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_SPECULATE");
        v = e ? atoi(e) : 1;
    }
    return v;
}

static int vlt_prune_setup(Context& c, size_t list_entries, size_t slots);

// A build whose host check is still pending: prepare the walk to run before
// that check (the inner-list buffers and the pruning state, assuming no
// overflow tiles), so the host waits on the build while the GPU already
// walks.  False: check first (speculation off, or the opt-in list reorder).
bool vlt_speculate(Context& c) {
    Verlet& v = c.vl;
    if (!v.build_pending || !v.tiled || !vlt_env_speculate() || vlt_env_order()) return false;
    long long slots = (long long)c.n + 32ll * v.ntiles;
    return vlt_prune_setup(c, (size_t)(slots * v.cap4) + 8, (size_t)slots + 32) == 0;
}

// the overflow tiles' rows through the row-space walk (after vlt_finish)
void vlt_big_rows(Context& c) {
    if (!c.vl.nbig) return;
    if (c.layout == AOS) vl_force_rows_launch<AOS>(c, c.vl.big_row.p);
    else vl_force_rows_launch<SOA>(c, c.vl.big_row.p);
}

// window ring: STAGES buffers of `budget` rows (MDG_VLT_STAGES, MDG_VLT_WIN)
static int vlt_env_stages() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_STAGES");
        v = e ? atoi(e) : 2;
        if (v != 3) v = 2;
    }
    return v;
}

static int vlt_env_budget() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_WIN");
        v = e ? atoi(e) : 2048;
        v = std::max(64, std::min(v, kWinRows)) & ~3;
    }
    return v;
}

template <int PLAYOUT, bool MT, int PF, bool KICK, int STAGES, bool PRUNE, bool WRITE>
static void vlt_launch_st(Context& c, const KickArgs& kick) {
    Verlet& v = c.vl;
    int wrows = v.win_rows;
    size_t smem = STAGES * (size_t)WinLayout<MT>::doubles(MT ? wrows : kWinRows) * sizeof(double);
    static int ctas_per_sm = 0;
    static size_t smem_set = 0;
    auto kern = vlt_force_kernel<PLAYOUT, MT, PF, KICK, STAGES, PRUNE, WRITE>;
    if (smem != smem_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, kTileThreads, smem);
        if (ctas_per_sm < 1) ctas_per_sm = 1;
        smem_set = smem;
    }
    int grid = std::min(v.ntiles, c.sm_count * ctas_per_sm);
    if (grid < 1) return;
    kern<<<grid, kTileThreads, smem, c.stream>>>(
        reinterpret_cast<const TileDesc*>(v.tdesc.p), v.tbase.p, v.ntiles, wrows, (int*)(c.scal.p + 6),
        s3_stride((int)v.grid.m), c.n, v.cap4, v.s3.p, v.grid.row_tid.p, v.tcnt.p,
        reinterpret_cast<const uint2*>(v.tl.p), v.grid.row_src.p, c.force, c.tab, c.scal.p, kick,
        v.pst.p, reinterpret_cast<uint2*>(v.tl_in.p), v.tcnt_in.p, v.disp.p, v.prune_rp2, v.bmax.p,
        v.nblk, c.n_force), note_launch();
}

template <int PLAYOUT, bool MT, int PF, bool KICK>
static void vlt_launch_pf(Context& c, const KickArgs& kick) {
    if (PF >= 3 && c.vl.prune) {
        vlt_launch_st<PLAYOUT, MT, PF, KICK, 2, true, false>(c, kick);   // runs on inner lists
        vlt_launch_st<PLAYOUT, MT, PF, KICK, 2, true, true>(c, kick);    // runs when a prune is due
    } else if (vlt_env_stages() == 3) {
        vlt_launch_st<PLAYOUT, MT, PF, KICK, 3, false, false>(c, kick);
    } else {
        vlt_launch_st<PLAYOUT, MT, PF, KICK, 2, false, false>(c, kick);
    }
}

static int vlt_env_pf() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MDG_VLT_PF");
        v = e ? atoi(e) : 3;
    }
    return v;
}

// Dynamic pruning: the inner radius is rc + delta, delta from
// mdg_set_prune, else MDG_VL_PRUNE_DELTA, else skin / 3 (MDG_VL_PRUNE=0: off).
// Only with the default window ring and list prefetch, and only when every
// owned row is walked by the tiles (the refresh checks owned rows, the tile
// walk resets them).
static double vlt_prune_delta(const Context& c) {
    static int on = -1;
    static double env_delta = -1.0;
    if (on < 0) {
        const char* e = getenv("MDG_VL_PRUNE");
        on = e ? atoi(e) : 1;
        const char* d = getenv("MDG_VL_PRUNE_DELTA");
        env_delta = d ? atof(d) : -1.0;
    }
    if (vlt_env_stages() == 3 || vlt_env_pf() < 3 || c.prune_delta == 0.0) return 0.0;
    double dl = c.prune_delta > 0.0 ? c.prune_delta : (!on ? 0.0 : env_delta > 0.0 ? env_delta : c.skin / 3.0);
    return dl < c.skin ? dl : 0.0;
}

void vl_prune_invalidate(Context& c) {
    Verlet& v = c.vl;
    if (v.prune && v.pst.p) cudaMemsetAsync(v.pst.p, 1, sizeof(int), c.stream);
}

// after the tile lists are built: inner-list storage and the state that makes
// the first walk prune
static int vlt_prune_setup(Context& c, size_t list_entries, size_t slots) {
    Verlet& v = c.vl;
    v.prune = false;
    double rc = c.cutoff;
    double delta = v.nbig == 0 ? vlt_prune_delta(c) : 0.0;
    if (delta <= 0.0) return 0;
    v.tl_in.ensure(list_entries);
    v.tcnt_in.ensure(slots);
    if (!v.tl_in.p || !v.tcnt_in.p || !v.disp.p || !v.pst.p || !v.prune_ready) {
        set_error("out of device memory (VL inner lists)");
        return -1;
    }
    v.prune_rp2 = (rc + delta) * (rc + delta);
    // rows may move (rp - rc) / 2 each; 1e-6 absorbs the rounding of r^2
    // and of the unwrapped copies (~1e-13 at these coordinates)
    v.prune_thr = (float)(0.5 * delta - 1e-6);
    // the path lengths were zeroed by vl_build_pos_kernel and the state
    // ("prune at the next walk") set by vlt_bmax_kernel: no memsets here,
    // between the build's host check and the walk
    v.prune = true;
    return 0;
}

// Before the build positions pass: the pruning state's buffers, so the
// build's own kernels initialise them (vl_rebuild).  The path lengths (nullptr:
// no pruning configured).
float* vlt_prune_prepare(Context& c) {
    Verlet& v = c.vl;
    v.prune_ready = false;
    if (vlt_prune_delta(c) <= 0.0) return nullptr;
    v.disp.ensure((size_t)v.grid.m + 1);
    v.pst.ensure(4);
    v.prune_ready = v.disp.p && v.pst.p;
    return v.prune_ready ? v.disp.p : nullptr;
}

template <int PLAYOUT, bool MT>
static void vlt_launch(Context& c, const KickArgs* kick) {
    // 1: list prefetched one round ahead; 3 (default): one round + the producer
    // pulls each tile's list into L2 while the window lands
    int pf = vlt_env_pf();
    KickArgs none{};
    if (kick) {
        if (pf == 1) vlt_launch_pf<PLAYOUT, MT, 1, true>(c, *kick);
        else vlt_launch_pf<PLAYOUT, MT, 3, true>(c, *kick);
    } else {
        if (pf == 1) vlt_launch_pf<PLAYOUT, MT, 1, false>(c, none);
        else if (pf == 4) vlt_launch_pf<PLAYOUT, MT, 4, false>(c, none);
        else if (pf == 5) vlt_launch_pf<PLAYOUT, MT, 5, false>(c, none);
        else if (pf == 6) vlt_launch_pf<PLAYOUT, MT, 6, false>(c, none);
        else vlt_launch_pf<PLAYOUT, MT, 3, false>(c, none);
    }
}

// `kick`: apply_gravity + finish_kick fused into the walk's epilogue (only
// when every row is walked here, i.e. no overflow tiles; the caller checks).
bool vlt_compute(Context& c, const KickArgs* kick) {
    Verlet& v = c.vl;
    int* next = (int*)(c.scal.p + 6);
    bool mt = c.tab.T > 1;
    if (c.layout == AOS) vl_refresh_launch<AOS, SOA>(c, next, c.scal.p);
    else vl_refresh_launch<SOA, SOA>(c, next, c.scal.p);
    c.prof_mark();
    if (c.layout == AOS) {
        if (mt) vlt_launch<AOS, true>(c, kick); else vlt_launch<AOS, false>(c, kick);
        if (v.nbig) vl_force_rows_launch<AOS>(c, v.big_row.p);
    } else {
        if (mt) vlt_launch<SOA, true>(c, kick); else vlt_launch<SOA, false>(c, kick);
        if (v.nbig) vl_force_rows_launch<SOA>(c, v.big_row.p);
    }
    c.prof_mark();
    return true;
}

// ---------------------------------------------------------------- fp32 walk

// The fp32-compute / fp64-accumulate variant on the same tiles and lists:
// the window holds each row's 16-byte record {position relative to its
// build-time cell in fp32, packed cell coordinates} (vl_refresh32_kernel), so
// a gather is one LDS.128 and a displacement is (r_i - r_j) + (c_i - c_j) * cl
// with an exact integer part; the pair arithmetic is fp32, the per-row sums
// fold into fp64 every 4 entries.  Same producer / consumer ring as the fp64
// walk (1-D bulk copies of the records).  Measured alternative: staging
// tile-relative fp32 coordinates converted by the producer warp itself
// (no bulk copy) starves the consumers, 0.41 ms against 0.24 ms.
// One tile row of the fp32 walk.  Branch-free like the fp64 walk: a rejected
// or padding entry selects fs = 0; the approximate reciprocal (MUFU.RCP,
// ~2^-22) is far inside the variant's 1e-4 bar; the per-row fp32 partial
// sums fold into fp64 every 4 entries.  WR (dynamic pruning, as in the fp64
// walk): the row's inner list -- the entries with r^2 <= rp^2 (1 + 1e-5), a
// superset of the exact set since the fp32 r^2 is within ~1e-6 relative --
// is written as the walk goes; the fp64 walk may read it too.
template <bool MT, bool WR>
__device__ __forceinline__ void vlt_walk_row32(const float4* w4, const int* wt, int li, int c,
                                               const uint2* lp, uint2* op, const uint2* sel,
                                               const LJTab& tab, const Cells32& cc, float rc2, float rp2f,
                                               float s2c, float e24c, double& fx, double& fy, double& fz,
                                               unsigned& hits, int& pc) {
    const float4 qi = w4[li];
    const int ci = __float_as_int(qi.w);
    const int ti = MT ? wt[li] : 0;
    const float cxi = (float)(ci >> 20), cyi = (float)((ci >> 10) & 1023), czi = (float)(ci & 1023);
    uint2 g0 = __ldcs(lp);
    unsigned long long pk = 0;
    pc = 0;
    for (int k0 = 0; k0 < c; k0 += 4) {
        uint2 cur = g0;
        if (k0 + 4 < c) g0 = __ldcs(lp + (size_t)(k0 / 4 + 1) * 32);
        int jj[4] = {(int)(cur.x & 0xffffu), (int)(cur.x >> 16), (int)(cur.y & 0xffffu),
                     (int)(cur.y >> 16)};
        float px = 0.f, py = 0.f, pz = 0.f;
        unsigned keep = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float4 qj = w4[jj[u]];
            int cj = __float_as_int(qj.w);
            // (r_i - r_j) + (c_i - c_j) cl: the cell difference is an exact small integer
            float dx = fmaf(cxi - (float)(cj >> 20), cc.cl[0], qi.x - qj.x);
            float dy = fmaf(cyi - (float)((cj >> 10) & 1023), cc.cl[1], qi.y - qj.y);
            float dz = fmaf(czi - (float)(cj & 1023), cc.cl[2], qi.z - qj.z);
            float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            bool live = k0 + u < c;
            bool ok = live && r2 < rc2;
            if (WR) keep |= (live && r2 <= rp2f) ? 1u << u : 0u;
            float s2f = s2c, e24f = e24c;
            if (MT) {
                double s2d, e24d;
                lj_params<MT>(tab, ti, wt[jj[u]], s2d, e24d);
                s2f = (float)s2d;
                e24f = (float)e24d;
            }
            float inv;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(inv) : "f"(r2));
            float a = s2f * inv;
            float a6 = a * a * a;
            float fs = (e24f * inv) * (a6 * fmaf(2.0f, a6, -1.0f));
            fs = ok ? fs : 0.f;
            hits += ok ? 1u : 0u;
            px = fmaf(fs, dx, px);
            py = fmaf(fs, dy, py);
            pz = fmaf(fs, dz, pz);
        }
        fx += (double)px;
        fy += (double)py;
        fz += (double)pz;
        if (WR && keep) {   // the fp64 walk's compaction (byte permutes, one 8-byte store per group)
            uint2 sl = sel[keep];
            int cnt = __popc(keep);
            unsigned long long nv = ((unsigned long long)__byte_perm(cur.x, cur.y, sl.y) << 32) |
                                    __byte_perm(cur.x, cur.y, sl.x);
            if (cnt < 4) nv &= (1ull << (16 * cnt)) - 1ull;
            int sft = 16 * (pc & 3);
            pk |= nv << sft;
            if ((pc & 3) + cnt >= 4) {
                op[(size_t)(pc >> 2) * 32] = make_uint2((unsigned)pk, (unsigned)(pk >> 32));
                pk = sft ? nv >> (64 - sft) : 0ull;
            }
            pc += cnt;
        }
    }
    if (WR && (pc & 3)) op[(size_t)(pc >> 2) * 32] = make_uint2((unsigned)pk, (unsigned)(pk >> 32));
}

template <int PLAYOUT, bool MT, int STAGES, bool PRUNE, bool WRITE>
__global__ void __launch_bounds__(kTileThreads, 2) vlt_force32_kernel(
    const TileDesc* __restrict__ desc, const int* __restrict__ tbase, int ntiles, int wrows,
    int* __restrict__ next, int64_t n, int cap4, const float4* __restrict__ q32,
    const int* __restrict__ row_tid, const int* __restrict__ tcnt_out, const uint2* __restrict__ tl_out,
    const int* __restrict__ row_src, double* __restrict__ force, LJTab tab, Cells32 cc,
    unsigned long long* counter, int* __restrict__ bmax, int64_t nblk, int* pst, uint2* tl_in,
    int* tcnt_in, float* __restrict__ disp, double rp2, int64_t n_force) {
    extern __shared__ __align__(128) double win[];
    __shared__ __align__(16) TileDesc d[STAGES];
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    __shared__ int rowctr[STAGES], tile_of[STAGES];
    __shared__ int s_mode;
    __shared__ uint2 s_sel[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (PRUNE) {
        if (threadIdx.x == 0) s_mode = *(volatile const int*)pst;
        if (threadIdx.x < 16) {
            unsigned mm = threadIdx.x, sl[2] = {0u, 0u};
            int h = 0;
            for (int e = 0; e < 4; ++e)
                if (mm >> e & 1) {
                    sl[h >> 1] |= (unsigned)((2 * e) | (2 * e + 1) << 4) << (8 * (h & 1));
                    ++h;
                }
            s_sel[mm] = make_uint2(sl[0], sl[1]);
        }
    }
    if (threadIdx.x == 0) {
        for (int b = 0; b < STAGES; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // per buffer: float4[wrows], then int[wrows] types (MT); in doubles
    const int kBuf = 2 * wrows + (MT ? wrows / 2 : 0);
    // pruning (as in vlt_force_kernel): the mode picks the lists of the launch
    const bool whole = !PRUNE || s_mode != 0;
    if (PRUNE && WRITE != whole) return;
    const uint2* tl = whole ? tl_out : tl_in;
    const int* tcnt = whole ? tcnt_out : tcnt_in;
    const int* bm = whole ? bmax : bmax + nblk;
    if (warp == kConsumerWarps) {
        for (int it = 0;; ++it) {
            int b = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[b], (it / STAGES - 1) & 1);
            // tiles with no walk work here -- no rows (vacuum: BASELINE
            // config 3 is 80% empty space) or overflow tiles (the row-space
            // kernel walks them) -- are skipped, not handed through the
            // window ring; a dense system pays nothing extra (its descriptor
            // load is the one the tile needs anyway)
            int t = 0;
            for (;;) {
                if (lane == 0) t = atomicAdd(next, 1);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= ntiles) break;
                if (lane < kDescInts / 4)
                    reinterpret_cast<int4*>(&d[b])[lane] = reinterpret_cast<const int4*>(desc + t)[lane];
                __syncwarp();
                if (d[b].ni > 0 && !d[b].big) break;
            }
            if (t >= ntiles) {
                if (PRUNE && WRITE && lane == 0 && t == ntiles + (int)gridDim.x - 1) {
                    pst[0] = 0;   // the inner lists are fresh
                    ++pst[1];
                }
                if (lane == 0) {
                    tile_of[b] = -1;
                    mbar_arrive(&full[b]);
                }
                break;
            }
            const TileDesc& D = d[b];
            if (D.big) {
                if (lane == 0) {
                    tile_of[b] = t;
                    mbar_arrive(&full[b]);
                }
                continue;
            }
            float4* w4 = reinterpret_cast<float4*>(win + b * kBuf);
            int* wt = reinterpret_cast<int*>(w4 + wrows);
            if (lane == 0) {
                tile_of[b] = t;
                rowctr[b] = 0;
                mbar_arrive_tx(&full[b], (unsigned)D.wrows * (MT ? 20u : 16u));
            }
            __syncwarp();
            if (lane < kRanges) {
                int R = lane, o = D.woff[R], rows = D.woff[R + 1] - o, g = D.wstart[R];
                if (rows > 0) {
                    bulk_g2s(w4 + o, q32 + g, rows * 16u, &full[b]);
                    if (MT) bulk_g2s(wt + o, row_tid + g, rows * 4u, &full[b]);
                }
            } else {
                // per 32-row block only the groups its longest row uses
                // (bmax), not the padded capacity cap4
                const int blk0 = tbase[t] >> 5, nb = (D.ni + 31) >> 5;
                const char* lb = reinterpret_cast<const char*>(tl) + (size_t)tbase[t] * cap4 * 2;
                for (int b = lane - kRanges; b < nb; b += 32 - kRanges) {
                    unsigned bytes = (unsigned)((bm[blk0 + b] + 3) & ~3) * 64u;
                    if (bytes) bulk_prefetch_l2(lb + (size_t)b * cap4 * 64, bytes);
                }
            }
        }
        return;
    }
    unsigned hits = 0;
    const float rc2 = (float)tab.rc2;
    const float rp2f = (float)rp2 * (1.0f + 1e-5f);
    float s2c = 0.f, e24c = 0.f;
    if (!MT) {
        s2c = (float)tab.sig2[0];
        e24c = (float)tab.eps24[0];
    }
    for (int it = 0;; ++it) {
        int b = it % STAGES;
        mbar_wait(&full[b], (it / STAGES) & 1);
        int t = tile_of[b];
        if (t < 0) break;
        const TileDesc& D = d[b];
        if (!D.big) {
            const float4* w4 = reinterpret_cast<const float4*>(win + b * kBuf);
            const int* wt = reinterpret_cast<const int*>(w4 + wrows);
            int slot0 = tbase[t];
            size_t base = (size_t)slot0 * cap4;
            int ni = D.ni;
            for (;;) {
                int q0 = 0;
                if (lane == 0) q0 = atomicAdd(&rowctr[b], 32);
                q0 = __shfl_sync(0xffffffffu, q0, 0);
                if (q0 >= ni) break;
                int q = q0 + lane;
                int cmax = 0;
                if (q < ni) {
                    int li;
                    int r = tile_row(D, q, li);
                    size_t go = ((size_t)base + (size_t)(q >> 5) * 32 * cap4) / 4 + (q & 31);
                    int c = tcnt[slot0 + q];
                    int i = row_src[r];
                    if (i >= n_force) c = 0;   // a ghost row of the decomposition
                    double fx = 0.0, fy = 0.0, fz = 0.0;
                    int pc;
                    if (PRUNE && WRITE) {
                        vlt_walk_row32<MT, true>(w4, wt, li, c, tl + go, tl_in + go, s_sel, tab, cc, rc2, rp2f,
                                                 s2c, e24c, fx, fy, fz, hits, pc);
                        tcnt_in[slot0 + q] = pc;
                        disp[r] = 0.f;
                        cmax = pc;
                    } else {
                        vlt_walk_row32<MT, false>(w4, wt, li, c, tl + go, nullptr, s_sel, tab, cc, rc2, rp2f,
                                                  s2c, e24c, fx, fy, fz, hits, pc);
                    }
                    force[pidx<PLAYOUT>(i, 0, n)] = fx;
                    force[pidx<PLAYOUT>(i, 1, n)] = fy;
                    force[pidx<PLAYOUT>(i, 2, n)] = fz;
                }
                if (PRUNE && WRITE) {   // the inner lists' block extent (producer prefetch)
                    cmax = __reduce_max_sync(0xffffffffu, cmax);
                    if (lane == 0) bmax[nblk + ((slot0 + q0) >> 5)] = cmax;
                }
                __syncwarp();
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[b]);
    }
    warp_count(counter, hits);
}

template <int PLAYOUT, bool MT, bool PRUNE, bool WRITE>
static void vlt_launch32_st(Context& c, const Cells32& cc) {
    Verlet& v = c.vl;
    int wrows = v.win_rows;
    constexpr int STAGES = 2;
    size_t smem = STAGES * (size_t)(wrows * 16 + (MT ? wrows * 4 : 0));
    static int ctas_per_sm = 0;
    static size_t smem_set = 0;
    auto kern = vlt_force32_kernel<PLAYOUT, MT, STAGES, PRUNE, WRITE>;
    if (smem != smem_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, kern, kTileThreads, smem);
        if (ctas_per_sm < 1) ctas_per_sm = 1;
        smem_set = smem;
    }
    int grid = std::min(v.ntiles, c.sm_count * ctas_per_sm);
    if (grid < 1) return;
    kern<<<grid, kTileThreads, smem, c.stream>>>(
        reinterpret_cast<const TileDesc*>(v.tdesc.p), v.tbase.p, v.ntiles, wrows, (int*)(c.scal.p + 6),
        c.n, v.cap4, v.q32.p, v.grid.row_tid.p, v.tcnt.p, reinterpret_cast<const uint2*>(v.tl.p),
        v.grid.row_src.p, c.force, c.tab, cc, c.scal.p, v.bmax.p, v.nblk, v.pst.p,
        reinterpret_cast<uint2*>(v.tl_in.p), v.tcnt_in.p, v.disp.p, v.prune_rp2, c.n_force), note_launch();
}

template <int PLAYOUT, bool MT>
static void vlt_launch32(Context& c, const Cells32& cc) {
    if (c.vl.prune) {   // the inner-list walk, then the prune walk (one returns at once)
        vlt_launch32_st<PLAYOUT, MT, true, false>(c, cc);
        vlt_launch32_st<PLAYOUT, MT, true, true>(c, cc);
    } else {
        vlt_launch32_st<PLAYOUT, MT, false, false>(c, cc);
    }
}

// fp32 walk over the tiles (after vl_refresh32_kernel, which zeroes the tile
// counter); overflow tiles are the caller's
void vlt_compute32(Context& c, const Cells32& cc) {
    bool mt = c.tab.T > 1;
    if (c.layout == AOS) {
        if (mt) vlt_launch32<AOS, true>(c, cc); else vlt_launch32<AOS, false>(c, cc);
    } else {
        if (mt) vlt_launch32<SOA, true>(c, cc); else vlt_launch32<SOA, false>(c, cc);
    }
}

}  // namespace mdg
