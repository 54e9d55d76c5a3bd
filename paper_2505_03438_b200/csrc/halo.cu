// Ghost (halo) exchange buffers of the spatial domain decomposition
// (paper_2505_03438_b200/decomp.py DeviceDecomposedSimulation).
// The reference has no decomposition; ghosts are the decomposed
// stand-in for its periodic images (cells.py:122-156, containers.py:93-118):
// fixed between rebuilds, refreshed every step.
//
// pack:   rows idx[0 .. nl+nr) of the bound positions -> one AoS (nl+nr, 3)
//         send buffer, + shift_l on `axis` for the first nl (to the left
//         neighbour's frame) and + shift_r for the rest -- one launch replaces
//         two gathers and two shifted adds;
// unpack: an AoS (count, 3) receive buffer -> bound rows [row0, row0+count)
//         in the bound layout (SoA needs it; AoS receives in place).
// Both are HBM-bound: 8 B index + 48 B per ghost.
#include "device.cuh"

namespace mdg {

template <int LAYOUT>
__global__ void ghost_pack_kernel(const double* __restrict__ pos, int64_t n, const int64_t* __restrict__ idx,
                                  int64_t nl, int64_t cnt, int axis, double sl, double sr,
                                  double* __restrict__ out) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt) return;
    int64_t i = idx[k];
    double s = k < nl ? sl : sr;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double v = pos[pidx<LAYOUT>(i, a, n)];
        out[3 * k + a] = a == axis ? v + s : v;
    }
}

template <int LAYOUT>
__global__ void ghost_unpack_kernel(const double* __restrict__ in, int64_t count, int64_t row0,
                                    double* __restrict__ pos, int64_t n) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) pos[pidx<LAYOUT>(row0 + k, a, n)] = in[3 * k + a];
}

void halo_pack(Context& c, const int64_t* idx, int64_t nl, int64_t cnt, int axis, double sl, double sr,
               double* out) {
    if (cnt <= 0) return;
    if (c.layout == AOS)
        ghost_pack_kernel<AOS><<<blocks_for(cnt, 256), 256, 0, c.stream>>>(c.pos, c.n, idx, nl, cnt, axis, sl, sr, out);
    else
        ghost_pack_kernel<SOA><<<blocks_for(cnt, 256), 256, 0, c.stream>>>(c.pos, c.n, idx, nl, cnt, axis, sl, sr, out);
    note_launch();
}

void halo_unpack(Context& c, const double* in, int64_t count, int64_t row0) {
    if (count <= 0) return;
    if (c.layout == AOS)
        ghost_unpack_kernel<AOS><<<blocks_for(count, 256), 256, 0, c.stream>>>(in, count, row0, c.pos, c.n);
    else
        ghost_unpack_kernel<SOA><<<blocks_for(count, 256), 256, 0, c.stream>>>(in, count, row0, c.pos, c.n);
    note_launch();
}

// Cell-order permutation of the particle arrays (Simulation(reorder=K)):
// dst_k[i] = src_k[order[i]] for the four (N,3)/(3,N) fp64 arrays and the
// int32 type ids, one pass (replaces five eager gathers).
template <int LAYOUT>
__global__ void gather_rows_kernel(const int64_t* __restrict__ order, int64_t n, Rows4 src, Rows4 dst,
                                   const int* __restrict__ tsrc, int* __restrict__ tdst) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t j = order[i];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k) dst.p[a][pidx<LAYOUT>(i, k, n)] = src.p[a][pidx<LAYOUT>(j, k, n)];
    if (tsrc) tdst[i] = tsrc[j];
}

void gather_rows(Context& c, const int64_t* order, int64_t n, int layout, Rows4 src, Rows4 dst,
                 const int* tsrc, int* tdst) {
    if (n <= 0) return;
    if (layout == AOS)
        gather_rows_kernel<AOS><<<blocks_for(n, 256), 256, 0, c.stream>>>(order, n, src, dst, tsrc, tdst);
    else
        gather_rows_kernel<SOA><<<blocks_for(n, 256), 256, 0, c.stream>>>(order, n, src, dst, tsrc, tdst);
    note_launch();
}

// Index permutations of the cell reorder (Simulation(reorder=K)), so the loop
// runs no eager torch kernels: op 0 out[i] = a[b[i]] (composition), 1
// out[a[i]] = i (inverse), 2 out[i] = ((const int32*)a)[i] (widening of
// mdg_owned_order's output).
__global__ void permutation_kernel(int op, int64_t n, const int64_t* __restrict__ a,
                                   const int64_t* __restrict__ b, int64_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (op == 0) out[i] = a[b[i]];
    else if (op == 1) out[a[i]] = i;
    else out[i] = (int64_t)reinterpret_cast<const int*>(a)[i];
}

void permutation(Context& c, int op, int64_t n, const int64_t* a, const int64_t* b, int64_t* out) {
    if (n > 0)
        permutation_kernel<<<blocks_for(n, 256), 256, 0, c.stream>>>(op, n, a, b, out), note_launch();
}

}  // namespace mdg
