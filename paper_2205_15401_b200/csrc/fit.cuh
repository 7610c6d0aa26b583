// Shape regularizers of the fitting loop (fit.cpp:44-115) on the device.
//
//   ShapeRegularizer::make  -> rest_edge_kernel, rest_laplacian_kernel (CSR adjacency in edge order)
//   edge_reg                -> edge_reg_kernel      (per edge; FP64 atomics into the gradient)
//   laplacian_reg           -> laplacian_reg_kernel (per vertex; gather in adjacency order, scatter -g/|N|)
//
// Values are block-reduced into one FP64 accumulator (sum order differs from the
// reference's sequential loop: tolerance-level), gradients are scaled by the
// caller's weight and added.
#pragma once

#include "gvr_common.cuh"

namespace gvrk {

struct RegView {
    int N, E;
    const int* edges;       // [2E] (a, b) as given
    const double* rest_len; // [E]
    const int* adj_start;   // [N+1] CSR offsets
    const int* adj;         // [2E] neighbours, per vertex in the order the edges list them (fit.cpp:53-55)
    const double* rest_lap; // [3N]
};

__device__ __forceinline__ void block_add(double v, double* acc) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __shared__ double red[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) s += red[w];
        if (s != 0.0) atomicAdd(acc, s);
    }
}

// rest_edge_length[e] = |c_a - c_b| (fit.cpp:56)
__global__ void rest_edge_kernel(RegView r, const double* __restrict__ centers, double* __restrict__ rest_len) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= r.E) return;
    const int a = r.edges[2 * e], b = r.edges[2 * e + 1];
    const double d0 = centers[3 * a] - centers[3 * b], d1 = centers[3 * a + 1] - centers[3 * b + 1],
                 d2 = centers[3 * a + 2] - centers[3 * b + 2];
    rest_len[e] = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
}

// rest_laplacian[i] = c_i - mean(neighbours) (fit.cpp:58-63); 0 for isolated vertices
__global__ void rest_laplacian_kernel(RegView r, const double* __restrict__ centers, double* __restrict__ rest_lap) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r.N) return;
    const int s0 = r.adj_start[i], s1 = r.adj_start[i + 1];
    double m[3] = {0.0, 0.0, 0.0};
    for (int q = s0; q < s1; ++q)
        for (int c = 0; c < 3; ++c) m[c] += centers[3 * r.adj[q] + c];
    for (int c = 0; c < 3; ++c) rest_lap[3 * i + c] = s1 > s0 ? centers[3 * i + c] - m[c] / (double)(s1 - s0) : 0.0;
}

// edge_reg (fit.cpp:66-85): mean squared deviation of edge lengths from rest.
__global__ void edge_reg_kernel(RegView r, const double* __restrict__ centers, double weight, double* value,
                                double* __restrict__ grad) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const double inv_n = 1.0 / r.E;
    double v = 0.0;
    if (e < r.E) {
        const int a = r.edges[2 * e], b = r.edges[2 * e + 1];
        double diff[3];
        for (int c = 0; c < 3; ++c) diff[c] = centers[3 * a + c] - centers[3 * b + c];
        const double len = fmax(sqrt(diff[0] * diff[0] + diff[1] * diff[1] + diff[2] * diff[2]), 1e-12);
        const double dev = len - r.rest_len[e];
        v = dev * dev * inv_n;
        if (grad) {
            const double s = weight * 2.0 * dev * inv_n / len;
            for (int c = 0; c < 3; ++c) {
                atomicAdd(grad + 3 * a + c, s * diff[c]);
                atomicAdd(grad + 3 * b + c, -s * diff[c]);
            }
        }
    }
    block_add(v, value);
}

// laplacian_reg (fit.cpp:87-113): mean squared deviation of the uniform
// Laplacian displacement from rest.
__global__ void laplacian_reg_kernel(RegView r, const double* __restrict__ centers, double weight, double* value,
                                     double* __restrict__ grad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const double inv_n = 1.0 / r.N;
    double v = 0.0;
    if (i < r.N) {
        const int s0 = r.adj_start[i], s1 = r.adj_start[i + 1];
        if (s1 > s0) {
            double m[3] = {0.0, 0.0, 0.0};
            for (int q = s0; q < s1; ++q)
                for (int c = 0; c < 3; ++c) m[c] += centers[3 * r.adj[q] + c];
            double delta[3];
            for (int c = 0; c < 3; ++c)
                delta[c] = (centers[3 * i + c] - m[c] / (double)(s1 - s0)) - r.rest_lap[3 * i + c];
            v = (delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]) * inv_n;
            if (grad) {
                for (int c = 0; c < 3; ++c) {
                    const double g = weight * 2.0 * inv_n * delta[c];
                    atomicAdd(grad + 3 * i + c, g);
                    const double gn = g / (double)(s1 - s0);
                    for (int q = s0; q < s1; ++q) atomicAdd(grad + 3 * r.adj[q] + c, -gn);
                }
            }
        }
    }
    block_add(v, value);
}

}  // namespace gvrk
