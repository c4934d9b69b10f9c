// Shared device helpers for libpintgpu (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PG_NT 256          // threads per CTA of the streamed kernels
#define PG_RES_NT 1024     // threads per CTA of the CTA-resident PCG
#define PG_RES_MAX 5000    // largest n solved CTA-resident (40 n bytes of smem)

// Column states of the batched PCG.
#define COL_ACTIVE    0
#define COL_CONVERGED 1
#define COL_MAXIT     2
#define COL_BREAKDOWN 3

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic CTA-wide sum of NV values per thread (fixed shuffle tree,
// then warps summed in index order by thread 0).  `scratch` holds
// (blockDim/32) * NV doubles.  Result valid in thread 0 only.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) scratch[warp * NV + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += scratch[w * NV + k];
            v[k] = s;
        }
    }
    __syncthreads();
}

// Read-only global loads through the non-coherent path.
template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }
