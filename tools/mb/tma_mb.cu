// L2 -> SM operand-stream ceiling for the band chains (dev microbenchmark).
//
// Every CTA streams nsteps operand blocks of BLK bytes (as PIECE-byte TMA
// bulk copies through an NBUF ring with full / empty mbarriers) -- the
// operand stream of k_band_pipe without the math.  Modes:
//   shared   all CTAs read the same blocks (one factor, L2-resident or not)
//   multicast  cluster of CS CTAs: CTA r issues pieces p = r (mod CS) with
//            .multicast::cluster to every CTA of the cluster
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mb/tma_mb.cu -o tools/mb/tma_mb
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1912_03106_b200/csrc/tma.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
    uint32_t a = smem_u32(bar), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory");
}
__device__ __forceinline__ void tma_load_mc(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(a), "r"(parity) : "memory");
    } while (!done);
}

template <int CS>
__global__ void __launch_bounds__(160) k_stream(const double* F, size_t blk_doubles, int nsteps,
                                                int piece_doubles, int npb, int nbuf,
                                                size_t cta_stride, double* sink) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t full[8], empty[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CS > 1 ? cluster_rank() : 0;
    const double* Fc = F + (size_t)(blockIdx.x % 4) * cta_stride;
    if (threadIdx.x == 0) {
        for (int q = 0; q < nbuf; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], 4 * CS); }
        mbar_fence_init();
    }
    if (CS > 1) cluster_sync_all(); else __syncthreads();
    const uint32_t pbytes = piece_doubles * 8;
    const int total = nsteps * npb;
    if (warp == 4) {
        if (lane == 0) {
            for (int P = 0; P < total; ++P) {
                const int buf = P % nbuf, use = P / nbuf;
                // every CTA arms its own full barrier for every piece
                if (CS > 1) {
                    if (use > 0) mbar_wait_cl(&full[buf], (use - 1) & 1);   // phase use-1 done here
                    mbar_arrive_expect_tx(&full[buf], pbytes);
                }
                if (CS == 1 || (uint32_t)(P % CS) == rank) {
                    if (use > 0) mbar_wait_cl(&empty[buf], (use - 1) & 1);
                    const double* src = Fc + (size_t)(P / npb) * blk_doubles + (size_t)(P % npb) * piece_doubles;
                    if (CS == 1) {
                        mbar_arrive_expect_tx(&full[buf], pbytes);
                        tma_load_1d(sm + (size_t)buf * piece_doubles, src, pbytes, &full[buf]);
                    } else {
                        tma_load_mc(sm + (size_t)buf * piece_doubles, src, pbytes, &full[buf],
                                    (uint16_t)((1u << CS) - 1));
                    }
                }
            }
        }
    } else {
        double acc = 0.0;
        for (int P = 0; P < total; ++P) {
            const int buf = P % nbuf;
            mbar_wait_cl(&full[buf], (P / nbuf) & 1);
            acc += sm[(size_t)buf * piece_doubles + threadIdx.x];
            __syncwarp();
            if (lane == 0) {
                if (CS == 1) mbar_arrive(&empty[buf]);
                else mbar_arrive_remote(&empty[buf], (uint32_t)(P % CS));
            }
        }
        if (acc == 12345.678) sink[0] = acc;
    }
    __syncwarp();
    if (CS > 1) cluster_sync_all();
}

int main(int argc, char** argv) {
    const int W = argc > 1 ? atoi(argv[1]) : 512;
    const int nsteps = argc > 2 ? atoi(argv[2]) : 2000;
    const int CW = W < 128 ? W : 128;
    const size_t blk = (size_t)32 * (36 + (W / CW) * (CW + 4));
    const size_t nblk_alloc = 8160;
    const size_t fd = nblk_alloc * blk;
    double* F;
    CK(cudaMalloc(&F, fd * 8 * 4));   // room for distinct-data mode
    CK(cudaMemset(F, 0, fd * 8 * 4));
    double* sink;
    CK(cudaMalloc(&sink, 8));
    int nsm;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    struct Case { int grid, cs, pieces_per_blk, nbuf; size_t stride; const char* what; };
    std::vector<Case> cases;
    const int npb_whole = 1 + W / CW;
    for (int g : {nsm, 128})
        for (int cs : {1, 2, 4})
            for (int nbuf : {4, 6}) cases.push_back({g - g % cs, cs, npb_whole, nbuf, 0, "shared"});
    cases.push_back({nsm, 1, npb_whole, 4, blk * 64, "distinct(4 groups)"});
    const int only = argc > 3 ? atoi(argv[3]) : -1;
    if (only >= (int)cases.size()) return 3;
    for (int ci = 0; ci < (int)cases.size(); ++ci) {
        if (only >= 0 && ci != only) continue;
        auto& c = cases[ci];
        const int piece = (int)(blk / c.pieces_per_blk);   // approx equal pieces (mb only)
        const int pd = (piece / 16) * 16;
        const size_t smem = (size_t)c.nbuf * pd * 8;
        const int steps = std::min<int>(nsteps, (int)nblk_alloc);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(160);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        size_t stride = c.stride ? (size_t)(fd / 4) : 0;
        auto run = [&]() {
            if (c.cs == 1) {
                CK(cudaFuncSetAttribute(k_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                CK(cudaLaunchKernelEx(&cfg, k_stream<1>, (const double*)F, blk, steps, pd, c.pieces_per_blk, c.nbuf, stride, sink));
            } else if (c.cs == 2) {
                CK(cudaFuncSetAttribute(k_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                CK(cudaLaunchKernelEx(&cfg, k_stream<2>, (const double*)F, blk, steps, pd, c.pieces_per_blk, c.nbuf, stride, sink));
            } else {
                CK(cudaFuncSetAttribute(k_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
                CK(cudaLaunchKernelEx(&cfg, k_stream<4>, (const double*)F, blk, steps, pd, c.pieces_per_blk, c.nbuf, stride, sink));
            }
        };
        run();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        run();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double bytes_sm = (double)c.grid * steps * c.pieces_per_blk * pd * 8;
        printf("W=%d %-20s grid=%3d cs=%d nbuf=%d piece=%6d B: %.3f us/step/CTA, SM-ingest %.2f TB/s, L2-read %.2f TB/s\n",
               W, c.what, c.grid, c.cs, c.nbuf, pd * 8, ms * 1e3 / steps, bytes_sm / ms / 1e9,
               bytes_sm / c.cs / ms / 1e9);
        fflush(stdout);
    }
    return 0;
}
