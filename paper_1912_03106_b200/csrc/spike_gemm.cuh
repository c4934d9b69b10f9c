// SPIKE correction for wide factor groups: the rank-W update
//     Y_p[rows][cols] += G_p[rows][W] * T_pb[W][cols]
// of every non-first (forward) / non-last (backward) chunk p of a partitioned
// chain (band.cuh: k_spike_border produces the border values T), as a tiled
// fp64 tensor-core GEMM (mma.sync m8n8k4.f64, SASS DMMA).  One CTA owns a
// 128-row x 64-column tile of one chunk and one factor; 8 warps as 4 (rows) x
// 2 (columns), 4 x 4 DMMA tiles per warp, so a k-step of 4 costs 8 fragment
// loads for 16 DMMAs.  Operands stream through a 4-stage cp.async ring in
// K-steps of 16 (three stages in flight, one barrier per K-step):
//     A = G[k][row]   (row contiguous in HBM: [W][ldy])       smem As[k][128 + 4]
//     B = T[col][k]   (k contiguous: [P][ldt][W])             smem Bs[col][16 + 4]
// Row strides of 4 mod 16 doubles make the 8 x 4 (A) and 4 x 8 (B) fragment
// loads of a half-warp hit 16 distinct bank pairs.  Narrow factor groups (a few columns per factor) stay
// on k_spike_fix, which keeps T in shared memory and streams G rows once per
// 8 columns.
#pragma once
#include "band.cuh"

#define SG_TM 128
#define SG_TN 64
#define SG_KS 16
#define SG_AP (SG_TM + 4)
#define SG_BP (SG_KS + 4)
#define SG_NST 4
#define SG_SMEM ((size_t)SG_NST * (SG_KS * SG_AP + SG_TN * SG_BP) * sizeof(double))

__device__ __forceinline__ void sg_cp16(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}

// tiles: (factor, first grouped column, columns <= SG_TN) per blockIdx.z
// grid (row tiles of the longest chunk, P - 1 chunks, column tiles)
template <bool FWD>
__global__ void __launch_bounds__(256, 2)
k_spike_gemm(SpikeArgs a, const int4* __restrict__ tiles) {
    extern __shared__ __align__(16) double sg[];
    double* As = sg;                                   // [NST][KS][AP]
    double* Bs = sg + SG_NST * SG_KS * SG_AP;          // [NST][TN][BP]
    const int4 tl = tiles[blockIdx.z];
    const double* G = a.G[tl.x];
    const int c0 = tl.y, nc = tl.z;
    const int p = FWD ? 1 + blockIdx.y : blockIdx.y;    // chunk being fixed
    const int pb = FWD ? p - 1 : p + 1;                  // chunk holding its border
    const int r0 = spike_s0(a, p) * BD_NB, r1 = spike_s1(a, p) * BD_NB;
    const int row0 = r0 + blockIdx.x * SG_TM;
    if (row0 >= r1) return;
    const double* Tb = a.T + ((size_t)pb * a.ldt + c0) * a.W;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q4 = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;

    auto stage_load = [&](int st, int k0) {
        double* as = As + st * SG_KS * SG_AP;
        double* bs = Bs + st * SG_TN * SG_BP;
        // A: 16 k-rows x 64 16-byte pieces
#pragma unroll
        for (int i = 0; i < (SG_KS * SG_TM / 2) / 256; ++i) {
            const int t = tid + 256 * i;
            const int k = t / (SG_TM / 2), m = 2 * (t % (SG_TM / 2));
            const int row = row0 + m;
            const int ok = row < r1 ? 16 : 0;            // rows past the chunk: zero fill
            sg_cp16(as + k * SG_AP + m, G + (size_t)(k0 + k) * a.ldy + (ok ? row : r0), ok);
        }
        // B: 64 columns x 8 16-byte pieces
#pragma unroll
        for (int i = 0; i < (SG_TN * SG_KS / 2) / 256; ++i) {
            const int t = tid + 256 * i;
            const int n = t / (SG_KS / 2), k = 2 * (t % (SG_KS / 2));
            const int ok = n < nc ? 16 : 0;
            sg_cp16(bs + n * SG_BP + k, Tb + (size_t)(ok ? n : 0) * a.W + k0 + k, ok);
        }
        cp_async_commit();
    };

    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    const int nk = a.W / SG_KS;
#pragma unroll
    for (int i = 0; i < SG_NST - 1; ++i) {
        if (i < nk) stage_load(i, i * SG_KS);
        else cp_async_commit();
    }
    for (int ks = 0; ks < nk; ++ks) {
        cp_async_wait<SG_NST - 2>();      // stage ks has landed (this thread's copies)
        __syncthreads();                  // ... everyone's; and stage ks - 1 is free again
        if (ks + SG_NST - 1 < nk) stage_load((ks + SG_NST - 1) % SG_NST, (ks + SG_NST - 1) * SG_KS);
        else cp_async_commit();
        const double* as = As + (ks % SG_NST) * SG_KS * SG_AP + wm * 32 + g;
        const double* bs = Bs + (ks % SG_NST) * SG_TN * SG_BP + (wn * 32 + g) * SG_BP;
#pragma unroll
        for (int u = 0; u < SG_KS / 4; ++u) {
            double av[4], bv[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) av[mi] = as[(4 * u + q4) * SG_AP + 8 * mi];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bv[ni] = bs[8 * ni * SG_BP + 4 * u + q4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
                    dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
        }
    }
    // C fragment: row g, columns 2 q4, 2 q4 + 1 of each 8 x 8 tile
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const int row = row0 + wm * 32 + 8 * mi + g;
        if (row >= r1) continue;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = wn * 32 + 8 * ni + 2 * q4 + h;
                if (c < nc) a.Y[(size_t)(c0 + c) * a.ldy + row] += acc[mi][ni][h];
            }
    }
}
