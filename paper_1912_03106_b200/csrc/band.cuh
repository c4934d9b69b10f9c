// Banded Cholesky Phi: the reference's own algorithm on the GPU.
//
// The reference factors (M/dt + K) once per (grid, float(dt)) with LAPACK's
// banded Cholesky and back-substitutes every step (problems.py:130-146,
// scipy cholesky_banded / cho_solve_banded = dpbtrf / dpbtrs).  Here:
//
//  * k_band_factor: one CTA per distinct dt.  Right-looking blocked band
//    Cholesky (block nb = 32) on the lower band [n][w+1]; emits, per block
//    row k, the solve operands in two layouts
//        FL[k] = [ D_k^-1 | L(k rows, W cols before k) ]      (forward)
//        FU[k] = [ D_k^-T | L(W rows after k, k cols)^T ]     (backward)
//    each nb x LDA row-major (LDA = nb + W + 4: bank-conflict padding).
//  * forward  L y = b:  y_k = D_k^-1 b_k - (D_k^-1 L_win,k) y_window
//    backward L^T x = y: x_k = D_k^-T y_k - (D_k^-T U_win,k) x_window
//    k_band_chain walks the block rows for a chunk of BC columns sharing one
//    factor: per block step two independent fp64 tensor-core GEMM chains
//    (mma.sync m8n8k4, SASS DMMA) -- D^-1 b_k on b staged one step ahead, and
//    the window product -- and one barrier; the next block's operands are
//    TMA-prefetched (2-stage mbarrier ring), the window is a smem ring.
//
// Folding the explicit 32 x 32 diagonal-block inverses into the window
// operators at factor time leaves one GEMM on the sequential critical path;
// the factorisation itself is the same arithmetic as dpbtrf.
#pragma once
#include "common.cuh"
#include "tma.cuh"

#define BD_NB 32
#define BD_RHS_SRC 8          // source shapes held in registers by the rhs kernels

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// factorisation: one CTA per factor, 256 threads
// LB[i][d] = A[i][i-d] (d = 0..w), A = c M + K built from the CSR (lower part)
// Solve-operand layout of one block row (doubles): piece 0 = the 32 x 32
// diagonal-block inverse (row stride BD_PD), then NCHK pieces of CW window
// columns each (row stride CW + 4): every piece is one contiguous TMA copy.
#define BD_PD 36
// window chunk width of the operand layout: 64-column chunks for W = 512
// (17 KB TMA pieces: a 4-deep ring fits beside k_band_rb's 32-column window)
__host__ __device__ __forceinline__ int bd_cw(int W) { return W < 128 ? W : (W >= 512 ? 64 : 128); }
__host__ __device__ __forceinline__ size_t bd_block_doubles(int W) {
    return (size_t)32 * (BD_PD + (W / bd_cw(W)) * (bd_cw(W) + 4));
}

struct BandFactorArgs {
    int n, w, W, LDA, nblk;     // LDA unused (kept for ABI stability of the struct)
    const int* row_ptr;
    const int* col_idx;
    const double* m_val;
    const double* k_val;
};

__global__ void __launch_bounds__(256)
k_band_build(BandFactorArgs a, const double* __restrict__ cvals, double* const* LBs,
             const double* const* kper) {
    const int f = blockIdx.y;
    const double c = cvals[f];
    double* LB = LBs[f];
    // per-factor stiffness values on the same CSR pattern (frozen Newton
    // Jacobians); NULL: the level's own stiffness for every factor
    const double* kv = kper ? kper[f] : a.k_val;
    const int stride = a.w + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        double* row = LB + (size_t)i * stride;
        for (int d = 0; d <= a.w; ++d) row[d] = 0.0;
        for (int e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e) {
            const int j = a.col_idx[e];
            if (j <= i) row[i - j] += fma(c, a.m_val[e], kv[e]);
        }
    }
}

// smem: D[32][36], Dinv[32][36], P[wp][36] (wp = w rounded up to 32, rows past
// the panel zero), Lw[32][CW + 4] (one window chunk).  Row strides of 4 mod 16
// doubles keep the DMMA fragment loads of a half-warp on distinct bank pairs.
// Per block row k it emits FL[k] = [D_k^-1 | D_k^-1 L_win] and
// FU[k] = [D_k^-T | D_k^-T U_win] (32 x LDA, LDA = 32 + W + 4): the solve
// step is y_k = D_k^-1 b_k - (D_k^-1 L_win) y_win, whose first term does not
// depend on the chain.
// The two GEMM-shaped parts of a block step run on the fp64 tensor cores
// (mma.sync m8n8k4, SASS DMMA): the solve operands (32 x 32 times 32 x W,
// twice) and the trailing update A -= P P^T of the w x w window (8.4 MFLOP per
// step at w = 512: as scalar FMAs with two shared-memory loads each it was
// 85 % of the factorisation time, round 2).  Warp w of 8 takes every 8th
// 32 x 32 super-tile of the lower triangle: 8 fragment loads per 16 DMMAs.
#define BD_FS 36
__host__ __device__ constexpr int bd_factor_wp(int w) { return (w + 31) / 32 * 32; }
__host__ __device__ constexpr size_t bd_factor_smem(int w, int cw) {
    return (size_t)(2 * BD_NB * BD_FS + bd_factor_wp(w) * BD_FS + BD_NB * (cw + 4)) * sizeof(double);
}

__global__ void __launch_bounds__(256)
k_band_factor(BandFactorArgs a, double* const* LBs, double* const* FLs, double* const* FUs,
              int* status) {
    extern __shared__ double sm[];
    const int f = blockIdx.x;
    double* LB = LBs[f];
    double* FL = FLs[f];
    double* FU = FUs[f];
    constexpr int NB = BD_NB, S = BD_FS;
    const int wp = bd_factor_wp(a.w);
    double* D = sm;
    double* Di = D + NB * S;
    double* P = Di + NB * S;
    double* Lw = P + (size_t)wp * S;
    const int stride = a.w + 1;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, q4 = lane & 3;
    auto lb = [&](int i, int j) -> double& { return LB[(size_t)i * stride + (i - j)]; };
    // unconditional read of band entry (i, j): the address is clamped into the
    // band so the load never depends on a branch (loads of a row issue together)
    auto lbv = [&](int i, int j, bool ok) -> double {
        const int ii = min(i, a.n - 1);
        const int d = min(max(ii - j, 0), a.w);
        const double v = LB[(size_t)ii * stride + d];
        return ok ? v : 0.0;
    };
    for (int t = tid; t < wp * S; t += blockDim.x) P[t] = 0.0;
    int m_prev = wp;

    for (int k = 0; k < a.nblk; ++k) {
        const int k0 = k * NB;
        const int kb = min(NB, a.n - k0);
        // 1. diagonal block (padded with identity beyond n)
        for (int t = tid; t < NB * NB; t += blockDim.x) {
            const int i = t / NB, j = t % NB;
            const bool in = i < kb && j < kb;
            double v = lbv(k0 + i, k0 + j, in && j <= i && i - j <= a.w);
            if (!in && i == j) v = 1.0;
            D[i * S + j] = (j <= i) ? v : 0.0;
        }
        __syncthreads();
        // 2. Cholesky of D (right-looking, column by column)
        for (int j = 0; j < NB; ++j) {
            if (tid == 0) {
                const double djj = D[j * S + j];
                if (!(djj > 0.0)) atomicExch(status, 1 + k0 + j);
                D[j * S + j] = sqrt(fmax(djj, 1e-300));
            }
            __syncthreads();
            const double piv = D[j * S + j];
            for (int i = j + 1 + tid; i < NB; i += blockDim.x) D[i * S + j] /= piv;
            __syncthreads();
            for (int t = tid; t < NB * NB; t += blockDim.x) {
                const int i = t / NB, q = t % NB;
                if (q > j && i >= q) D[i * S + q] -= D[i * S + j] * D[q * S + j];
            }
            __syncthreads();
        }
        // 3. D^-1 (lower triangular), column per thread
        if (tid < NB) {
            const int cc = tid;
            for (int i = 0; i < NB; ++i) {
                double s = (i == cc) ? 1.0 : 0.0;
                for (int p = cc; p < i; ++p) s -= D[i * S + p] * Di[p * S + cc];
                Di[i * S + cc] = (i >= cc) ? s / D[i * S + i] : 0.0;
            }
        }
        // 4. panel rows r = k0+NB .. k0+NB+m-1 :  P = A_panel D^-T
        const int r0 = k0 + NB;
        const int m = max(0, min(a.w, a.n - r0));
        for (int r = tid; r < m; r += blockDim.x) {
            const int gr = r0 + r;
            double x[BD_NB];
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                const int gc = k0 + j;
                x[j] = lbv(gr, gc, j < kb && gr - gc <= a.w);
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                double s = x[j];
#pragma unroll
                for (int p = 0; p < j; ++p) s -= x[p] * D[j * S + p];
                x[j] = s / D[j * S + j];
            }
#pragma unroll
            for (int j = 0; j < NB; ++j) P[r * S + j] = x[j];
        }
        // rows past the panel stay zero (the panel shrinks at the end of the band)
        for (int t = m * S + tid; t < m_prev * S; t += blockDim.x) P[t] = 0.0;
        m_prev = m;
        __syncthreads();
        // write L back into the band (diagonal block + panel)
        for (int t = tid; t < NB * NB; t += blockDim.x) {
            const int i = t / NB, j = t % NB;
            if (i < kb && j <= i && i - j <= a.w) lb(k0 + i, k0 + j) = D[i * S + j];
        }
        for (int t = tid; t < m * NB; t += blockDim.x) {
            const int r = t / NB, j = t % NB;
            const int gr = r0 + r, gc = k0 + j;
            if (j < kb && gr - gc <= a.w) lb(gr, gc) = P[r * S + j];
        }
        // 5. solve operands of block k, piece by piece (layout: bd_block_doubles)
        {
            const int CW = bd_cw(a.W), nchk = a.W / CW, LW = CW + 4;
            double* fl = FL + (size_t)k * bd_block_doubles(a.W);
            double* fu = FU + (size_t)k * bd_block_doubles(a.W);
            for (int t = tid; t < NB * BD_PD; t += blockDim.x) {
                const int i = t / BD_PD, j = t % BD_PD;
                fl[t] = j < NB ? Di[i * S + j] : 0.0;              // D^-1
                fu[t] = j < NB ? Di[j * S + i] : 0.0;              // D^-T
            }
            for (int c = 0; c < nchk; ++c) {
                // Lw[i][q] = L[k0+i][k0-W+c CW+q] (final: earlier panels)
                for (int t = tid; t < NB * CW; t += blockDim.x) {
                    const int i = t / CW, ql = t % CW, q = c * CW + ql;
                    const int gr = k0 + i, gc = k0 - a.W + q;
                    Lw[i * LW + ql] = lbv(gr, max(gc, 0), i < kb && gc >= 0 && gr - gc <= a.w);
                }
                __syncthreads();
                double* flc = fl + NB * BD_PD + (size_t)c * NB * LW;
                double* fuc = fu + NB * BD_PD + (size_t)c * NB * LW;
                // (D^-1 L_win)[i][q] = sum_p Di[i][p] Lw[p][q]     (Di lower, zeros stored)
                // (D^-T U_win)[i][q] = sum_p Di[p][i] P[q][p]      (P rows >= m are zero)
                // 32 x CW each: 8-column tiles dealt round-robin to the warps
                for (int nt = warp; nt < CW / 8; nt += 8) {
                    double cl[4][2], cu[4][2];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) cl[mi][0] = cl[mi][1] = cu[mi][0] = cu[mi][1] = 0.0;
                    const int qb = c * CW + 8 * nt;              // first window column of the tile
#pragma unroll
                    for (int u = 0; u < NB / 4; ++u) {
                        const int kk = 4 * u + q4;
                        const double bl = Lw[kk * LW + 8 * nt + g];
                        const double bu = qb + g < wp ? P[(qb + g) * S + kk] : 0.0;
#pragma unroll
                        for (int mi = 0; mi < 4; ++mi) {
                            dmma_8x8x4(cl[mi][0], cl[mi][1], Di[(8 * mi + g) * S + kk], bl);
                            dmma_8x8x4(cu[mi][0], cu[mi][1], Di[kk * S + 8 * mi + g], bu);
                        }
                    }
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int o = (8 * mi + g) * LW + 8 * nt + 2 * q4 + h;
                            flc[o] = cl[mi][h];
                            fuc[o] = cu[mi][h];
                        }
                }
                // the 4 pad columns of every row
                for (int t = tid; t < NB * 4; t += blockDim.x) {
                    const int o = (t / 4) * LW + CW + t % 4;
                    flc[o] = 0.0;
                    fuc[o] = 0.0;
                }
                __syncthreads();
            }
        }
        // 6. trailing update of the band: A[r][s] -= P[r] . P[s], s <= r, by
        // 32 x 32 super-tiles of the lower triangle
        {
            const int nR = (m + 31) / 32, nST = nR * (nR + 1) / 2;
            for (int idx = warp; idx < nST; idx += 8) {
                int R = (int)((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
                while (R * (R + 1) / 2 > idx) --R;
                while ((R + 1) * (R + 2) / 2 <= idx) ++R;
                const int Sx = idx - R * (R + 1) / 2;
                double acc[4][4][2];
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
                const double* pa = P + (32 * R + g) * S + q4;
                const double* pb = P + (32 * Sx + g) * S + q4;
#pragma unroll
                for (int u = 0; u < NB / 4; ++u) {
                    double av[4], bv[4];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) av[mi] = pa[8 * mi * S + 4 * u];
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) bv[ni] = pb[8 * ni * S + 4 * u];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int ni = 0; ni < 4; ++ni)
                            dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
                }
                // read-modify-write of the band, 8 loads in flight per lane
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) {
                    const int r = 32 * R + 8 * mi + g;
                    double* row = LB + (size_t)(r0 + r) * stride + r;    // entry (r, s) at row[-s]
                    double old[4][2];
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int sc = 32 * Sx + 8 * ni + 2 * q4 + h;
                            old[ni][h] = (r < m && sc <= r) ? row[-sc] : 0.0;
                        }
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int sc = 32 * Sx + 8 * ni + 2 * q4 + h;
                            if (r < m && sc <= r) row[-sc] = old[ni][h] - acc[mi][ni][h];
                        }
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// batched solves
struct BandSolveArgs {
    int np, W, LDA, nblk, ldy;
    int nst;                     // unused
    double* Y;                   // [n_cols][ldy] grouped columns, in place
    const int4* chunks;          // (factor, first grouped column, count, 0)
    double* const* F;            // per factor: FL or FU base (chain operands)
    // SPIKE partition of the block chain (latency-bound batches): blockIdx.y
    // = chunk p0 + y of P, blocks [p q, (p + 1) q) (the last chunk to nblk);
    // q >= nblk, P = 1 is the plain sequential chain.  spike != 0: b = 0 and
    // the window before (FWD) / after (BWD) the chunk starts as unit vectors
    // (column c of the chunk group = window index col0 + c).
    int q, P, p0, spike;
    // k_band_chain_ks only: the scatter fused into the backward chain (x
    // written straight to u_out (+ g), skipping a [B][n] pass over HBM).
    // Zero-initialised = off.  (Forming b = c M u + f inside the forward
    // chain was measured 1.9x slower: the stencil loads compete with the
    // chain's shared-memory operand stream for the LSU pipe.)
    struct Fuse {
        int scatter;
        int n;
        const int* perm;                 // grouped column -> batch column
        double* u_out;                   // [B][n]
        const double* g;                 // optional [*][n], row g_idx[b]
        const int* g_idx;
    } fz;
};

// The sequential chain:  y_k = D_k^-1 b_k - (D_k^-1 L_win) y_window
// (backward: D^-T, U_win), for windows W <= 256 (whole block <= 77 KB).
// 4 warps, warp w owns rows 8w..8w+7.  Per block step: one DMMA chain for
// D_k^-1 b_k (b_k staged in smem one step ahead -- independent of the
// window) plus NCH chains over the window, a single barrier.  The next
// block's operands arrive by TMA (2-stage mbarrier ring); the window is a
// shared-memory ring holding the last 2*NSLOT blocks.
// smem (doubles): stage[2][block], ring[2 NSLOT][NB][BC + 4], sb[2][NB][BC + 4]
#define BD_CT 128
#define BD_NST 2
template <int BC, int CW, int NCHK, bool FWD>
__global__ void __launch_bounds__(BD_CT)
k_band_chain(BandSolveArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar[BD_NST];
    constexpr int NST = BD_NST;
    constexpr int NSLOT = CW * NCHK / BD_NB;
    constexpr int BLK = BD_NB * (BD_PD + NCHK * (CW + 4));
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    constexpr int NB = BD_NB, RS = BC + 4, NT8 = BC / 8;
    constexpr int W = NSLOT * NB;
    constexpr int NCH = W >= 128 ? 8 : 4;
    constexpr int RMASK = 2 * NSLOT - 1;
    double* stage = sm;
    double* ring = stage + (size_t)NST * BLK;
    double* sb = ring + (size_t)2 * NSLOT * NB * RS;   // [2][NB][RS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q4 = lane & 3;
    const int lrow = 8 * warp + g;
    const uint32_t blk_bytes = (uint32_t)(BLK * 8);
    // b staging: thread t moves (row t & 31, columns (t >> 5) + 4 j)
    constexpr int BPT = BC / 4;
    const int brow = threadIdx.x & 31, bcol = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    const int pch = a.p0 + blockIdx.y;
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const int lo = s0 - (a.spike ? NSLOT : 0), hi = s1 + (a.spike ? NSLOT : 0);
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };
    // window ring: zero, or (spike) unit vectors in the blocks before / after
    for (int t = threadIdx.x; t < 2 * NSLOT * NB * RS; t += BD_CT) {
        double v = 0.0;
        if (a.spike) {
            const int slot = t / (NB * RS), rr = (t / RS) % NB, c = t % RS;
            const int wb = (slot - (FWD ? s0 - NSLOT : s1)) & RMASK;
            v = (wb < NSLOT && c < ncol && wb * NB + rr == col0 + c) ? 1.0 : 0.0;
        }
        ring[t] = v;
    }
    double breg[BPT];
    auto load_b = [&](int s) {
        const int rr = NB * blk_of(s) + brow;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const int cc = bcol + 4 * j;
            breg[j] = (!a.spike && cc < ncol) ? a.Y[(size_t)(col0 + cc) * a.ldy + rr] : 0.0;
        }
    };
    auto store_b = [&](int buf) {
#pragma unroll
        for (int j = 0; j < BPT; ++j) sb[((size_t)buf * NB + brow) * RS + bcol + 4 * j] = breg[j];
    };
    load_b(0);
    store_b(0);
    if (nsteps > 1) load_b(1);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q + 1 < NST && q < nsteps; ++q) {
            mbar_arrive_expect_tx(&bar[q], blk_bytes);
            tma_load_1d(stage + (size_t)q * BLK, F + (size_t)blk_of(q) * BLK,
                        blk_bytes, &bar[q]);
        }
    }
    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        const int st = s & 1;
        const int sb_cur = s & 1;
        // keep nst - 1 blocks in flight: issue block s + nst - 1 into the stage
        // freed by block s - 1 (all threads passed the previous barrier)
        if (threadIdx.x == 0 && s + NST - 1 < nsteps) {
            const int sn = (s + 1) & 1;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[sn], blk_bytes);
            tma_load_1d(stage + (size_t)sn * BLK,
                        F + (size_t)blk_of(s + NST - 1) * BLK, blk_bytes, &bar[sn]);
        }
        // b of block s+1 (in registers since the previous step) -> smem; prefetch s+2
        if (s + 1 < nsteps) {
            store_b(sb_cur ^ 1);
            if (s + 2 < nsteps) load_b(s + 2);
        }
        double acc[NCH][NT8][2], dacc[2][NT8][2];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) dacc[c][nt][0] = dacc[c][nt][1] = 0.0;
        const int row = NB * k + lrow;
        mbar_wait(&bar[st], (s >> 1) & 1);
        const double* Lst = stage + (size_t)st * BLK;
        const double* Lrow = Lst + lrow * BD_PD;
        // D_k^-1 b_k  (independent of the window)
        const double* bb = sb + (size_t)sb_cur * NB * RS;
#pragma unroll
        for (int j = 0; j < NB; j += 4) {
            const double av = Lrow[j + q4];
            const double* rr = bb + (j + q4) * RS + g;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
                dmma_8x8x4(dacc[(j >> 2) & 1][nt][0], dacc[(j >> 2) & 1][nt][1], av, rr[8 * nt]);
        }
        // - (D_k^-1 L_win) y_window
#pragma unroll
        for (int j = 0; j < W; j += 4) {
            const int wbi = j / NB;
            const int blk = FWD ? (k - NSLOT + wbi) : (k + 1 + wbi);
            const bool ok = FWD ? (blk >= lo) : (blk < hi);
            const int slot = blk & RMASK;
            const double av = -Lst[NB * BD_PD + (j / CW) * NB * (CW + 4) + lrow * (CW + 4) +
                                   (j % CW) + q4];
            const double* rr = ring + ((size_t)slot * NB + (j % NB) + q4) * RS + g;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                const double bv = ok ? rr[8 * nt] : 0.0;
                dmma_8x8x4(acc[(j >> 2) % NCH][nt][0], acc[(j >> 2) % NCH][nt][1], av, bv);
            }
        }
        double* slotp = ring + (size_t)(k & RMASK) * NB * RS;
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cc = 8 * nt + 2 * q4 + h;
                double v = dacc[0][nt][h] + dacc[1][nt][h];
#pragma unroll
                for (int c = 0; c < NCH; ++c) v += acc[c][nt][h];
                slotp[lrow * RS + cc] = v;
                if (cc < ncol) a.Y[(size_t)(col0 + cc) * a.ldy + row] = v;
            }
        __syncthreads();            // block k visible in the ring; stage / sb buffers free
    }
}

// k-split chain: the same block step as k_band_chain with the 40 (W = 128)
// k-steps of every 8-row tile split between KS warps, so each SM
// sub-partition runs KS warps: while one waits for its DMMA issue slot the
// others issue their shared-memory loads (a single warp per sub-partition
// serialises DMMA issue, LDS latency and index math -- measured 1,665 cycles
// per step against 720 of DMMA issue).  128 KS threads: warp w owns rows
// 8 (w & 3) .. + 7 and k-slice w >> 2 of the block's k-steps (k-step t < 8:
// D^-1 b_k, t >= 8: window columns 4 (t - 8) ..).  Slices 1.. hand their
// partial tiles to slice 0 through shared memory under a named barrier per
// row tile; slice 0 finishes the block.
#include <type_traits>
#ifndef BD_KS_NCH
#define BD_KS_NCH 2
#endif
template <int BC, int CW, int NCHK, bool FWD, int KS>
__global__ void __launch_bounds__(128 * KS)
k_band_chain_ks(BandSolveArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar[BD_NST];
    constexpr int NT = 128 * KS;
    constexpr int NST = BD_NST;
    constexpr int NSLOT = CW * NCHK / BD_NB;
    constexpr int BLK = BD_NB * (BD_PD + NCHK * (CW + 4));
    constexpr int NB = BD_NB, RS = BC + 4, NT8 = BC / 8;
    constexpr int W = NSLOT * NB;
    constexpr int RMASK = 2 * NSLOT - 1;
    constexpr int KT = NB / 4 + W / 4;                  // k-steps per block step
    static_assert(KT % KS == 0, "k-steps must split evenly");
    constexpr int KPS = KT / KS;                        // k-steps per slice
    // DMMA latency ~27 cycles vs ~16 per issue: two chains keep the pipe busy
    constexpr int NCH = KPS >= 4 ? BD_KS_NCH : 1;
    __shared__ __align__(16) double part[KS > 1 ? KS - 1 : 1][4][32][2 * NT8];
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    double* stage = sm;
    double* ring = stage + (size_t)NST * BLK;
    double* sb = ring + (size_t)2 * NSLOT * NB * RS;   // [2][NB][RS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = warp & 3, kh = warp >> 2;
    const int g = lane >> 2, q4 = lane & 3;
    const int lrow = 8 * mt + g;
    const uint32_t blk_bytes = (uint32_t)(BLK * 8);
    // b staging: thread t moves (row t & 31, columns (t >> 5) + (NT / 32) j)
    constexpr int CST = NT / 32;
    constexpr int BPT = (BC + CST - 1) / CST;
    const int brow = threadIdx.x & 31, bcol = threadIdx.x >> 5;

    if (threadIdx.x == 0) {
        for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    const int pch = a.p0 + blockIdx.y;
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const int lo = s0 - (a.spike ? NSLOT : 0), hi = s1 + (a.spike ? NSLOT : 0);
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };
    for (int t = threadIdx.x; t < 2 * NSLOT * NB * RS; t += NT) {
        double v = 0.0;
        if (a.spike) {
            const int slot = t / (NB * RS), rr = (t / RS) % NB, c = t % RS;
            const int wb = (slot - (FWD ? s0 - NSLOT : s1)) & RMASK;
            v = (wb < NSLOT && c < ncol && wb * NB + rr == col0 + c) ? 1.0 : 0.0;
        }
        ring[t] = v;
    }
    double breg[BPT];
    auto load_b = [&](int s) {
        const int rr = NB * blk_of(s) + brow;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const int cc = bcol + CST * j;
            breg[j] = (!a.spike && cc < ncol) ? a.Y[(size_t)(col0 + cc) * a.ldy + rr] : 0.0;
        }
    };
    auto store_b = [&](int buf) {
#pragma unroll
        for (int j = 0; j < BPT; ++j)
            if (bcol + CST * j < BC) sb[((size_t)buf * NB + brow) * RS + bcol + CST * j] = breg[j];
    };
    // fused scatter (BWD, unpartitioned chain): output pointers of this
    // thread's (row, column) entries, resolved once
    const bool fsc = !FWD && a.fz.scatter && a.P == 1 && !a.spike;
    double* fo[NT8][2];
    const double* fg[NT8][2];
    if (fsc && kh == 0) {
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cc = 8 * nt + 2 * q4 + h;
                const int b = cc < ncol ? a.fz.perm[col0 + cc] : -1;
                fo[nt][h] = b >= 0 ? a.fz.u_out + (size_t)b * a.fz.n : nullptr;
                const int gi = (b >= 0 && a.fz.g) ? a.fz.g_idx[b] : -1;
                fg[nt][h] = gi >= 0 ? a.fz.g + (size_t)gi * a.fz.n : nullptr;
            }
    }
    load_b(0);
    store_b(0);
    if (nsteps > 1) load_b(1);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q + 1 < NST && q < nsteps; ++q) {
            mbar_arrive_expect_tx(&bar[q], blk_bytes);
            tma_load_1d(stage + (size_t)q * BLK, F + (size_t)blk_of(q) * BLK, blk_bytes, &bar[q]);
        }
    }
    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        const int st = s & 1;
        const int sb_cur = s & 1;
        if (threadIdx.x == 0 && s + NST - 1 < nsteps) {
            const int sn = (s + 1) & 1;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[sn], blk_bytes);
            tma_load_1d(stage + (size_t)sn * BLK, F + (size_t)blk_of(s + NST - 1) * BLK,
                        blk_bytes, &bar[sn]);
        }
        if (s + 1 < nsteps) {
            store_b(sb_cur ^ 1);
            if (s + 2 < nsteps) load_b(s + 2);
        }
        double acc[NCH][NT8][2];
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
        mbar_wait(&bar[st], (s >> 1) & 1);
        const double* Lst = stage + (size_t)st * BLK;
        const double* bb = sb + (size_t)sb_cur * NB * RS;
        // this warp's k-slice; the slice index is made a compile-time constant
        // so every operand address below folds to base + immediate
        auto slice = [&](auto KHC) {
            constexpr int KH = decltype(KHC)::value;
#pragma unroll
            for (int u = 0; u < KPS; ++u) {
                const int t = KH * KPS + u;
                double av;
                const double* rr;
                bool ok = true;
                if (t < NB / 4) {                       // D_k^-1 b_k
                    av = Lst[lrow * BD_PD + 4 * t + q4];
                    rr = bb + (4 * t + q4) * RS + g;
                } else {                                // - (D_k^-1 L_win) y_window
                    const int j = 4 * (t - NB / 4);
                    const int wbi = j / NB;
                    const int blk = FWD ? (k - NSLOT + wbi) : (k + 1 + wbi);
                    ok = FWD ? (blk >= lo) : (blk < hi);
                    av = -Lst[NB * BD_PD + (j / CW) * NB * (CW + 4) + lrow * (CW + 4) +
                              (j % CW) + q4];
                    rr = ring + ((size_t)(blk & RMASK) * NB + (j % NB) + q4) * RS + g;
                }
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt) {
                    const double bv = ok ? rr[8 * nt] : 0.0;
                    dmma_8x8x4(acc[u % NCH][nt][0], acc[u % NCH][nt][1], av, bv);
                }
            }
        };
        if constexpr (KS == 1) {
            slice(std::integral_constant<int, 0>{});
        } else {
            switch (kh) {
                case 0: slice(std::integral_constant<int, 0>{}); break;
                case 1: slice(std::integral_constant<int, 1>{}); break;
                case 2: if constexpr (KS > 2) slice(std::integral_constant<int, (KS > 2 ? 2 : 0)>{}); break;
                default: if constexpr (KS > 3) slice(std::integral_constant<int, (KS > 3 ? 3 : 0)>{}); break;
            }
        }
        double v[NT8][2];
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double x = acc[0][nt][h];
#pragma unroll
                for (int c = 1; c < NCH; ++c) x += acc[c][nt][h];
                v[nt][h] = x;
            }
        if constexpr (KS > 1) {
            if (kh > 0) {
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt) {
                    part[kh - 1][mt][lane][2 * nt] = v[nt][0];
                    part[kh - 1][mt][lane][2 * nt + 1] = v[nt][1];
                }
            }
            // the KS warps of row tile mt: named barrier 1 + mt
            asm volatile("bar.sync %0, %1;" ::"r"(1 + mt), "r"(32 * KS) : "memory");
        }
        if (kh == 0) {
            double* slotp = ring + (size_t)(k & RMASK) * NB * RS;
            const int row = NB * k + lrow;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = 8 * nt + 2 * q4 + h;
                    double y = v[nt][h];
#pragma unroll
                    for (int q = 0; q < KS - 1; ++q) y += part[q][mt][lane][2 * nt + h];
                    slotp[lrow * RS + cc] = y;
                    if (fsc) {
                        if (fo[nt][h] && row < a.fz.n)
                            fo[nt][h][row] = fg[nt][h] ? y + fg[nt][h][row] : y;
                    } else if (cc < ncol) {
                        a.Y[(size_t)(col0 + cc) * a.ldy + row] = y;
                    }
                }
        }
        __syncthreads();            // block k visible in the ring; stage / sb / part free
    }
}

// One-column chain for small batches (B <= #SMs: the coarsest chain, the
// sequential stepper, sparse coarse levels): 128 threads = 32 rows x 4 lanes,
// each lane a quarter of the K = 32 + W dot product with plain fp64 FMAs in
// two accumulators, reduced by two shuffles; one barrier per block step.
// NS-deep TMA ring (the one-column chain is latency-bound: keep NS - 1
// blocks in flight).  smem (doubles): stage[NS][block], ring[2 NSLOT][NB], sb[2][NB]
template <int CW, int NCHK, int NS, bool FWD>
__global__ void __launch_bounds__(BD_CT)
k_band_chain1(BandSolveArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar[NS];
    constexpr int NST = NS;
    constexpr int NSLOT = CW * NCHK / BD_NB;
    constexpr int BLK = BD_NB * (BD_PD + NCHK * (CW + 4));
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col = ch.y;
    constexpr int NB = BD_NB;
    constexpr int W = NSLOT * NB;
    constexpr int RMASK = 2 * NSLOT - 1;
    double* stage = sm;
    double* ring = stage + (size_t)NST * BLK;
    double* sb = ring + 2 * NSLOT * NB;
    const int r = threadIdx.x >> 2, sub = threadIdx.x & 3;
    const uint32_t blk_bytes = (uint32_t)(BLK * 8);
    double* Ycol = a.Y + (size_t)col * a.ldy;

    for (int t = threadIdx.x; t < 2 * NSLOT * NB; t += BD_CT) ring[t] = 0.0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < NST; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    const int pch = a.p0 + blockIdx.y;
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const int lo = s0 - (a.spike ? NSLOT : 0), hi = s1 + (a.spike ? NSLOT : 0);
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };
    double breg = 0.0;
    if (threadIdx.x < NB) sb[threadIdx.x] = Ycol[NB * blk_of(0) + threadIdx.x];
    if (threadIdx.x < NB && nsteps > 1) breg = Ycol[NB * blk_of(1) + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q + 1 < NST && q < nsteps; ++q) {
            mbar_arrive_expect_tx(&bar[q], blk_bytes);
            tma_load_1d(stage + (size_t)q * BLK, F + (size_t)blk_of(q) * BLK,
                        blk_bytes, &bar[q]);
        }
    }
    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        const int st = s % NST;
        const int sb_cur = s & 1;
        // keep nst - 1 blocks in flight: issue block s + nst - 1 into the stage
        // freed by block s - 1 (all threads passed the previous barrier)
        if (threadIdx.x == 0 && s + NST - 1 < nsteps) {
            const int sn = (s + NST - 1) % NST;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[sn], blk_bytes);
            tma_load_1d(stage + (size_t)sn * BLK,
                        F + (size_t)blk_of(s + NST - 1) * BLK, blk_bytes, &bar[sn]);
        }
        if (threadIdx.x < NB && s + 1 < nsteps) {
            sb[(sb_cur ^ 1) * NB + threadIdx.x] = breg;
            if (s + 2 < nsteps) breg = Ycol[NB * blk_of(s + 2) + threadIdx.x];
        }
        mbar_wait(&bar[st], (s / NST) & 1);
        const double* Lst = stage + (size_t)st * BLK;
        const double* Lrow = Lst + r * BD_PD;
        const double* bb = sb + sb_cur * NB;
        // 8 independent accumulators: the fp64 FMA latency, not the issue
        // rate, bounds a 4-lane row dot product
        double acc[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) acc[t] = Lrow[sub + 4 * t] * bb[sub + 4 * t];
        const double* Lw = Lst + NB * BD_PD + r * (CW + 4) + sub;
#pragma unroll
        for (int t = 0; t < W / 4; ++t) {
            const int wb = t / 8;                     // window block (compile time)
            const int blk = FWD ? (k - NSLOT + wb) : (k + 1 + wb);
            const bool ok = FWD ? (blk >= lo) : (blk < hi);
            const double w = ok ? ring[(blk & RMASK) * NB + sub + 4 * (t % 8)] : 0.0;
            const int j = 4 * t;                      // + sub
            acc[t % 8] = fma(-Lw[(j / CW) * NB * (CW + 4) + j % CW], w, acc[t % 8]);
        }
        const double a0 = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        const double a1 = (acc[4] + acc[5]) + (acc[6] + acc[7]);
        double v = a0 + a1;
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (sub == 0) {
            ring[(k & RMASK) * NB + r] = v;
            Ycol[NB * k + r] = v;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// SPIKE recombination.  Chunk p of the partitioned chain produced z_p with a
// zero window; the true solution is y_p = z_p + G_p t, t = the true values
// of the W rows bordering the chunk (the tail of chunk p - 1 forward, the
// head of chunk p + 1 backward) and G_p = the chunk's response to unit
// window values (computed once per factor with spike = 1).  Only the border
// rows need the sequential pass over the chunks; everything else is a
// parallel rank-W update.
struct SpikeArgs {
    int W, q, P, nblk, ldy, ldt;
    double* Y;                   // [cols][ldy]
    const int4* chunks;          // column groups (factor, first column, count)
    double* const* G;            // per factor: [W][ldy]
    double* T;                   // [P][ldt][W] border values per chunk
};

__device__ __forceinline__ int spike_s0(const SpikeArgs& a, int p) { return p * a.q; }
__device__ __forceinline__ int spike_s1(const SpikeArgs& a, int p) {
    return p + 1 == a.P ? a.nblk : (p + 1) * a.q;
}

// sequential border pass: one 1024-thread CTA per column group; thread
// (row i, slice sl) owns W / S terms of the row's W-term dot product, the
// S partials are reduced by all threads (output (c, i) per thread), so every
// border step is one round of independent loads, FMAs and two barriers.
// smem: tv[BCM][W] border values, red[S][BCM][W] partials.  T: [P][ldt][W].
template <int BCM, int W, bool FWD>
__global__ void __launch_bounds__(1024)
k_spike_border(SpikeArgs a) {
    constexpr int S = 1024 / W, JP = W / S, NO = W * BCM;
    extern __shared__ __align__(16) double sh[];
    double* tv = sh;
    double* red = sh + NO;
    const int4 ch = a.chunks[blockIdx.x];
    const double* G = a.G[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    const int i = threadIdx.x % W, sl = threadIdx.x / W;
    auto border = [&](int p) {                          // first row of the border of chunk p
        return FWD ? spike_s1(a, p) * BD_NB - W : spike_s0(a, p) * BD_NB;
    };
    auto zval = [&](int p, int t) {                     // z of output t = (c, row)
        const int c = t / W, r = border(p) + t % W;
        return c < ncol ? a.Y[(size_t)(col0 + c) * a.ldy + r] : 0.0;
    };
    auto tout = [&](int p, int t, double v) {
        const int c = t / W;
        if (c < ncol) a.T[((size_t)p * a.ldt + col0 + c) * W + t % W] = v;
    };
    int p = FWD ? 0 : a.P - 1;
    for (int t = threadIdx.x; t < NO; t += 1024) {
        const double v = zval(p, t);
        tv[t] = v;
        tout(p, t, v);
    }
    __syncthreads();
    for (int step = 1; step + 1 < a.P; ++step) {        // the far end's border is unused
        p = FWD ? step : a.P - 1 - step;
        double zv[(NO + 1023) / 1024];
#pragma unroll
        for (int u = 0; u < (NO + 1023) / 1024; ++u) {
            const int t = threadIdx.x + 1024 * u;
            zv[u] = t < NO ? zval(p, t) : 0.0;
        }
        const int r = border(p) + i;
        constexpr int JB = JP < 16 ? JP : 16;           // loads in flight per batch
        double acc[BCM];
#pragma unroll
        for (int c = 0; c < BCM; ++c) acc[c] = 0.0;
#pragma unroll
        for (int j0 = 0; j0 < JP; j0 += JB) {
            double gv[JB];
#pragma unroll
            for (int jj = 0; jj < JB; ++jj) gv[jj] = G[(size_t)(sl * JP + j0 + jj) * a.ldy + r];
#pragma unroll
            for (int c = 0; c < BCM; ++c)
#pragma unroll
                for (int jj = 0; jj < JB; ++jj)
                    acc[c] = fma(gv[jj], tv[c * W + sl * JP + j0 + jj], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < BCM; ++c) red[(sl * BCM + c) * W + i] = acc[c];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < (NO + 1023) / 1024; ++u) {
            const int t = threadIdx.x + 1024 * u;
            if (t < NO) {
                double v = zv[u];
#pragma unroll 8
                for (int q = 0; q < S; ++q) v += red[q * NO + t];
                tv[t] = v;
                tout(p, t, v);
            }
        }
        __syncthreads();
    }
}

// parallel rank-W update of every non-first chunk
// grid (row tiles of 256, P - 1 chunks, column groups)
template <int BCM, bool FWD>
__global__ void __launch_bounds__(256)
k_spike_fix(SpikeArgs a) {
    extern __shared__ __align__(16) double tv[];        // [W][BCM]
    const int4 ch = a.chunks[blockIdx.z];
    const double* G = a.G[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    const int p = FWD ? 1 + blockIdx.y : blockIdx.y;    // chunk being fixed
    const int pb = FWD ? p - 1 : p + 1;                  // chunk holding its border
    const int r0 = spike_s0(a, p) * BD_NB, r1 = spike_s1(a, p) * BD_NB;
    const int r = r0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (r0 + blockIdx.x * blockDim.x >= r1) return;      // whole tile past the chunk
    for (int t = threadIdx.x; t < a.W * BCM; t += blockDim.x) {
        const int c = t / a.W, j = t % a.W;
        tv[j * BCM + c] = c < ncol ? a.T[((size_t)pb * a.ldt + col0 + c) * a.W + j] : 0.0;
    }
    __syncthreads();
    if (r >= r1) return;
    double acc[BCM];
#pragma unroll
    for (int c = 0; c < BCM; ++c) acc[c] = 0.0;
#pragma unroll 8
    for (int j = 0; j < a.W; ++j) {
        const double gv = G[(size_t)j * a.ldy + r];
        if constexpr (BCM % 2 == 0) {
            const double2* t2 = reinterpret_cast<const double2*>(tv + j * BCM);
#pragma unroll
            for (int c = 0; c < BCM / 2; ++c) {
                const double2 t = t2[c];
                acc[2 * c] = fma(gv, t.x, acc[2 * c]);
                acc[2 * c + 1] = fma(gv, t.y, acc[2 * c + 1]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < BCM; ++c) acc[c] = fma(gv, tv[j * BCM + c], acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < BCM; ++c)
        if (c < ncol) a.Y[(size_t)(col0 + c) * a.ldy + r] += acc[c];
}

// single-column rank-W update (the coarsest chain's spike correction): the
// W-term dot product of every row is split over 8 thread slices so a call
// spreads over (rows / 32) x (P - 1) CTAs instead of a few long serial loops.
// grid (row tiles of 32, P - 1 chunks, column groups); 256 threads = 32 rows x 8 slices
template <bool FWD>
__global__ void __launch_bounds__(256)
k_spike_fix1(SpikeArgs a) {
    __shared__ double red[8][33];
    const int4 ch = a.chunks[blockIdx.z];
    const double* G = a.G[ch.x];
    const int col = ch.y;
    const int p = FWD ? 1 + blockIdx.y : blockIdx.y;    // chunk being fixed
    const int pb = FWD ? p - 1 : p + 1;                  // chunk holding its border
    const int r0 = spike_s0(a, p) * BD_NB, r1 = spike_s1(a, p) * BD_NB;
    const int rl = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int r = r0 + blockIdx.x * 32 + rl;
    if (r0 + blockIdx.x * 32 >= r1) return;             // whole tile past the chunk
    const double* t = a.T + ((size_t)pb * a.ldt + col) * a.W;
    const int JS = a.W / 8;
    double acc0 = 0.0, acc1 = 0.0;
    if (r < r1) {
        int j = sl * JS;
        const int je = j + JS;
        for (; j + 1 < je; j += 2) {
            acc0 = fma(G[(size_t)j * a.ldy + r], t[j], acc0);
            acc1 = fma(G[(size_t)(j + 1) * a.ldy + r], t[j + 1], acc1);
        }
        if (j < je) acc0 = fma(G[(size_t)j * a.ldy + r], t[j], acc0);
    }
    red[sl][rl] = acc0 + acc1;
    __syncthreads();
    if (sl == 0 && r < r1) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) v += red[q][rl];
        a.Y[(size_t)col * a.ldy + r] += v;
    }
}

// The 512-wide window (511^2 grid; 140 KB of operands per block, two
// blocks no longer fit in smem).  Warp-specialised pipeline: warp 4 is a TMA
// producer streaming the block operands piece by piece (D^-1, then CW-column
// window chunks) through a ring of BD_NBUF buffers with full / empty
// mbarriers, so operand bandwidth overlaps compute for any window width (the
// 512-wide window of the 511^2 grid is 140 KB per block).  Warps 0-3 consume:
//   BC >= 8: warp w owns rows 8w..8w+7, fp64 tensor-core MMAs (m8n8k4,
//            SASS DMMA), NACC independent accumulator chains;
//   BC == 1: 32 rows x 4 lanes, plain fp64 FMAs, two shuffles.
// The window lives in a smem ring of NSLOT + 1 slots (block b in slot
// b mod (NSLOT + 1): never the slot the current window reads), b_k is
// staged in smem one step ahead; one named barrier (128 consumer threads)
// per block step.
#define BD_PCT 160
#define BD_NBUF_MAX 6
__host__ __device__ constexpr int bd_nbuf(int BC) { return BC == 1 ? 6 : 4; }
// one-column chain: TMA ring depth by window
// (measured round 1: 2 -- a 4-deep ring is 13% slower at W = 128, and a
// register-direct LDG variant without TMA 60% slower)
__host__ __device__ constexpr int bd_ns1(int W) { return W > 0 ? 2 : 2; }
template <int BC, int CW, int NCHK, bool FWD>
__global__ void __launch_bounds__(BD_PCT)
k_band_pipe(BandSolveArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t full[BD_NBUF_MAX], empty[BD_NBUF_MAX];
    constexpr int BD_NBUF = bd_nbuf(BC);
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    constexpr int NB = 32;
    constexpr int W = CW * NCHK;
    constexpr int NSLOT = W / NB;
    constexpr int NR = NSLOT + 1;
    constexpr int RS = BC == 1 ? 1 : BC + 4;
    constexpr int NT8 = BC >= 8 ? BC / 8 : 1;
    constexpr int NACC = W >= 128 ? 8 : 4;
    constexpr int PIECE = NB * (CW + 4) > NB * BD_PD ? NB * (CW + 4) : NB * BD_PD;
    constexpr int NPB = 1 + NCHK;                      // pieces per block
    const size_t blk_doubles = (size_t)NB * (BD_PD + NCHK * (CW + 4));
    double* bufs = sm;
    double* ring = bufs + (size_t)BD_NBUF * PIECE;
    double* sb = ring + (size_t)NR * NB * RS;          // [2][NB][RS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pch = a.p0 + blockIdx.y;                 // SPIKE chunk (BandSolveArgs)
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const int lo = s0 - (a.spike ? NSLOT : 0), hi = s1 + (a.spike ? NSLOT : 0);
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };

    if (threadIdx.x == 0) {
        for (int q = 0; q < BD_NBUF; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], 4);
        }
        mbar_fence_init();
    }
    // window ring (block b in slot b mod NR): zero, or (spike) unit vectors
    // in the NSLOT blocks before (FWD) / after (BWD) the chunk
    for (int t = threadIdx.x; t < NR * NB * RS; t += BD_PCT) {
        double v = 0.0;
        if (a.spike) {
            const int slot = t / (NB * RS), rr = (t / RS) % NB, c = t % RS;
            const int base = FWD ? s0 - NSLOT : s1;
            const int wb = ((slot - base) % NR + NR) % NR;
            v = (wb < NSLOT && c < (BC == 1 ? 1 : ncol) && wb * NB + rr == col0 + c) ? 1.0 : 0.0;
        }
        ring[t] = v;
    }
    __syncthreads();

    if (warp == 4) {
        // ---------------- producer ----------------
        if (lane == 0) {
            const int total = nsteps * NPB;
            for (int P = 0; P < total; ++P) {
                const int buf = P % BD_NBUF, use = P / BD_NBUF;
                if (use > 0) {
                    mbar_wait(&empty[buf], (use - 1) & 1);
                    fence_proxy_async_smem();   // consumers' generic reads before the refill
                }
                const int s = P / NPB, j = P % NPB;
                const double* src = F + (size_t)blk_of(s) * blk_doubles +
                                    (j == 0 ? 0 : (size_t)NB * BD_PD + (size_t)(j - 1) * NB * (CW + 4));
                const uint32_t bytes = (uint32_t)((j == 0 ? NB * BD_PD : NB * (CW + 4)) * 8);
                mbar_arrive_expect_tx(&full[buf], bytes);
                tma_load_1d(bufs + (size_t)buf * PIECE, src, bytes, &full[buf]);
            }
        }
        return;
    }

    // ---------------- consumers (warps 0..3) ----------------
    const int g = lane >> 2, q4 = lane & 3;
    const int lrow = 8 * warp + g;                      // DMMA row
    const int r1 = threadIdx.x >> 2, sub = threadIdx.x & 3;   // FMA row / lane
    double* Ycol0 = a.Y + (size_t)col0 * a.ldy;
    // b staging: thread t moves row t & 31 of columns (t >> 5) + 4 i
    constexpr int BPT = BC == 1 ? 1 : BC / 4;
    const int brow = threadIdx.x & 31, bcol = threadIdx.x >> 5;
    double breg[BPT];
    auto load_b = [&](int s) {
        const int rr = NB * blk_of(s) + brow;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const int cc = bcol + 4 * i;
            breg[i] = (!a.spike && (BC == 1 ? bcol == 0 : cc < ncol))
                          ? a.Y[(size_t)(col0 + (BC == 1 ? 0 : cc)) * a.ldy + rr] : 0.0;
        }
    };
    auto store_b = [&](int bufi) {
#pragma unroll
        for (int i = 0; i < BPT; ++i)
            if (BC > 1 || bcol == 0) sb[((size_t)bufi * NB + brow) * RS + (BC == 1 ? 0 : bcol + 4 * i)] = breg[i];
    };
    load_b(0);
    store_b(0);
    if (nsteps > 1) load_b(1);
    asm volatile("bar.sync 1, 128;" ::: "memory");

    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        const int sbc = s & 1;
        if (s + 1 < nsteps) {
            store_b(sbc ^ 1);
            if (s + 2 < nsteps) load_b(s + 2);
        }
        // window slot of window block 0 and validity
        const int blk0 = FWD ? (k - NSLOT) : (k + 1);
        const int slot0 = ((blk0 % NR) + NR) % NR;
        double acc[NACC][NT8][2];
#pragma unroll
        for (int c = 0; c < NACC; ++c)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
        double f[8];                                    // BC == 1 accumulators
#pragma unroll
        for (int t = 0; t < 8; ++t) f[t] = 0.0;
        const double* bb = sb + (size_t)sbc * NB * RS;
#pragma unroll
        for (int j = 0; j < NPB; ++j) {
            const int P = s * NPB + j;
            const int buf = P % BD_NBUF;
            mbar_wait(&full[buf], (P / BD_NBUF) & 1);
            const double* pc = bufs + (size_t)buf * PIECE;
            if (j == 0) {
                // D^-1 b_k  (piece 0, row stride BD_PD)
                if (BC == 1) {
                    const double* Lr = pc + r1 * BD_PD + sub;
#pragma unroll
                    for (int t = 0; t < 8; ++t) f[t] = fma(Lr[4 * t], bb[sub + 4 * t], f[t]);
                } else {
                    const double* Lr = pc + lrow * BD_PD;
#pragma unroll
                    for (int q = 0; q < NB; q += 4) {
                        const double av = Lr[q + q4];
                        const double* rr = bb + (q + q4) * RS + g;
#pragma unroll
                        for (int nt = 0; nt < NT8; ++nt)
                            dmma_8x8x4(acc[(q >> 2) % NACC][nt][0], acc[(q >> 2) % NACC][nt][1],
                                       av, rr[8 * nt]);
                    }
                }
            } else {
                const int jc = j - 1;                   // window chunk
                if (BC == 1) {
                    const double* Lr = pc + r1 * (CW + 4) + sub;
#pragma unroll
                    for (int t = 0; t < CW / 4; ++t) {
                        const int jg = jc * CW + 4 * t;     // window row - sub
                        const int wb = jg / NB;
                        const bool ok = FWD ? (blk0 + wb >= lo) : (blk0 + wb < hi);
                        int sl = slot0 + wb; if (sl >= NR) sl -= NR;
                        const double w = ok ? ring[sl * NB + (jg % NB) + sub] : 0.0;
                        f[t % 8] = fma(-Lr[4 * t], w, f[t % 8]);
                    }
                } else {
                    const double* Lr = pc + lrow * (CW + 4);
#pragma unroll
                    for (int q = 0; q < CW; q += 4) {
                        const int jg = jc * CW + q;     // window row (multiple of 4)
                        const int wb = jg / NB;
                        const bool ok = FWD ? (blk0 + wb >= lo) : (blk0 + wb < hi);
                        int sl = slot0 + wb; if (sl >= NR) sl -= NR;
                        const double av = -Lr[q + q4];
                        const double* rr = ring + ((size_t)sl * NB + (jg % NB) + q4) * RS + g;
#pragma unroll
                        for (int nt = 0; nt < NT8; ++nt) {
                            const double bv = ok ? rr[8 * nt] : 0.0;
                            dmma_8x8x4(acc[(q >> 2) % NACC][nt][0], acc[(q >> 2) % NACC][nt][1],
                                       av, bv);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[buf]);
        }
        // combine, store into the ring slot of block k and to global
        double* slotp = ring + (size_t)(k % NR) * NB * RS;
        if (BC == 1) {
            double v = ((f[0] + f[1]) + (f[2] + f[3])) + ((f[4] + f[5]) + (f[6] + f[7]));
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (sub == 0) {
                slotp[r1] = v;
                Ycol0[NB * k + r1] = v;
            }
        } else {
            const int row = NB * k + lrow;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = 8 * nt + 2 * q4 + h;
                    double v = 0.0;
#pragma unroll
                    for (int c = 0; c < NACC; ++c) v += acc[c][nt][h];
                    slotp[lrow * RS + cc] = v;
                    if (cc < ncol) a.Y[(size_t)(col0 + cc) * a.ldy + row] = v;
                }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");   // block k visible; sb free
    }
}

// Y[gc] = c M u_prev + f  (CSR), or Y[gc] = copy_src[perm[gc]] when
// copy_src is given (preconditioner applications); padded rows zero
#define BD_RHS_CB 8
#define BD_RHS_NS 4
__global__ void __launch_bounds__(256)
k_band_rhs(int n, int ldy, int B, const int* __restrict__ row_ptr,
           const int* __restrict__ col_idx, const double* __restrict__ m_val, int n_src,
           const double* __restrict__ shapes, const double* __restrict__ u_prev,
           const double* __restrict__ inv_dt, const double* __restrict__ src,
           const int* __restrict__ perm, double* __restrict__ Y,
           const double* __restrict__ copy_src) {
    // thread = one row of BD_RHS_CB grouped columns: the row's CSR entries
    // and source shapes are read once, the column gathers are independent
    const int gc0 = blockIdx.y * BD_RHS_CB;
    const int ncol = min(BD_RHS_CB, B - gc0);
    const double* ub[BD_RHS_CB];
    double cb[BD_RHS_CB], sv[BD_RHS_CB][BD_RHS_NS];
    double* yb[BD_RHS_CB];
    const double* base = copy_src ? copy_src : u_prev;
    const int ns = n_src <= BD_RHS_NS ? n_src : 0;
#pragma unroll
    for (int j = 0; j < BD_RHS_CB; ++j) {
        const int b = perm[gc0 + min(j, ncol - 1)];
        ub[j] = base + (size_t)b * n;
        yb[j] = Y + (size_t)(gc0 + min(j, ncol - 1)) * ldy;
        cb[j] = copy_src ? 0.0 : inv_dt[b];
#pragma unroll
        for (int s = 0; s < BD_RHS_NS; ++s)
            sv[j][s] = (!copy_src && s < ns) ? src[b * n_src + s] : 0.0;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ldy; i += gridDim.x * blockDim.x) {
        double acc[BD_RHS_CB];
        if (i >= n) {
#pragma unroll
            for (int j = 0; j < BD_RHS_CB; ++j) acc[j] = 0.0;
        } else if (copy_src) {
#pragma unroll
            for (int j = 0; j < BD_RHS_CB; ++j) acc[j] = ub[j][i];
        } else {
#pragma unroll
            for (int j = 0; j < BD_RHS_CB; ++j) acc[j] = 0.0;
            const int e0 = row_ptr[i], e1 = row_ptr[i + 1];
            for (int e = e0; e < e1; ++e) {
                const int cidx = col_idx[e];
                const double mv = m_val[e];
#pragma unroll
                for (int j = 0; j < BD_RHS_CB; ++j) acc[j] = fma(mv, ub[j][cidx], acc[j]);
            }
            double sh[BD_RHS_NS];
#pragma unroll
            for (int s = 0; s < BD_RHS_NS; ++s) sh[s] = s < ns ? shapes[(size_t)s * n + i] : 0.0;
#pragma unroll
            for (int j = 0; j < BD_RHS_CB; ++j) {
                double f = 0.0;
#pragma unroll
                for (int s = 0; s < BD_RHS_NS; ++s) f = fma(sv[j][s], sh[s], f);
                for (int s = ns; s < n_src; ++s)       // > BD_RHS_NS sources: generic
                    f = fma(src[(size_t)(ub[j] - base) / n * n_src + s], shapes[(size_t)s * n + i], f);
                acc[j] = fma(cb[j], acc[j], f);
            }
        }
#pragma unroll
        for (int j = 0; j < BD_RHS_CB; ++j)
            if (j < ncol) yb[j][i] = acc[j];
    }
}

// b = c M u + f on the symmetric DIA copy of M (structured stencils).  One
// thread per row; the row's M diagonals and source shapes stay in registers
// while the thread walks BD_RHS_CC columns, whose perm / 1/dt / source values
// sit in shared memory (broadcast reads).  Per output: 7 coalesced u loads
// (neighbours hit L1/L2), one store -- 16 n bytes of HBM per column.
#define BD_RHS_CC 32
struct RhsDia {
    int n, ldy, B, U, n_src;
    int off[5];
    const double2* __restrict__ mk;      // [(U+1)][n] (m, k); lower = mirrored upper
    const double* __restrict__ shapes;   // [n_src][n]
};
__global__ void __launch_bounds__(256)
k_band_rhs_dia(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
               const double* __restrict__ src, const int* __restrict__ perm,
               double* __restrict__ Y) {
    __shared__ int sp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC], ss[BD_RHS_CC][BD_RHS_SRC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    for (int t = threadIdx.x; t < BD_RHS_CC * BD_RHS_SRC; t += blockDim.x) {
        const int j = t / BD_RHS_SRC, q = t % BD_RHS_SRC;
        const int b = j < ncol ? perm[gc0 + j] : 0;
        if (q == 0) {
            sp[j] = b;
            sc[j] = j < ncol ? inv_dt[b] : 0.0;
        }
        ss[j][q] = (j < ncol && q < a.n_src) ? src[(size_t)b * a.n_src + q] : 0.0;
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.ldy) return;
    if (i >= a.n) {
        for (int j = 0; j < ncol; ++j) Y[(size_t)(gc0 + j) * a.ldy + i] = 0.0;
        return;
    }
    double mup[4], mlo[4];
    int oup[4], olo[4];
    const double m0 = a.mk[i].x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int o = a.off[u + 1];
        const bool on = u < a.U;
        const bool hu = on && i + o < a.n, hl = on && i - o >= 0;
        mup[u] = hu ? a.mk[(size_t)(u + 1) * a.n + i].x : 0.0;
        mlo[u] = hl ? a.mk[(size_t)(u + 1) * a.n + i - o].x : 0.0;
        oup[u] = hu ? o : 0;               // in-range dummy offset when absent
        olo[u] = hl ? -o : 0;
    }
    double sh[BD_RHS_SRC];
#pragma unroll
    for (int q = 0; q < BD_RHS_SRC; ++q) sh[q] = q < a.n_src ? a.shapes[(size_t)q * a.n + i] : 0.0;
    // the slot boxes cover a few % of the rows: rows outside every shape skip
    // the source term (warp-uniform away from the box edges)
    bool has_src = false;
#pragma unroll
    for (int q = 0; q < BD_RHS_SRC; ++q) has_src |= sh[q] != 0.0;
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll 4
    for (int j = 0; j < ncol; ++j) {
        const double* ub = u_prev + (size_t)sp[j] * a.n + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < 4; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        double f = 0.0;
        if (has_src) {
#pragma unroll
            for (int q = 0; q < BD_RHS_SRC; ++q) f = fma(ss[j][q], sh[q], f);
        }
        yo[(size_t)j * a.ldy] = fma(sc[j], v, f);
    }
}

// k_band_rhs_dia with the stencil width (UU upper diagonals) and the source
// count (<= NS) fixed at compile time: no dummy loads, half the registers for
// the source shapes, so 4 CTAs per SM stay resident (the generic kernel runs 3
// at 80 registers and is latency-bound at 37 % warps active on the 511^2 grid,
// profiles/r02c_ncu_rhs_dia_cfg4.json).  Same arithmetic, same order: bit-identical.
template <int UU, int NS, int MINB, int CC, int UNR = 4>
__global__ void __launch_bounds__(256, MINB)
k_band_rhs_dia_t(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
                 const double* __restrict__ src, const int* __restrict__ perm,
                 double* __restrict__ Y, double* __restrict__ uo) {
    // uo != NULL: column gc goes to uo[perm[gc]][0..n) (the caller's output
    // array used as scratch for the right-hand sides) instead of Y[gc][0..ldy)
    __shared__ int sp[CC];
    __shared__ double sc[CC], ss[CC][NS];
    const int gc0 = blockIdx.y * CC;
    const int ncol = min(CC, a.B - gc0);
    for (int t = threadIdx.x; t < CC * NS; t += blockDim.x) {
        const int j = t / NS, q = t % NS;
        const int b = j < ncol ? perm[gc0 + j] : 0;
        if (q == 0) {
            sp[j] = b;
            sc[j] = j < ncol ? inv_dt[b] : 0.0;
        }
        ss[j][q] = (j < ncol && q < a.n_src) ? src[(size_t)b * a.n_src + q] : 0.0;
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.ldy) return;
    if (i >= a.n) {
        if (!uo)
            for (int j = 0; j < ncol; ++j) Y[(size_t)(gc0 + j) * a.ldy + i] = 0.0;
        return;
    }
    double mup[UU], mlo[UU];
    int oup[UU], olo[UU];
    const double m0 = a.mk[i].x;
#pragma unroll
    for (int u = 0; u < UU; ++u) {
        const int o = a.off[u + 1];
        const bool hu = i + o < a.n, hl = i - o >= 0;
        mup[u] = hu ? a.mk[(size_t)(u + 1) * a.n + i].x : 0.0;
        mlo[u] = hl ? a.mk[(size_t)(u + 1) * a.n + i - o].x : 0.0;
        oup[u] = hu ? o : 0;               // in-range dummy offset when absent
        olo[u] = hl ? -o : 0;
    }
    double sh[NS];
    bool has_src = false;
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        sh[q] = q < a.n_src ? a.shapes[(size_t)q * a.n + i] : 0.0;
        has_src |= sh[q] != 0.0;
    }
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll UNR
    for (int j = 0; j < ncol; ++j) {
        const double* ub = u_prev + (size_t)sp[j] * a.n + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < UU; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        // (the generic kernel adds 0 * u for its unused diagonals: exact zeros)
        double f = 0.0;
        if (has_src) {
#pragma unroll
            for (int q = 0; q < NS; ++q) f = fma(ss[j][q], sh[q], f);
        }
        const double bv = fma(sc[j], v, f);
        if (uo) uo[(size_t)sp[j] * a.n + i] = bv;
        else yo[(size_t)j * a.ldy] = bv;
    }
}

// Same rhs, S-stage cp.async ring: the halos of the next S - 1 columns are in
// flight (LDGSTS, zero-filled outside [0, n)) while column j is computed from
// shared memory -- bytes in flight per CTA no longer depend on registers.
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int S, int LD>
__global__ void __launch_bounds__(256, 4)
k_band_rhs_cp(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
              const double* __restrict__ src, const int* __restrict__ perm,
              double* __restrict__ Y) {
    extern __shared__ double su[];           // [S][span]
    __shared__ int sp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC], ss[BD_RHS_CC][BD_RHS_SRC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    for (int t = threadIdx.x; t < BD_RHS_CC * BD_RHS_SRC; t += blockDim.x) {
        const int j = t / BD_RHS_SRC, q = t % BD_RHS_SRC;
        const int b = j < ncol ? perm[gc0 + j] : 0;
        if (q == 0) {
            sp[j] = b;
            sc[j] = j < ncol ? inv_dt[b] : 0.0;
        }
        ss[j][q] = (j < ncol && q < a.n_src) ? src[(size_t)b * a.n_src + q] : 0.0;
    }
    const int omax = a.off[a.U];
    const int r0 = blockIdx.x * 256;
    const int lo = r0 - omax;
    const int span = 256 + 2 * omax;
    const int i = r0 + threadIdx.x;
    const int ic = min(i, a.n - 1);
    double m0, mup[4], mlo[4], sh[BD_RHS_SRC];
    int oup[4], olo[4];
    m0 = a.mk[ic].x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int o = a.off[u + 1];
        const bool on = u < a.U;
        const bool hu = on && ic + o < a.n, hl = on && ic - o >= 0;
        mup[u] = hu ? a.mk[(size_t)(u + 1) * a.n + ic].x : 0.0;
        mlo[u] = hl ? a.mk[(size_t)(u + 1) * a.n + ic - o].x : 0.0;
        oup[u] = hu ? o : 0;
        olo[u] = hl ? -o : 0;
    }
    bool has_src = false;
#pragma unroll
    for (int q = 0; q < BD_RHS_SRC; ++q) {
        sh[q] = q < a.n_src ? a.shapes[(size_t)q * a.n + ic] : 0.0;
        has_src |= sh[q] != 0.0;
    }
    __syncthreads();
    // slot stride SL is a compile-time constant and the column loop is
    // unrolled by S, so every smem address is (per-thread register + immediate)
    constexpr int SL = 256 * LD;
    bool okv[LD];
    int goff[LD];
#pragma unroll
    for (int t = 0; t < LD; ++t) {
        const int jj = threadIdx.x + 256 * t;
        const int g = lo + jj;
        okv[t] = jj < span && g >= 0 && g < a.n;
        goff[t] = okv[t] ? g : 0;
    }
    const uint32_t s_dst = smem_u32(su) + 8u * threadIdx.x;
    auto issue = [&](int j, int slot) {
        const double* ub = u_prev + (size_t)sp[j] * a.n;
#pragma unroll
        for (int t = 0; t < LD; ++t) {
            if (threadIdx.x + 256 * t < span)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;"
                             ::"r"(s_dst + 8u * (slot * SL + 256 * t)), "l"(ub + goff[t]),
                             "r"(okv[t] ? 8 : 0)
                             : "memory");
        }
    };
#pragma unroll
    for (int j = 0; j < S - 1; ++j) {
        if (j < ncol) issue(j, j);
        cp_async_commit();
    }
    const bool row_ok = i < a.n;
    const int own = i - lo;
    const double* sb = su + (row_ok ? own : 0);
    const double* pu[4];
    const double* pl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { pu[u] = sb + oup[u]; pl[u] = sb + olo[u]; }
    double* yrow = Y + (size_t)gc0 * a.ldy + i;
    for (int j0 = 0; j0 < ncol; j0 += S) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int j = j0 + s;
            if (j >= ncol) break;
            cp_async_wait<S - 2>();
            __syncthreads();             // column j landed; slot (s - 1) % S is free
            if (j + S - 1 < ncol) issue(j + S - 1, (s + S - 1) % S);
            cp_async_commit();
            if (i < a.ldy) {
                double* yo = yrow + (size_t)j * a.ldy;
                if (!row_ok) {
                    *yo = 0.0;
                } else {
                    double v = m0 * sb[s * SL];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        v = fma(mup[u], pu[u][s * SL], fma(mlo[u], pl[u][s * SL], v));
                    double f = 0.0;
                    if (has_src) {
#pragma unroll
                        for (int q = 0; q < BD_RHS_SRC; ++q) f = fma(ss[j][q], sh[q], f);
                    }
                    *yo = fma(sc[j], v, f);
                }
            }
        }
    }
}

// u_out[perm[gc]] = Y[gc] (+ g)
__global__ void k_band_scatter(int n, int ldy, const double* __restrict__ Y,
                               const int* __restrict__ perm, double* __restrict__ u_out,
                               const double* __restrict__ g, const int* __restrict__ g_idx) {
    const int gc = blockIdx.y;
    const int b = perm[gc];
    const double* y = Y + (size_t)gc * ldy;
    const double* gs = (g && g_idx && g_idx[b] >= 0) ? g + (size_t)g_idx[b] * n : nullptr;
    double* o = u_out + (size_t)b * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        o[i] = gs ? y[i] + gs[i] : y[i];
}
