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
//  * k_band_solve<FWD/BWD>: each CTA walks all block rows for a chunk of BC
//    columns sharing one factor.  Per block row: TMA bulk-copies the next
//    block's operands (2-stage mbarrier ring) while the current block does
//        acc = rhs_blk - Lwin * y_window      (nb x W x BC)
//        y_blk = D^-1 acc                     (nb x nb x BC)
//    as fp64 tensor-core MMAs (mma.sync m8n8k4 f64: SASS DMMA), the window
//    living in a shared-memory ring of the last W/nb blocks.
//
// Explicit inverses of the 32 x 32 diagonal blocks turn the triangular
// solves into GEMMs; the factor is otherwise the same arithmetic as dpbtrf.
#pragma once
#include "common.cuh"
#include "tma.cuh"

#define BD_NB 32
#define BD_NT 256          // 8 warps: 4 row groups x 2 window halves

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// factorisation: one CTA per factor, 256 threads
// LB[i][d] = A[i][i-d] (d = 0..w), A = c M + K built from the CSR (lower part)
struct BandFactorArgs {
    int n, w, W, LDA, nblk;
    const int* row_ptr;
    const int* col_idx;
    const double* m_val;
    const double* k_val;
};

__global__ void __launch_bounds__(256)
k_band_build(BandFactorArgs a, const double* __restrict__ cvals, double* const* LBs) {
    const int f = blockIdx.y;
    const double c = cvals[f];
    double* LB = LBs[f];
    const int stride = a.w + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        double* row = LB + (size_t)i * stride;
        for (int d = 0; d <= a.w; ++d) row[d] = 0.0;
        for (int e = a.row_ptr[i]; e < a.row_ptr[i + 1]; ++e) {
            const int j = a.col_idx[e];
            if (j <= i) row[i - j] += fma(c, a.m_val[e], a.k_val[e]);
        }
    }
}

// smem: D[32][33], Dinv[32][33], P[w][33]
__global__ void __launch_bounds__(256)
k_band_factor(BandFactorArgs a, double* const* LBs, double* const* FLs, double* const* FUs,
              int* status) {
    extern __shared__ double sm[];
    const int f = blockIdx.x;
    double* LB = LBs[f];
    double* FL = FLs[f];
    double* FU = FUs[f];
    const int NB = BD_NB, S = NB + 1;
    double* D = sm;
    double* Di = D + NB * S;
    double* P = Di + NB * S;
    const int stride = a.w + 1;
    const int tid = threadIdx.x;
    auto lb = [&](int i, int j) -> double& { return LB[(size_t)i * stride + (i - j)]; };

    for (int k = 0; k < a.nblk; ++k) {
        const int k0 = k * NB;
        const int kb = min(NB, a.n - k0);
        // 1. diagonal block (padded with identity beyond n)
        for (int t = tid; t < NB * NB; t += blockDim.x) {
            const int i = t / NB, j = t % NB;
            double v = 0.0;
            if (i < kb && j < kb) {
                if (j <= i && i - j <= a.w) v = lb(k0 + i, k0 + j);
            } else if (i == j) {
                v = 1.0;
            }
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
                x[j] = (j < kb && gr - gc <= a.w) ? lb(gr, gc) : 0.0;
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
        // 5. solve operands of block k
        double* fl = FL + (size_t)k * NB * a.LDA;
        double* fu = FU + (size_t)k * NB * a.LDA;
        for (int t = tid; t < NB * a.LDA; t += blockDim.x) {
            const int i = t / a.LDA, j = t % a.LDA;
            double vl = 0.0, vu = 0.0;
            if (j < NB) {
                vl = Di[i * S + j];              // D^-1
                vu = Di[j * S + i];              // D^-T
            } else if (j < NB + a.W) {
                const int q = j - NB;            // window column
                // forward: L[k0+i][k0-W+q]  (final: earlier panels)
                const int gr = k0 + i, gc = k0 - a.W + q;
                if (i < kb && gc >= 0 && gr - gc <= a.w) vl = lb(gr, gc);
                // backward: L[k0+NB+q][k0+i] = P[q][i]
                if (q < m && i < kb && (r0 + q) - (k0 + i) <= a.w) vu = P[q * S + i];
            }
            fl[t] = vl;
            fu[t] = vu;
        }
        __syncthreads();
        // 6. trailing update of the band: A[r][s] -= P[r] . P[s], s <= r
        for (int t = tid; t < m * m; t += blockDim.x) {
            const int r = t / m, s = t % m;
            if (s > r || r - s > a.w) continue;
            double acc = 0.0;
#pragma unroll 8
            for (int j = 0; j < NB; ++j) acc = fma(P[r * S + j], P[s * S + j], acc);
            lb(r0 + r, r0 + s) -= acc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// batched solves
struct BandSolveArgs {
    int np, W, LDA, nblk, ldy;
    double* Y;                   // [n_cols][ldy] grouped columns, in place
    const int4* chunks;          // (factor, first grouped column, count, 0)
    double* const* F;            // per factor: FL or FU base
};

// smem layout (doubles): stage[2][NB * LDA], ring[NSLOT][NB][BC + 4], T[NB][BC + 4]
// 8 warps: warp w -> row group rg = w & 3 (rows 8 rg .. 8 rg + 7) and window
// half kh = w >> 2.  The window (NSLOT = W / 32 blocks, a power of two, so
// ring slots are masks) is fully unrolled; each warp keeps four independent
// DMMA accumulator chains; the two halves are summed through T.
template <int BC, int NSLOT, bool FWD>
__global__ void __launch_bounds__(BD_NT)
k_band_solve(BandSolveArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(8) uint64_t bar[2];
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    constexpr int NB = BD_NB, RS = BC + 4, NT8 = BC / 8;
    constexpr int W = NSLOT * NB;
    // per-half window rows: [kh * HALF, kh * HALF + HALF)
    constexpr int HALF = W / 2;
    double* stage = sm;
    double* ring = stage + 2 * (size_t)NB * a.LDA;
    double* T = ring + (size_t)NSLOT * NB * RS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, q4 = lane & 3;
    const int rg = warp & 3, kh = warp >> 2;
    const int lrow = 8 * rg + g;
    const uint32_t blk_bytes = (uint32_t)(NB * a.LDA * 8);

    for (int t = threadIdx.x; t < NSLOT * NB * RS; t += BD_NT) ring[t] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto blk_of = [&](int s) { return FWD ? s : a.nblk - 1 - s; };
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[0], blk_bytes);
        tma_load_1d(stage, F + (size_t)blk_of(0) * NB * a.LDA, blk_bytes, &bar[0]);
    }
    double nxt[NT8][2];
    auto load_rhs = [&](int s) {
        const int rrow = NB * blk_of(s) + lrow;
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int cc = 8 * nt + 2 * q4 + h;
                nxt[nt][h] = (kh == 0 && cc < ncol) ? a.Y[(size_t)(col0 + cc) * a.ldy + rrow] : 0.0;
            }
    };
    load_rhs(0);
    for (int s = 0; s < a.nblk; ++s) {
        const int k = blk_of(s);
        const int st = s & 1;
        if (threadIdx.x == 0 && s + 1 < a.nblk) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[st ^ 1], blk_bytes);
            tma_load_1d(stage + (size_t)(st ^ 1) * NB * a.LDA,
                        F + (size_t)blk_of(s + 1) * NB * a.LDA, blk_bytes, &bar[st ^ 1]);
        }
        double acc[4][NT8][2];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt) {
            acc[0][nt][0] = nxt[nt][0];
            acc[0][nt][1] = nxt[nt][1];
        }
        const int row = NB * k + lrow;
        if (s + 1 < a.nblk) load_rhs(s + 1);
        mbar_wait(&bar[st], (s >> 1) & 1);
        const double* Lt = stage + (size_t)st * NB * a.LDA;
        const double* Lrow = Lt + lrow * a.LDA + NB;
        // window: rows j in [kh*HALF, kh*HALF + HALF); block wbi = j / NB
        const int kbeg = kh * HALF;
#pragma unroll
        for (int jj = 0; jj < HALF; jj += 4) {
            const int j = kbeg + jj;                    // uniform per warp
            const int wbi = j / NB;                     // j multiple of 4: exact
            const int blk = FWD ? (k - NSLOT + wbi) : (k + 1 + wbi);
            const bool ok = FWD ? (blk >= 0) : (blk < a.nblk);
            const int slot = (FWD ? (k + wbi) : (k + 1 + wbi)) & (NSLOT - 1);
            const double av = -Lrow[j + q4];
            const double* rr = ring + ((size_t)slot * NB + (j % NB) + q4) * RS + g;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                const double bv = ok ? rr[8 * nt] : 0.0;
                dmma_8x8x4(acc[(jj >> 2) & 3][nt][0], acc[(jj >> 2) & 3][nt][1], av, bv);
            }
        }
        double r0v[NT8][2];
#pragma unroll
        for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                r0v[nt][h] = (acc[0][nt][h] + acc[1][nt][h]) + (acc[2][nt][h] + acc[3][nt][h]);
        if (kh == 1) {
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                T[lrow * RS + 8 * nt + 2 * q4] = r0v[nt][0];
                T[lrow * RS + 8 * nt + 2 * q4 + 1] = r0v[nt][1];
            }
        }
        __syncthreads();
        if (kh == 0) {
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt) {
                T[lrow * RS + 8 * nt + 2 * q4] += r0v[nt][0];
                T[lrow * RS + 8 * nt + 2 * q4 + 1] += r0v[nt][1];
            }
        }
        __syncthreads();
        if (kh == 0) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt) acc[c][nt][0] = acc[c][nt][1] = 0.0;
            const double* Ld = Lt + lrow * a.LDA;
#pragma unroll
            for (int kq = 0; kq < NB; kq += 4) {
                const double av = Ld[kq + q4];
                const double* tt = T + (kq + q4) * RS + g;
#pragma unroll
                for (int nt = 0; nt < NT8; ++nt)
                    dmma_8x8x4(acc[(kq >> 2) & 3][nt][0], acc[(kq >> 2) & 3][nt][1], av, tt[8 * nt]);
            }
            double* slot = ring + (size_t)(k & (NSLOT - 1)) * NB * RS;
#pragma unroll
            for (int nt = 0; nt < NT8; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cc = 8 * nt + 2 * q4 + h;
                    const double v = (acc[0][nt][h] + acc[1][nt][h]) + (acc[2][nt][h] + acc[3][nt][h]);
                    slot[lrow * RS + cc] = v;
                    if (cc < ncol) a.Y[(size_t)(col0 + cc) * a.ldy + row] = v;
                }
        }
        __syncthreads();
    }
}

// Y[gc] = c M u_prev + f  (CSR), padded rows zero
__global__ void k_band_rhs(int n, int ldy, const int* __restrict__ row_ptr,
                           const int* __restrict__ col_idx, const double* __restrict__ m_val,
                           int n_src, const double* __restrict__ shapes,
                           const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
                           const double* __restrict__ src, const int* __restrict__ perm,
                           double* __restrict__ Y) {
    const int gc = blockIdx.y;
    const int b = perm[gc];
    const double c = inv_dt[b];
    const double* u = u_prev + (size_t)b * n;
    double* y = Y + (size_t)gc * ldy;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ldy; i += gridDim.x * blockDim.x) {
        if (i >= n) { y[i] = 0.0; continue; }
        double mu = 0.0;
        for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) mu = fma(m_val[e], u[col_idx[e]], mu);
        double f = 0.0;
        for (int s = 0; s < n_src; ++s) f = fma(src[b * n_src + s], shapes[(size_t)s * n + i], f);
        y[i] = fma(c, mu, f);
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
