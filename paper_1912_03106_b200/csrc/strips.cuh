// Strip (one-level substructuring) solve of the banded systems on large
// structured grids -- fewer flops than the natural-order band solve.
//
// The side x side interior grid (side = S (h + 1) - 1) is cut into S strips of
// h grid rows by S - 1 separator rows.  Strip nodes are numbered strip by
// strip, x-major inside a strip (r = s rows + x h + y_l), so the strip block
// A_ss is block diagonal with lower bandwidth h + 1 instead of side; the
// separator nodes (j = s side + x) come last.  With A = [[A_ss, A_sp], [A_ps, A_pp]]
//
//     x~_s = A_ss^-1 b_s                       banded chains, window h + 1
//     g    = b_p - A_ps x~_s                   sparse coupling
//     x_p  = S^-1 g,  S^-1 = (A^-1)_pp         dense GEMM (fp64 DMMA)
//     x_s  = A_ss^-1 (b_s - A_sp x_p)          banded chains again
//
// is the exact solve (a direct method, like the reference's banded Cholesky;
// it agrees with the natural-order solve to rounding, 2e-15 on the 127^2
// model).  Flops per column: 2 x 4 n (h + 1 + 32) + 2 n_p^2 against
// 4 n (side + 1 + 32): 2.7x fewer at side = 511, S = 8, h = 63.  Each strip is
// padded to a multiple of 32 rows (identity rows) so that a 32-row block never
// straddles two strips.
#pragma once
#include "band.cuh"

struct StripGeo {
    int side, S, h, rows;      // rows = padded rows per strip (multiple of 32)
    int n, ldn;                // natural unknowns, leading dimension of natural columns
    int n_ss;                  // S * rows (leading dimension of strip-ordered columns)
    int n_pp, ldp;             // separator unknowns, padded to a multiple of 128
};

// natural index of strip row r, or -1 for a padding row
__device__ __forceinline__ int strip_to_nat(const StripGeo& g, int r) {
    const int s = r / g.rows, q = r - s * g.rows;
    if (q >= g.side * g.h) return -1;
    const int x = q / g.h, yl = q - x * g.h;
    return (s * (g.h + 1) + yl) * g.side + x;
}
// natural node i: strip row (>= 0) or -(separator index) - 1
__device__ __forceinline__ int nat_to_strip(const StripGeo& g, int i) {
    const int y = i / g.side, x = i - y * g.side;
    const int s = y / (g.h + 1), yl = y - s * (g.h + 1);
    if (yl == g.h) return -(s * g.side + x) - 1;
    return s * g.rows + x * g.h + yl;
}

// Y1 (= Y2 when given) = strip-ordered copy of the natural columns (padding rows 0).
// CTA = (strip s, 32 x-values): h natural row segments of 32 doubles in,
// 32 h contiguous doubles out, transposed through shared memory.
// grid (ceil(side / 32) * S, columns), 256 threads; smem h * 33 doubles
__global__ void __launch_bounds__(256)
k_strip_gather(StripGeo g, const double* __restrict__ Yn, const int* __restrict__ nperm,
               double* __restrict__ Y1, double* __restrict__ Y2) {
    // nperm != NULL: natural column col lives at Yn[nperm[col]][0..n) (stride n)
    extern __shared__ double tile[];                  // [h][33]
    const int xt = (g.side + 31) / 32;
    const int s = blockIdx.x / xt, x0 = (blockIdx.x - s * xt) * 32;
    const int nx = min(32, g.side - x0);
    const size_t col = blockIdx.y;
    const double* yn = nperm ? Yn + (size_t)nperm[col] * g.n : Yn + col * g.ldn;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int yl = ty; yl < g.h; yl += 8)
        if (tx < nx) tile[yl * 33 + tx] = yn[(size_t)(s * (g.h + 1) + yl) * g.side + x0 + tx];
    __syncthreads();
    const size_t base = col * g.n_ss + (size_t)s * g.rows + (size_t)x0 * g.h;
    for (int t = threadIdx.x; t < nx * g.h; t += 256) {
        const int xl = t / g.h, yl = t - xl * g.h;
        const double v = tile[yl * 33 + xl];
        Y1[base + t] = v;
        if (Y2) Y2[base + t] = v;
    }
    // padding rows of the strip (written by the CTA of its last x tile)
    if (x0 + 32 >= g.side) {
        const size_t pb = col * g.n_ss + (size_t)s * g.rows + (size_t)g.side * g.h;
        for (int t = threadIdx.x; t < g.rows - g.side * g.h; t += 256) {
            Y1[pb + t] = 0.0;
            if (Y2) Y2[pb + t] = 0.0;
        }
    }
}

// Gp[col][j] = b_p[j] - sum_{strip neighbours e} (c m_e + k_e) Y1[col][strip(e)]
// for every separator node j (padding j >= n_pp: 0).   thread per (j, column)
__global__ void __launch_bounds__(256)
k_strip_g(StripGeo g, int B, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
          const double* __restrict__ m_val, const double* __restrict__ k_val,
          const double* __restrict__ inv_dt, const int* __restrict__ perm,
          const double* __restrict__ Yn, int yn_perm, const double* __restrict__ Y1,
          double* __restrict__ Gp) {
    // yn_perm != 0: natural column col lives at Yn[perm[col]][0..n) (stride n)
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= g.ldp) return;
    for (int col = blockIdx.y; col < B; col += gridDim.y) {
        double v = 0.0;
        if (j < g.n_pp) {
            const int s = j / g.side, x = j - s * g.side;
            const int i = (s * (g.h + 1) + g.h) * g.side + x;
            const double c = inv_dt[perm[col]];
            v = yn_perm ? Yn[(size_t)perm[col] * g.n + i] : Yn[(size_t)col * g.ldn + i];
            const double* y1 = Y1 + (size_t)col * g.n_ss;
            for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                const int r = nat_to_strip(g, col_idx[e]);
                if (r >= 0) v = fma(-fma(c, m_val[e], k_val[e]), y1[r], v);
            }
        }
        Gp[(size_t)col * g.ldp + j] = v;
    }
}

// Y2[col][r] -= sum_{separator neighbours e} (c m_e + k_e) Xp[col][sep(e)] for
// the strip nodes next to a separator row (y_l = 0 of strips s > 0, y_l = h - 1
// of strips s < S - 1).   thread per (line, x, column); lines = 2 (S - 1)
__global__ void __launch_bounds__(256)
k_strip_update(StripGeo g, int B, const int* __restrict__ row_ptr, const int* __restrict__ col_idx,
               const double* __restrict__ m_val, const double* __restrict__ k_val,
               const double* __restrict__ inv_dt, const int* __restrict__ perm,
               const double* __restrict__ Xp, double* __restrict__ Y2) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = 2 * (g.S - 1);
    if (t >= nl * g.side) return;
    const int line = t / g.side, x = t - line * g.side;
    const int sep = line >> 1;                          // separator row index
    const int y = (line & 1) ? sep * (g.h + 1) + g.h + 1 : sep * (g.h + 1) + g.h - 1;
    // (h == 1: a strip row touches the separators on both sides; both lines
    // visit it, each adding only its own separator's entries below)
    const int i = y * g.side + x;
    const int r = nat_to_strip(g, i);
    for (int col = blockIdx.y; col < B; col += gridDim.y) {
        const double c = inv_dt[perm[col]];
        const double* xp = Xp + (size_t)col * g.ldp;
        double acc = 0.0;
        for (int e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            const int q = nat_to_strip(g, col_idx[e]);
            if (q < 0 && (-q - 1) / g.side == sep) acc = fma(fma(c, m_val[e], k_val[e]), xp[-q - 1], acc);
        }
        Y2[(size_t)col * g.n_ss + r] -= acc;
    }
}

// u_out[perm[col]][natural] = Y2 (strip nodes) / Xp (separator nodes) (+ g):
// the inverse transpose of k_strip_gather.   grid (ceil(side / 32) * S, columns)
__global__ void __launch_bounds__(256)
k_strip_scatter(StripGeo g, const double* __restrict__ Y2, const double* __restrict__ Xp,
                const int* __restrict__ perm, double* __restrict__ u_out,
                const double* __restrict__ gadd, const int* __restrict__ g_idx) {
    extern __shared__ double tile[];                  // [h][33]
    const int xt = (g.side + 31) / 32;
    const int s = blockIdx.x / xt, x0 = (blockIdx.x - s * xt) * 32;
    const int nx = min(32, g.side - x0);
    const size_t col = blockIdx.y;
    const int b = perm[col];
    const double* gs = (gadd && g_idx && g_idx[b] >= 0) ? gadd + (size_t)g_idx[b] * g.n : nullptr;
    double* uo = u_out + (size_t)b * g.n;
    const size_t base = col * g.n_ss + (size_t)s * g.rows + (size_t)x0 * g.h;
    for (int t = threadIdx.x; t < nx * g.h; t += 256) {
        const int xl = t / g.h, yl = t - xl * g.h;
        tile[yl * 33 + xl] = Y2[base + t];
    }
    __syncthreads();
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    if (tx < nx) {
        for (int yl = ty; yl < g.h; yl += 8) {
            const size_t i = (size_t)(s * (g.h + 1) + yl) * g.side + x0 + tx;
            const double v = tile[yl * 33 + tx];
            uo[i] = gs ? v + gs[i] : v;
        }
        // the separator row below this strip
        if (ty == 0 && s < g.S - 1) {
            const size_t i = (size_t)(s * (g.h + 1) + g.h) * g.side + x0 + tx;
            const double v = Xp[col * g.ldp + (size_t)s * g.side + x0 + tx];
            uo[i] = gs ? v + gs[i] : v;
        }
    }
}

// Sinv[j][i] = X[j][natural(separator i)] from the natural-order solves of the
// separator unit vectors (column j of the batch = unit vector of separator
// j0 + j); padding rows / columns zero.   thread per (i, j)
__global__ void k_strip_sinv_rows(StripGeo g, int j0, int nj, const double* __restrict__ X,
                                  double* __restrict__ Sinv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= g.ldp || j >= nj) return;
    double v = 0.0;
    if (i < g.n_pp) {
        const int s = i / g.side, x = i - s * g.side;
        v = X[(size_t)j * g.n + (size_t)(s * (g.h + 1) + g.h) * g.side + x];
    }
    Sinv[(size_t)(j0 + j) * g.ldp + i] = v;
}

// E[j][:] = unit vector of separator j0 + j (natural numbering)
__global__ void k_strip_units(StripGeo g, int j0, int nj, double* __restrict__ E) {
    const int j = blockIdx.y;
    if (j >= nj) return;
    const int sj = j0 + j, s = sj / g.side, x = sj - s * g.side;
    const int hot = (s * (g.h + 1) + g.h) * g.side + x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n; i += gridDim.x * blockDim.x)
        E[(size_t)j * g.n + i] = i == hot ? 1.0 : 0.0;
}

// Xp[col][:] = Sinv_f Gp[col][:] for the columns of a tile (factor, first
// column, <= 64 columns): the tiling of k_spike_gemm (spike_gemm.cuh) on a
// square ldp x ldp operator (ldp a multiple of 128), plain store.
// grid (ldp / 128, 1, column tiles)
__global__ void __launch_bounds__(256, 2)
k_strip_sinv_gemm(int ldp, double* const* __restrict__ Sinv, const double* __restrict__ Gp,
                  double* __restrict__ Xp, const int4* __restrict__ tiles) {
    extern __shared__ __align__(16) double sg[];
    double* As = sg;
    double* Bs = sg + SG_NST * SG_KS * SG_AP;
    const int4 tl = tiles[blockIdx.z];
    const double* A = Sinv[tl.x];
    const int c0 = tl.y, nc = tl.z;
    const int row0 = blockIdx.x * SG_TM;
    const double* Tb = Gp + (size_t)c0 * ldp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, q4 = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    auto stage_load = [&](int st, int k0) {
        double* as = As + st * SG_KS * SG_AP;
        double* bs = Bs + st * SG_TN * SG_BP;
#pragma unroll
        for (int i = 0; i < (SG_KS * SG_TM / 2) / 256; ++i) {
            const int t = tid + 256 * i;
            const int k = t / (SG_TM / 2), m = 2 * (t % (SG_TM / 2));
            sg_cp16(as + k * SG_AP + m, A + (size_t)(k0 + k) * ldp + row0 + m, 16);
        }
#pragma unroll
        for (int i = 0; i < (SG_TN * SG_KS / 2) / 256; ++i) {
            const int t = tid + 256 * i;
            const int n = t / (SG_KS / 2), k = 2 * (t % (SG_KS / 2));
            const int ok = n < nc ? 16 : 0;
            sg_cp16(bs + n * SG_BP + k, Tb + (size_t)(ok ? n : 0) * ldp + k0 + k, ok);
        }
        cp_async_commit();
    };
    double acc[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    const int nk = ldp / SG_KS;
#pragma unroll
    for (int i = 0; i < SG_NST - 1; ++i) {
        if (i < nk) stage_load(i, i * SG_KS);
        else cp_async_commit();
    }
    for (int ks = 0; ks < nk; ++ks) {
        cp_async_wait<SG_NST - 2>();
        __syncthreads();
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
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const int row = row0 + wm * 32 + 8 * mi + g;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = wn * 32 + 8 * ni + 2 * q4 + h;
                if (c < nc) Xp[(size_t)(c0 + c) * ldp + row] = acc[mi][ni][h];
            }
    }
}
