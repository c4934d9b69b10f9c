// Streamed batched Jacobi-PCG on a symmetric banded (DIA) operator.
//
// pg_add_level converts the CSR it is given into this layout whenever the
// pattern has at most PG_DIA_MAX distinct upper offsets and M, K are exactly
// symmetric (every FE mass / stiffness pair on a structured grid is):
//
//   mk[u][i] = (M[i][i+o_u], K[i][i+o_u])   u = 0 (diagonal) .. U
//   A[i][i-o_u] = A[i-o_u][i] read from mk[u][i-o_u]
//
// so a row costs 16 (U+1) bytes of matrix from L2 instead of 20 nnz bytes of
// CSR, no index loads, and every access is coalesced.  Vectors are internal
// [B][ld] buffers (ld a multiple of 32 doubles) so halo loads are 16-byte
// vector loads.  Per active column and PCG iteration the HBM traffic is
// 64 n bytes:
//
//   k_dia_dir : read r, p_old (halo) -> p_new = D^-1 r + beta p_old into smem,
//               write own rows of p_new, q = A p_new, partial p.q      24 n
//   k_dia_upd : read p_new (halo), x, r -> q = A p_new (recomputed),
//               x += alpha p, r -= alpha q, write x, r, partial r.z, r.r 40 n
//
// Memory-level parallelism: halo staging issues 4 x 16-byte loads per array
// per thread before consuming any (>= 32 KB in flight per CTA), own-row
// operands are prefetched into registers before the staging barrier, and
// CTAs are sized for >= 3 resident per SM.
#pragma once
#include "common.cuh"
#include "pcg.cuh"

#define PG_DIA_MAX 4          // max upper offsets (7-point stencil uses 3)
#define PG_DIA_NT 256

struct DiaLevel {
    int n, ld;
    int U;                      // number of upper offsets
    int off[PG_DIA_MAX + 1];    // off[0] = 0
    int omax;
    const double2* __restrict__ mk;    // [(U+1)][n] (m, k)
    int n_src;
    const double* __restrict__ shapes;
    int R, n_tiles;
};

struct DiaWork {
    double* x;                  // [B][ld] internal solution
    double* r;                  // [B][ld]
    double* p[2];               // [B][ld] ping-pong
};

__device__ __forceinline__ double2 ld2(const double* p) {
    return *reinterpret_cast<const double2*>(p);
}

// y_i = (cb M + K) p  for row i, p read from smem window sp (indexed by
// global row; caller guarantees [i - omax, i + omax] staged or out of range)
template <int UMAX>
__device__ __forceinline__ double dia_row(const DiaLevel& L, int i, double cb,
                                          const double* sp, const double2* dg,
                                          const double2* up, const double2* lo_) {
    double y = fma(cb, dg->x, dg->y) * sp[i];
#pragma unroll
    for (int u = 1; u <= UMAX; ++u) {
        const int o = L.off[u];
        const double au = fma(cb, up[u - 1].x, up[u - 1].y);
        const double al = fma(cb, lo_[u - 1].x, lo_[u - 1].y);
        if (i + o < L.n) y = fma(au, sp[i + o], y);
        if (i - o >= 0) y = fma(al, sp[i - o], y);
    }
    return y;
}

// load the (U+1) own + U mirrored matrix entries of row i
template <int UMAX>
__device__ __forceinline__ void dia_load_row(const DiaLevel& L, int i, double2& dg,
                                             double2 (&up)[UMAX], double2 (&lw)[UMAX]) {
    dg = __ldg(L.mk + i);
#pragma unroll
    for (int u = 1; u <= UMAX; ++u) {
        const int o = L.off[u];
        up[u - 1] = __ldg(L.mk + (size_t)u * L.n + i);
        lw[u - 1] = (i - o >= 0) ? __ldg(L.mk + (size_t)u * L.n + i - o) : make_double2(0.0, 0.0);
    }
}

__device__ __forceinline__ void tile_span(const DiaLevel& L, int tile, int& r0, int& r1,
                                          int& lo, int& hi) {
    r0 = tile * L.R;
    r1 = min(L.n, r0 + L.R);
    lo = max(0, r0 - L.omax) & ~1;            // even -> 16-byte aligned pairs
    hi = min(L.ld, (r1 + L.omax + 1) & ~1);   // even, within the padded row
}

// --- setup: x0 = guess or u_prev, r0 = b - A x0, |b|^2, rho0 ----------------------
template <int C, int UU>
__global__ void __launch_bounds__(PG_DIA_NT)
k_dia_setup(DiaLevel L, DiaWork V, PcgWork W, int B, const double* __restrict__ u_prev,
            const double* __restrict__ guess, const double* __restrict__ inv_dt,
            const double* __restrict__ src, double rtol2, int max_iters) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_DIA_NT / 32) * 3];
    __shared__ int s_flag;
    const int n = L.n, tile = blockIdx.x;
    int r0, r1, lo, hi;
    tile_span(L, tile, r0, r1, lo, hi);
    const int span = hi - lo;
    // smem: [C][2][span]: u_prev window, guess window
    for (int c = 0; c < C; ++c) {
        const int b = blockIdx.y * C + c;
        if (b >= B) break;
        const double* u = u_prev + (size_t)b * n;
        const double* g = guess ? guess + (size_t)b * n : nullptr;
        double* su = smem + (size_t)c * 2 * span;
        double* sg = su + span;
        for (int j = lo + threadIdx.x; j < hi; j += PG_DIA_NT) {
            su[j - lo] = j < n ? u[j] : 0.0;
            if (g) sg[j - lo] = j < n ? g[j] : 0.0;
        }
    }
    __syncthreads();
    for (int c = 0; c < C; ++c) {
        const int b = blockIdx.y * C + c;
        if (b >= B) break;                                  // uniform
        const double cb = inv_dt[b];
        const double* su = smem + (size_t)c * 2 * span - lo;
        const double* sg = guess ? su + span : su;
        double acc[3] = {0.0, 0.0, 0.0};
        for (int i = r0 + threadIdx.x; i < r1; i += PG_DIA_NT) {
            double2 dg, up[UU], lw[UU];
            dia_load_row<UU>(L, i, dg, up, lw);
            // M u and K x0 separately (b = cb M u + f, r = b - (cb M x0 + K x0))
            double mu = dg.x * su[i], mx = dg.x * sg[i], kx = dg.y * sg[i];
#pragma unroll
            for (int u = 1; u <= UU; ++u) {
                const int o = L.off[u];
                if (i + o < n) {
                    mu = fma(up[u - 1].x, su[i + o], mu);
                    mx = fma(up[u - 1].x, sg[i + o], mx);
                    kx = fma(up[u - 1].y, sg[i + o], kx);
                }
                if (i - o >= 0) {
                    mu = fma(lw[u - 1].x, su[i - o], mu);
                    mx = fma(lw[u - 1].x, sg[i - o], mx);
                    kx = fma(lw[u - 1].y, sg[i - o], kx);
                }
            }
            double f = 0.0;
            for (int s = 0; s < L.n_src; ++s)
                f = fma(src[b * L.n_src + s], __ldg(L.shapes + (size_t)s * n + i), f);
            const double bi = fma(cb, mu, f);
            const double ri = guess ? bi - fma(cb, mx, kx) : f - kx;
            V.x[(size_t)b * L.ld + i] = sg[i];
            V.r[(size_t)b * L.ld + i] = ri;
            acc[0] = fma(bi, bi, acc[0]);
            acc[1] = fma(ri * ri, dinv_of(cb, dg.x, dg.y), acc[1]);
            acc[2] = fma(ri, ri, acc[2]);
        }
        block_sum<3>(acc, red);
        if (threadIdx.x == 0) {
            double* pp = W.partial + ((size_t)b * L.n_tiles + tile) * 3;
            pp[0] = acc[0]; pp[1] = acc[1]; pp[2] = acc[2];
        }
        if (column_last(W.cnt, b, L.n_tiles, &s_flag) && threadIdx.x == 0) {
            double bb = 0.0, rz = 0.0, rr = 0.0;
            const double* pp = W.partial + (size_t)b * L.n_tiles * 3;
            for (int t = 0; t < L.n_tiles; ++t) { bb += pp[3 * t]; rz += pp[3 * t + 1]; rr += pp[3 * t + 2]; }
            W.bnorm2[b] = bb;
            W.tol2[b] = rtol2 * bb;
            W.rho[b] = rz;
            W.beta[b] = 0.0;
            W.it[b] = 0;
            W.flag[b] = (rr <= rtol2 * bb || rr == 0.0) ? COL_CONVERGED
                        : (max_iters <= 0 ? COL_MAXIT : COL_ACTIVE);
        }
    }
    if (grid_last(W.gcnt, &s_flag)) {
        __shared__ int s_scan[PG_DIA_NT + 1];
        int base = 0;
        for (int off = 0; off < B; off += PG_DIA_NT) {
            const int b = off + threadIdx.x;
            const int keep = (b < B) && (((volatile int*)W.flag)[b] == COL_ACTIVE);
            s_scan[threadIdx.x] = keep;
            __syncthreads();
            for (int d = 1; d < PG_DIA_NT; d <<= 1) {
                const int v = (threadIdx.x >= (unsigned)d) ? s_scan[threadIdx.x - d] : 0;
                __syncthreads();
                s_scan[threadIdx.x] += v;
                __syncthreads();
            }
            if (keep) W.act[0][base + s_scan[threadIdx.x] - 1] = b;
            const int tot = s_scan[PG_DIA_NT - 1];
            __syncthreads();
            base += tot;
        }
        if (threadIdx.x == 0) W.nact[0] = base;
    }
}

// --- direction update + SpMV + p.q --------------------------------------------------
template <int C, int UU>
__global__ void __launch_bounds__(PG_DIA_NT, 2)
k_dia_dir(DiaLevel L, DiaWork V, PcgWork W, int cur, const double* __restrict__ inv_dt) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_DIA_NT / 32)];
    __shared__ int s_flag;
    const int na = W.nact[cur];
    const int slot0 = blockIdx.y * C;
    if (slot0 >= na) return;
    const int tile = blockIdx.x;
    int r0, r1, lo, hi;
    tile_span(L, tile, r0, r1, lo, hi);
    const int span = hi - lo;
    const double* __restrict__ p_old = V.p[cur];
    double* __restrict__ p_new = V.p[cur ^ 1];
    const int nc = min(C, na - slot0);

    // stage p_new = D^-1 r + beta p_old over the halo window, column by column
    for (int c = 0; c < nc; ++c) {
        const int b = W.act[cur][slot0 + c];
        const double cb = inv_dt[b];
        const double beta = W.beta[b];
        const bool first = W.it[b] == 0;
        const double* rr = V.r + (size_t)b * L.ld;
        const double* po = p_old + (size_t)b * L.ld;
        double* sp = smem + (size_t)c * span;
        for (int base = lo + 2 * threadIdx.x; base < hi; base += 2 * PG_DIA_NT * 4) {
            double2 rv[4], pv[4], dv[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = base + 2 * PG_DIA_NT * k;
                if (j < hi) {
                    rv[k] = ld2(rr + j);
                    pv[k] = first ? make_double2(0.0, 0.0) : ld2(po + j);
                    dv[2 * k] = j < L.n ? __ldg(L.mk + j) : make_double2(1.0, 1.0);
                    dv[2 * k + 1] = j + 1 < L.n ? __ldg(L.mk + j + 1) : make_double2(1.0, 1.0);
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int j = base + 2 * PG_DIA_NT * k;
                if (j < hi) {
                    const double z0 = rv[k].x * dinv_of(cb, dv[2 * k].x, dv[2 * k].y);
                    const double z1 = rv[k].y * dinv_of(cb, dv[2 * k + 1].x, dv[2 * k + 1].y);
                    double2 o;
                    o.x = first ? z0 : fma(beta, pv[k].x, z0);
                    o.y = first ? z1 : fma(beta, pv[k].y, z1);
                    *reinterpret_cast<double2*>(sp + j - lo) = o;
                }
            }
        }
    }
    __syncthreads();
    double pq[C];
#pragma unroll
    for (int c = 0; c < C; ++c) pq[c] = 0.0;
    double cbv[C];
    int bv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        bv[c] = c < nc ? W.act[cur][slot0 + c] : 0;
        cbv[c] = inv_dt[bv[c]];
    }
    for (int i = r0 + threadIdx.x; i < r1; i += PG_DIA_NT) {
        double2 dg, up[UU], lw[UU];
        dia_load_row<UU>(L, i, dg, up, lw);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c >= nc) break;
            const double* sp = smem + (size_t)c * span - lo;
            const double q = dia_row<UU>(L, i, cbv[c], sp, &dg, up, lw);
            const double pi = sp[i];
            pq[c] = fma(pi, q, pq[c]);
            p_new[(size_t)bv[c] * L.ld + i] = pi;
        }
    }
    for (int c = 0; c < nc; ++c) {
        const int b = W.act[cur][slot0 + c];
        double v[1] = {pq[c]};
        block_sum<1>(v, red);
        if (threadIdx.x == 0) W.partial[((size_t)b * L.n_tiles + tile) * 3] = v[0];
        if (column_last(W.cnt, b, L.n_tiles, &s_flag) && threadIdx.x == 0) {
            double s = 0.0;
            const double* pp = W.partial + (size_t)b * L.n_tiles * 3;
            for (int t = 0; t < L.n_tiles; ++t) s += pp[3 * t];
            if (s > 0.0) {
                W.alpha[b] = W.rho[b] / s;
            } else {
                W.alpha[b] = 0.0;
                W.flag[b] = COL_BREAKDOWN;
            }
        }
    }
}

// --- x, r update + r.z, r.r + convergence + compaction --------------------------------
template <int C, int UU>
__global__ void __launch_bounds__(PG_DIA_NT, 2)
k_dia_upd(DiaLevel L, DiaWork V, PcgWork W, int cur, const double* __restrict__ inv_dt,
          int max_iters) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_DIA_NT / 32) * 2];
    __shared__ int s_flag;
    __shared__ int s_scan[PG_DIA_NT + 1];
    const int na = W.nact[cur];
    const int slot0 = blockIdx.y * C;
    const int tile = blockIdx.x;
    if (slot0 < na) {
        int r0, r1, lo, hi;
        tile_span(L, tile, r0, r1, lo, hi);
        const int span = hi - lo;
        const double* __restrict__ p = V.p[cur ^ 1];
        const int nc = min(C, na - slot0);
        for (int c = 0; c < nc; ++c) {
            const int b = W.act[cur][slot0 + c];
            const double* pc = p + (size_t)b * L.ld;
            double* sp = smem + (size_t)c * span;
            for (int base = lo + 2 * threadIdx.x; base < hi; base += 2 * PG_DIA_NT * 4) {
                double2 v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = base + 2 * PG_DIA_NT * k;
                    if (j < hi) v[k] = ld2(pc + j);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int j = base + 2 * PG_DIA_NT * k;
                    if (j < hi) *reinterpret_cast<double2*>(sp + j - lo) = v[k];
                }
            }
        }
        __syncthreads();
        double acc[C][2];
        double cbv[C], alv[C];
        int bv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            acc[c][0] = acc[c][1] = 0.0;
            bv[c] = c < nc ? W.act[cur][slot0 + c] : 0;
            cbv[c] = inv_dt[bv[c]];
            alv[c] = W.alpha[bv[c]];
        }
        for (int i = r0 + threadIdx.x; i < r1; i += PG_DIA_NT) {
            double2 dg, up[UU], lw[UU];
            dia_load_row<UU>(L, i, dg, up, lw);
            double xv[C], rv[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c < nc) {
                    xv[c] = V.x[(size_t)bv[c] * L.ld + i];
                    rv[c] = V.r[(size_t)bv[c] * L.ld + i];
                }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c >= nc) break;
                const double* sp = smem + (size_t)c * span - lo;
                const double q = dia_row<UU>(L, i, cbv[c], sp, &dg, up, lw);
                const double pi = sp[i];
                const size_t k = (size_t)bv[c] * L.ld + i;
                V.x[k] = fma(alv[c], pi, xv[c]);
                const double ri = fma(-alv[c], q, rv[c]);
                V.r[k] = ri;
                acc[c][0] = fma(ri * ri, dinv_of(cbv[c], dg.x, dg.y), acc[c][0]);
                acc[c][1] = fma(ri, ri, acc[c][1]);
            }
        }
        for (int c = 0; c < nc; ++c) {
            const int b = bv[c];
            double v[2] = {acc[c][0], acc[c][1]};
            block_sum<2>(v, red);
            if (threadIdx.x == 0) {
                double* pp = W.partial + ((size_t)b * L.n_tiles + tile) * 3;
                pp[1] = v[0]; pp[2] = v[1];
            }
            if (column_last(W.cnt, b, L.n_tiles, &s_flag) && threadIdx.x == 0) {
                double rz = 0.0, rr = 0.0;
                const double* pp = W.partial + (size_t)b * L.n_tiles * 3;
                for (int t = 0; t < L.n_tiles; ++t) { rz += pp[3 * t + 1]; rr += pp[3 * t + 2]; }
                const int it = W.it[b] + 1;
                W.it[b] = it;
                W.beta[b] = rz / W.rho[b];
                W.rho[b] = rz;
                atomicAdd(W.iters, 1ull);
                atomicAdd(W.iters + 1, 1ull);
                atomicMax(W.ictr, it);
                if (W.flag[b] == COL_ACTIVE) {
                    if (rr <= W.tol2[b] || rr == 0.0) W.flag[b] = COL_CONVERGED;
                    else if (it >= max_iters) {
                        W.flag[b] = COL_MAXIT;
                        atomicAdd(W.ictr + 1, 1);
                        atomicAdd(W.ictr + 2, 1);
                    }
                }
            }
        }
    }
    if (grid_last(W.gcnt, &s_flag))
        compact_active(W.act[cur], na, W.flag, W.act[cur ^ 1], &W.nact[cur ^ 1], s_scan);
}

// u_out[b] = x[b] (+ g[g_idx[b]])
__global__ void k_dia_finish(int n, int ld, int B, const double* __restrict__ x,
                             double* __restrict__ u, const double* __restrict__ g,
                             const int* __restrict__ g_idx) {
    const int b = blockIdx.y;
    const double* xs = x + (size_t)b * ld;
    const double* gs = (g && g_idx && g_idx[b] >= 0) ? g + (size_t)g_idx[b] * n : nullptr;
    double* us = u + (size_t)b * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        us[i] = gs ? xs[i] + gs[i] : xs[i];
}
