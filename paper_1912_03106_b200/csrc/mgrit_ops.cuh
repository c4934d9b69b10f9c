// MGRIT-side batched kernels: spatial restriction / prolongation between
// nested structured grids, C-point residual + norm + Joule loss, FAS RHS.
// States are [B][n] fp64 with x-fastest interior numbering on a grid of
// `side` x `side` interior nodes; coarse node (I, J) sits on fine node
// (2I+1, 2J+1) (0-based) -- the 2D form of the reference's field[1::2].
//
// Transfer arithmetic uses explicitly rounded adds/multiplies (no FMA
// contraction) in the same association as the CPU oracle, so transfers are
// bitwise identical to it.
#pragma once
#include "common.cuh"

// R(in)[I] on a fine grid of side sf, coarse side sc = (sf - 1) / 2.
// mode 0: injection (spatial.py:71); mode 1: full weighting.
__device__ __forceinline__ double restrict_at(const double* __restrict__ fin, int sf,
                                              int Ix, int Iy, int mode) {
    const int fx = 2 * Ix + 1, fy = 2 * Iy + 1;
    if (mode == 0) return fin[fy * sf + fx];
    double acc = 0.0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
        const double wy = dy == 0 ? 2.0 : 1.0;
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
            const double wx = dx == 0 ? 2.0 : 1.0;
            const double w = __dmul_rn(wy, wx) / 16.0;   // exact
            acc = __dadd_rn(acc, __dmul_rn(w, fin[(fy + dy) * sf + fx + dx]));
        }
    }
    return acc;
}

__global__ void k_restrict(int sf, int sc, int B, const double* __restrict__ in,
                           double* __restrict__ out, int mode) {
    const size_t nc = (size_t)sc * sc, nf = (size_t)sf * sf;
    const size_t total = nc * B;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const size_t b = k / nc, I = k % nc;
        const int Ix = (int)(I % sc), Iy = (int)(I / sc);
        out[k] = restrict_at(in + b * nf, sf, Ix, Iy, mode);
    }
}

// coarse padded value (zero Dirichlet ring), 1-based coarse indices
__device__ __forceinline__ double cval(const double* __restrict__ c, int sc, int I, int J) {
    return (I >= 1 && I <= sc && J >= 1 && J <= sc) ? c[(J - 1) * sc + (I - 1)] : 0.0;
}

// P(in)[i] for fine 0-based (x, y); mode 0 bilinear, 1 P1 on '/' diagonals.
__device__ __forceinline__ double prolong_at(const double* __restrict__ c, int sc,
                                             int x, int y, int mode) {
    const int ii = x + 1, jj = y + 1;          // 1-based fine indices
    const int I0 = ii >> 1, J0 = jj >> 1;
    const bool ie = !(ii & 1), je = !(jj & 1);
    if (ie && je) return cval(c, sc, I0, J0);
    if (ie) return __dmul_rn(0.5, __dadd_rn(cval(c, sc, I0, J0), cval(c, sc, I0, J0 + 1)));
    if (je) return __dmul_rn(0.5, __dadd_rn(cval(c, sc, I0, J0), cval(c, sc, I0 + 1, J0)));
    const double ll = cval(c, sc, I0, J0), lr = cval(c, sc, I0 + 1, J0);
    const double ul = cval(c, sc, I0, J0 + 1), ur = cval(c, sc, I0 + 1, J0 + 1);
    if (mode == 0)
        return __dmul_rn(0.25, __dadd_rn(__dadd_rn(__dadd_rn(ll, lr), ul), ur));
    return __dmul_rn(0.5, __dadd_rn(ll, ur));
}

__global__ void k_prolong_add(int sc, int sf, int B, const double* __restrict__ in,
                              double* __restrict__ out, const int* __restrict__ out_idx,
                              double beta, int mode) {
    const size_t nc = (size_t)sc * sc, nf = (size_t)sf * sf;
    const size_t total = nf * B;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const size_t b = k / nf, i = k % nf;
        const int x = (int)(i % sf), y = (int)(i / sf);
        const double v = prolong_at(in + b * nc, sc, x, y, mode);
        const size_t ob = out_idx ? (size_t)out_idx[b] : b;
        double* o = out + ob * nf + i;
        *o = (beta == 0.0) ? v : __dadd_rn(*o, v);
    }
}

// res = prop - c (+ g); |res|^2; Joule loss.  One CTA per column.
__global__ void __launch_bounds__(512)
k_c_residual(int n, const double* __restrict__ prop, const double* __restrict__ c,
             const int* __restrict__ c_idx, const double* __restrict__ g,
             const int* __restrict__ g_idx, double* __restrict__ res,
             double* __restrict__ sumsq, const double* __restrict__ last_f,
             const double* __restrict__ inv_dt, const double* __restrict__ w,
             double* __restrict__ loss) {
    __shared__ double red[(512 / 32) * 2];
    const int b = blockIdx.x;
    const double* pb = prop + (size_t)b * n;
    const double* cbp = c + (size_t)(c_idx ? c_idx[b] : b) * n;
    const double* gb = (g && (!g_idx || g_idx[b] >= 0))
                           ? g + (size_t)(g_idx ? g_idx[b] : b) * n : nullptr;
    const double* lf = last_f ? last_f + (size_t)b * n : nullptr;
    const double idt = last_f ? inv_dt[b] : 0.0;
    double acc[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double ci = cbp[i];
        double r = __dsub_rn(pb[i], ci);
        if (gb) r = __dadd_rn(r, gb[i]);
        if (res) res[(size_t)b * n + i] = r;
        acc[0] = fma(r, r, acc[0]);
        if (lf) {
            const double du = (ci - lf[i]) * idt;
            acc[1] = fma(w[i], du * du, acc[1]);
        }
    }
    block_sum<2>(acc, red);
    if (threadIdx.x == 0) {
        sumsq[b] = acc[0];
        if (loss) loss[b] = acc[1];
    }
}

// rhs = kept - cprop + R(res)   (coarsen) or kept - cprop + res (same grid)
__global__ void k_fas_rhs(int sf, int sc, int coarsen, int B, const double* __restrict__ kept,
                          const double* __restrict__ cprop, const double* __restrict__ res,
                          double* __restrict__ rhs, int mode) {
    const size_t nc = (size_t)sc * sc, nf = (size_t)sf * sf;
    const size_t total = nc * B;
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < total;
         k += (size_t)gridDim.x * blockDim.x) {
        const size_t b = k / nc, I = k % nc;
        double rr;
        if (coarsen) {
            const int Ix = (int)(I % sc), Iy = (int)(I / sc);
            rr = restrict_at(res + b * nf, sf, Ix, Iy, mode);
        } else {
            rr = res[k];
        }
        rhs[k] = __dadd_rn(__dsub_rn(kept[k], cprop[k]), rr);
    }
}

// Row algebra of the engine's level stores (rows of n doubles):
//   out[ro(b)] = a[ra(b)]                      (c == NULL)
//   out[ro(b)] = a[ra(b)] + sgn * c[rc(b)]     (sgn = +1 / -1)
// with r*(b) = idx ? idx[b] : start + b * step.  Covers the error payload
// v - kept (mgrit.py:483-490, :545-560), the C-store seeding / correction
// c_store (+)= e[C rows] (mgrit.py:447-450, :562-571) and strided F-point
// views.  Plain IEEE add / subtract per entry; out may alias a or c row-wise.
struct RowSel {
    const int* idx;
    int start, step;
    __device__ __forceinline__ size_t row(int b) const {
        return idx ? (size_t)idx[b] : (size_t)(start + (long long)b * step);
    }
};
__global__ void k_rows_axpby(int n, int B, const double* __restrict__ a, RowSel ra,
                             const double* c, RowSel rc, int sgn, double* out, RowSel ro) {
    for (int b = blockIdx.y; b < B; b += gridDim.y) {
        const double* ap = a + ra.row(b) * n;
        const double* cp = c ? c + rc.row(b) * n : nullptr;
        double* op = out + ro.row(b) * n;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            const double av = ap[i];
            op[i] = cp ? (sgn > 0 ? __dadd_rn(av, cp[i]) : __dsub_rn(av, cp[i])) : av;
        }
    }
}
