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
#include "tma.cuh"

#define PG_DIA_MAX 4          // max upper offsets (7-point stencil uses 3)
#define PG_DIA_NT 256
#define PG_PT_NT 512          // threads of the persistent tile kernels

struct DiaLevel {
    int n, ld;
    int U;                      // number of upper offsets
    int off[PG_DIA_MAX + 1];    // off[0] = 0
    int omax;
    const double2* __restrict__ mk;    // [(U+1)][n] (m, k)
    // uniform-1/dt fast path (k_dia_cb0, every call): for columns whose 1/dt
    // equals *cb0 the kernels read a0 = fma(cb0, M, K) per entry and
    // dinv0 = 1/(cb0 M_ii + K_ii) -- the same expressions the generic path
    // evaluates per column, so results are bit-identical
    const double* __restrict__ a0;     // [(U+1)][n]
    const double* __restrict__ dinv0;  // [ld], 0 on padding rows
    const double* __restrict__ cb0;    // [1]
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

// a0 / dinv0 / cb0 for cb0 = inv_dt[0]
__global__ void k_dia_cb0(DiaLevel L, double* __restrict__ a0, double* __restrict__ dinv0,
                          double* __restrict__ cb0, const double* __restrict__ inv_dt) {
    const double cb = inv_dt[0];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *cb0 = cb;
    if (i >= L.ld) return;
    if (i >= L.n) { dinv0[i] = 0.0; return; }
    const double2 d = L.mk[i];
    dinv0[i] = dinv_of(cb, d.x, d.y);
    for (int u = 0; u <= L.U; ++u) {
        const double2 e = L.mk[(size_t)u * L.n + i];
        a0[(size_t)u * L.n + i] = fma(cb, e.x, e.y);
    }
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


// CTA partial sum of NV values (no trailing barrier: callers pass another
// __syncthreads before `red` is rewritten).  Result valid in thread 0.
template <int NV, int NT>
__device__ __forceinline__ void cta_partial_nt(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) red[warp * NV + k] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double s = 0.0;
            for (int w = 0; w < NT / 32; ++w) s += red[w * NV + k];
            v[k] = s;
        }
    }
}

__device__ __forceinline__ double ld_cg(const double* p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Warp-0 deferred finalize: after one fence per CTA, count this CTA's tiles
// in and, for columns whose last tile this was, sum the per-tile partials
// (fixed lane-strided order + shuffle tree: deterministic).
template <typename F>
__device__ __forceinline__ void finalize_columns(const PcgWork& W, int n_tiles, int cur,
                                                 int j0, int na, int kper, int comp, F&& fin) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    for (int s = j0; s < na; s += kper) {
        const int b = W.act[cur][s];
        unsigned prev = 0;
        if (lane == 0) prev = atomicAdd(&W.cnt[b], 1u);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != (unsigned)(n_tiles - 1)) continue;
        if (lane == 0) W.cnt[b] = 0u;
        __threadfence();
        double a = 0.0, c = 0.0;
        const double* pp = W.partial + (size_t)b * n_tiles * 3;
        for (int t = lane; t < n_tiles; t += 32) {
            a += ld_cg(pp + 3 * t + comp);
            if (comp == 1) c += ld_cg(pp + 3 * t + 2);
        }
        a = warp_sum(a);
        c = warp_sum(c);
        if (lane == 0) fin(b, a, c);
    }
}

// --- persistent, TMA-pipelined iteration kernels ---------------------------------
// Grid = n_tiles * k CTAs; CTA (tile = blockIdx.x % n_tiles, j = blockIdx.x /
// n_tiles) walks the active columns j, j+k, j+2k, ...  Each work item's halo
// (and own rows) arrive by cp.async.bulk into a 2-stage smem ring, so the
// next column streams in while the current one is computed; the tile's
// matrix rows stay hot in L1 across the columns a CTA visits.

// --- v4: SpMV/direction kernel + streaming update kernel -------------------------
//
//   k_sdir (tile, C columns): TMA-stage the r and p_old halos of C columns
//          (one mbarrier), p_new = D^-1 r + beta p_old in place, q = A p_new
//          with each matrix row loaded once into registers and applied to all
//          C columns; writes p_new and q (own rows), partial p.q.   32 n B
//   k_supd (chunk, column): x += alpha p, r -= alpha q, partial r.z, r.r -
//          a pure stream (no halo, no smem).                           48 n B
//
// 80 n bytes per column-iteration (16 n more than the 2-SpMV variant) but
// each kernel is shaped for the memory system: one halo-staged SpMV, one
// perfectly coalesced stream.  Cross-CTA reductions are deferred: partials
// per (column, tile|chunk), one fence per CTA, warp-parallel finalize by the
// CTA that completes a column.

template <int C, int UU>
__global__ void __launch_bounds__(PG_DIA_NT, 3)
k_sdir(DiaLevel L, DiaWork V, PcgWork W, double* __restrict__ qv, int cur,
       const double* __restrict__ inv_dt, int SPAN) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ double red[(PG_DIA_NT / 32) * C];
    const int na = W.nact[cur];
    const int slot0 = blockIdx.y * C;
    if (slot0 >= na) return;
    const int tile = blockIdx.x;
    int r0, r1, lo, hi;
    tile_span(L, tile, r0, r1, lo, hi);
    const int span = hi - lo;
    const int nc = min(C, na - slot0);
    const double* __restrict__ p_old = V.p[cur];
    double* __restrict__ p_new = V.p[cur ^ 1];
    int bv[C];
    bool firstv[C];
    double cbv[C], betav[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        bv[c] = c < nc ? W.act[cur][slot0 + c] : 0;
        firstv[c] = W.it[bv[c]] == 0;
        cbv[c] = inv_dt[bv[c]];
        betav[c] = W.beta[bv[c]];
    }
    bool same = true;
    {
        const double c0 = *L.cb0;
#pragma unroll
        for (int c = 0; c < C; ++c) same &= (c >= nc) || cbv[c] == c0;
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
        uint32_t tx = 0;
        const uint32_t bytes = (uint32_t)span * 8u;
        for (int c = 0; c < nc; ++c) tx += firstv[c] ? bytes : 2u * bytes;
        mbar_arrive_expect_tx(&bar, tx);
        for (int c = 0; c < nc; ++c) {
            double* sr = smem + (size_t)c * 2 * SPAN;
            tma_load_1d(sr, V.r + (size_t)bv[c] * L.ld + lo, bytes, &bar);
            if (!firstv[c])
                tma_load_1d(sr + SPAN, p_old + (size_t)bv[c] * L.ld + lo, bytes, &bar);
        }
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    // p_new over the halo, in place (column-major loop so D^-1 loads are shared)
    for (int jj = 2 * threadIdx.x; jj < span; jj += 2 * PG_DIA_NT) {
        const int j = lo + jj;
        double2 d0, d1, dv;
        if (same) {
            dv = __ldg(reinterpret_cast<const double2*>(L.dinv0 + j));
        } else {
            d0 = j < L.n ? __ldg(L.mk + j) : make_double2(1.0, 1.0);
            d1 = j + 1 < L.n ? __ldg(L.mk + j + 1) : make_double2(1.0, 1.0);
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c >= nc) break;
            double* sr = smem + (size_t)c * 2 * SPAN;
            double* sp = sr + SPAN;
            const double2 rv = *reinterpret_cast<const double2*>(sr + jj);
            double2 o;
            if (same) {
                o.x = rv.x * dv.x;
                o.y = rv.y * dv.y;
            } else {
                o.x = rv.x * dinv_of(cbv[c], d0.x, d0.y);
                o.y = rv.y * dinv_of(cbv[c], d1.x, d1.y);
            }
            if (!firstv[c]) {
                const double2 pv = *reinterpret_cast<const double2*>(sp + jj);
                o.x = fma(betav[c], pv.x, o.x);
                o.y = fma(betav[c], pv.y, o.y);
            }
            *reinterpret_cast<double2*>(sp + jj) = o;
        }
    }
    __syncthreads();
    double pq[C];
#pragma unroll
    for (int c = 0; c < C; ++c) pq[c] = 0.0;
    if (same) {
#pragma unroll 2
        for (int i = r0 + threadIdx.x; i < r1; i += PG_DIA_NT) {
            // a0 entries: the row's diagonal, U upper and U mirrored lower
            const double ad = __ldg(L.a0 + i);
            double au[UU], al[UU];
#pragma unroll
            for (int u = 1; u <= UU; ++u) {
                const int o = L.off[u];
                au[u - 1] = __ldg(L.a0 + (size_t)u * L.n + i);
                al[u - 1] = (i - o >= 0) ? __ldg(L.a0 + (size_t)u * L.n + i - o) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (c >= nc) break;
                const double* spw = smem + (size_t)c * 2 * SPAN + SPAN - lo;
                double q = ad * spw[i];             // dia_row with fma(cb, m, k) precomputed
#pragma unroll
                for (int u = 1; u <= UU; ++u) {
                    const int o = L.off[u];
                    if (i + o < L.n) q = fma(au[u - 1], spw[i + o], q);
                    if (i - o >= 0) q = fma(al[u - 1], spw[i - o], q);
                }
                const double pi = spw[i];
                pq[c] = fma(pi, q, pq[c]);
                const size_t k = (size_t)bv[c] * L.ld + i;
                p_new[k] = pi;
                qv[k] = q;
            }
        }
    } else
    for (int i = r0 + threadIdx.x; i < r1; i += PG_DIA_NT) {
        double2 dg, up[UU], lw[UU];
        dia_load_row<UU>(L, i, dg, up, lw);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (c >= nc) break;
            const double* spw = smem + (size_t)c * 2 * SPAN + SPAN - lo;
            const double q = dia_row<UU>(L, i, cbv[c], spw, &dg, up, lw);
            const double pi = spw[i];
            pq[c] = fma(pi, q, pq[c]);
            const size_t k = (size_t)bv[c] * L.ld + i;
            p_new[k] = pi;
            qv[k] = q;
        }
    }
    cta_partial_nt<C, PG_DIA_NT>(pq, red);
    if (threadIdx.x == 0)
        for (int c = 0; c < nc; ++c) W.partial[((size_t)bv[c] * L.n_tiles + tile) * 3] = pq[c];
    // deferred finalize of the columns of this CTA
    __syncthreads();
    if (threadIdx.x == 0) __threadfence();
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        for (int c = 0; c < nc; ++c) {
            const int b = bv[c];
            unsigned prev = 0;
            if (lane == 0) prev = atomicAdd(&W.cnt[b], 1u);
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev != (unsigned)(L.n_tiles - 1)) continue;
            if (lane == 0) W.cnt[b] = 0u;
            __threadfence();
            double a = 0.0;
            const double* pp = W.partial + (size_t)b * L.n_tiles * 3;
            for (int t = lane; t < L.n_tiles; t += 32) a += ld_cg(pp + 3 * t);
            a = warp_sum(a);
            if (lane == 0) {
                if (a > 0.0) {
                    W.alpha[b] = W.rho[b] / a;
                } else {
                    W.alpha[b] = 0.0;
                    W.flag[b] = COL_BREAKDOWN;
                }
            }
        }
    }
}

// streaming update: grid (n_chunks, active slots)
#define PG_UPD_NT 256
#define PG_UPD_V 4          // double2 per thread per array -> 2048 rows / CTA
template <int UU>
__global__ void __launch_bounds__(PG_UPD_NT, 3)
k_supd(DiaLevel L, DiaWork V, PcgWork W, const double* __restrict__ qv, int cur,
       const double* __restrict__ inv_dt, int max_iters, int n_chunks) {
    __shared__ double red[(PG_UPD_NT / 32) * 2];
    __shared__ int s_flag;
    __shared__ int s_scan[PG_UPD_NT + 1];
    const int na = W.nact[cur];
    const int slot = blockIdx.y;
    const int chunk = blockIdx.x;
    if (slot < na) {
        const int b = W.act[cur][slot];
        const double cb = inv_dt[b];
        const bool same = cb == *L.cb0;
        const double al = W.alpha[b];
        const size_t base = (size_t)b * L.ld;
        const double* __restrict__ p = V.p[cur ^ 1] + base;
        const double* __restrict__ q = qv + base;
        double* __restrict__ x = V.x + base;
        double* __restrict__ r = V.r + base;
        const int i0 = chunk * (PG_UPD_NT * PG_UPD_V * 2);
        double2 xv[PG_UPD_V], rv[PG_UPD_V], pv[PG_UPD_V], qq[PG_UPD_V];
#pragma unroll
        for (int k = 0; k < PG_UPD_V; ++k) {
            const int i = i0 + 2 * (threadIdx.x + k * PG_UPD_NT);
            if (i < L.n) {
                xv[k] = ld2(x + i);
                rv[k] = ld2(r + i);
                pv[k] = ld2(p + i);
                qq[k] = ld2(q + i);
            }
        }
        double acc[2] = {0.0, 0.0};
#pragma unroll
        for (int k = 0; k < PG_UPD_V; ++k) {
            const int i = i0 + 2 * (threadIdx.x + k * PG_UPD_NT);
            if (i < L.n) {
                double2 dv;
                if (same) {
                    dv = __ldg(reinterpret_cast<const double2*>(L.dinv0 + i));
                } else {
                    const double2 d0 = __ldg(L.mk + i);
                    const double2 d1 = (i + 1 < L.n) ? __ldg(L.mk + i + 1) : make_double2(1.0, 1.0);
                    dv.x = dinv_of(cb, d0.x, d0.y);
                    dv.y = dinv_of(cb, d1.x, d1.y);
                }
                double2 xo, ro;
                xo.x = fma(al, pv[k].x, xv[k].x);
                xo.y = fma(al, pv[k].y, xv[k].y);
                ro.x = fma(-al, qq[k].x, rv[k].x);
                ro.y = fma(-al, qq[k].y, rv[k].y);   // padding rows: q = r = 0
                *reinterpret_cast<double2*>(x + i) = xo;
                *reinterpret_cast<double2*>(r + i) = ro;
                acc[0] = fma(ro.x * ro.x, dv.x, acc[0]);
                acc[1] = fma(ro.x, ro.x, acc[1]);
                if (i + 1 < L.n) {
                    acc[0] = fma(ro.y * ro.y, dv.y, acc[0]);
                    acc[1] = fma(ro.y, ro.y, acc[1]);
                }
            }
        }
        cta_partial_nt<2, PG_UPD_NT>(acc, red);
        if (threadIdx.x == 0) {
            double* pp = W.partial + ((size_t)b * n_chunks + chunk) * 3;
            pp[1] = acc[0]; pp[2] = acc[1];
        }
        __syncthreads();
        if (threadIdx.x == 0) __threadfence();
        __syncthreads();
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;
            unsigned prev = 0;
            if (lane == 0) prev = atomicAdd(&W.cnt[b], 1u);
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev == (unsigned)(n_chunks - 1)) {
                if (lane == 0) W.cnt[b] = 0u;
                __threadfence();
                double rz = 0.0, rr = 0.0;
                const double* pp = W.partial + (size_t)b * n_chunks * 3;
                for (int t = lane; t < n_chunks; t += 32) {
                    rz += ld_cg(pp + 3 * t + 1);
                    rr += ld_cg(pp + 3 * t + 2);
                }
                rz = warp_sum(rz);
                rr = warp_sum(rr);
                if (lane == 0) {
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
