// Batched Jacobi-PCG for (c_b M + K) x_b = c_b M u_b + f_b, one column per
// MGRIT C-interval.  Layout: states [B][n] fp64, CSR of the union pattern of
// M and K shared by all columns (L2-resident), c_b = 1/dt_b per column.
//
// Streamed path (n > PG_RES_MAX): two kernels per PCG iteration over
// (row tile, column group) CTAs.  Each CTA stages the halo range
// [tile_lo, tile_hi) of the direction vector of its C columns in shared
// memory, so every vector element crosses HBM once per kernel:
//
//   k_dir: p_new = D^-1 r + beta p_old (computed once per halo element into
//          smem; own rows written back), q = A p_new, partial p.q
//          -> last CTA of the column: alpha = rho / p.q
//   k_upd: q = A p_new recomputed from the staged halo (cheaper than storing
//          q: 16 n bytes saved for one extra CSR pass from L2),
//          x += alpha p, r -= alpha q, partial r.z and r.r
//          -> last CTA of the column: beta, rho, convergence flag;
//          -> last CTA of the grid compacts the active-column list.
//
// HBM bytes per active column per iteration: k_dir reads r, p_old and writes
// p_new (24 n), k_upd reads p_new, x, r and writes x, r (40 n): 64 n.
// Reductions are deterministic: per-(column, tile) partials are summed in
// tile order by the last CTA to finish (threadfence-reduction pattern).
#pragma once
#include "common.cuh"

struct PcgLevel {
    int n;
    const int* __restrict__ row_ptr;
    const int* __restrict__ col_idx;
    const double* __restrict__ m_val;
    const double* __restrict__ k_val;
    const double* __restrict__ dM;
    const double* __restrict__ dK;
    int n_src;
    const double* __restrict__ shapes;
    int R;                 // rows per tile
    int n_tiles;
    const int* __restrict__ tile_lo;
    const int* __restrict__ tile_hi;
};

struct PcgWork {
    double* r;
    double* p[2];          // ping-pong direction vectors
    double* rho;
    double* alpha;
    double* beta;
    double* tol2;
    double* bnorm2;
    int* it;
    int* flag;
    double* partial;       // [B][n_tiles][3]
    unsigned* cnt;         // [B] per-column CTA counters
    unsigned* gcnt;        // [1] grid counter
    int* act[2];           // active column lists
    int* nact;             // [2]
    unsigned long long* iters;  // [0] cumulative, [1] this call: column iterations
    int* ictr;             // [0] max iterations this call, [1] failed total, [2] failed call
};

__device__ __forceinline__ double dinv_of(double cb, double dm, double dk) {
    return 1.0 / (cb * dm + dk);
}

// Last-CTA election for column b: returns true in all threads of the CTA
// that completed the column's tile set last.  Partials must be written by
// thread 0 before the call.
__device__ __forceinline__ bool column_last(unsigned* cnt, int b, int n_tiles,
                                            int* s_flag) {
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned prev = atomicAdd(&cnt[b], 1u);
        *s_flag = (prev == (unsigned)(n_tiles - 1));
        if (*s_flag) cnt[b] = 0u;   // reset for the next launch
    }
    __syncthreads();
    bool last = *s_flag;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// Grid-level last-CTA election.
__device__ __forceinline__ bool grid_last(unsigned* gcnt, int* s_flag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned total = gridDim.x * gridDim.y;
        unsigned prev = atomicAdd(gcnt, 1u);
        *s_flag = (prev == total - 1);
        if (*s_flag) *gcnt = 0u;
    }
    __syncthreads();
    bool last = *s_flag;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// Order-preserving compaction of the active columns, run by one CTA.
__device__ void compact_active(const int* src, int n_src, const int* flag,
                               int* dst, int* n_dst, int* s_scan) {
    // s_scan: blockDim.x + 1 ints
    int base = 0;
    for (int off = 0; off < n_src; off += blockDim.x) {
        int i = off + threadIdx.x;
        int keep = 0, b = -1;
        if (i < n_src) {
            b = src[i];
            keep = (((volatile const int*)flag)[b] == COL_ACTIVE);
        }
        s_scan[threadIdx.x] = keep;
        __syncthreads();
        // inclusive Hillis-Steele scan
        for (int d = 1; d < (int)blockDim.x; d <<= 1) {
            int v = (threadIdx.x >= (unsigned)d) ? s_scan[threadIdx.x - d] : 0;
            __syncthreads();
            s_scan[threadIdx.x] += v;
            __syncthreads();
        }
        if (keep) dst[base + s_scan[threadIdx.x] - 1] = b;
        int tot = s_scan[blockDim.x - 1];
        __syncthreads();
        base += tot;
    }
    if (threadIdx.x == 0) *n_dst = base;
}

// --- setup: r0 = b - A x0, x0 = guess, |b|^2, rho0 = r.z ----------------------
template <int C, bool GUESS>
__global__ void __launch_bounds__(PG_NT)
k_pcg_setup(PcgLevel L, PcgWork W, int B, const double* __restrict__ u_prev,
            const double* __restrict__ guess, const double* __restrict__ inv_dt,
            const double* __restrict__ src, double* __restrict__ x, double rtol2,
            int max_iters) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_NT / 32) * 3 * C];
    __shared__ int s_flag;
    const int n = L.n, tile = blockIdx.x;
    const int lo = L.tile_lo[tile], hi = L.tile_hi[tile], span = hi - lo;
    const int r0 = tile * L.R, r1 = min(n, r0 + L.R);
    double* s_u = smem;                  // [C][span]
    double* s_g = smem + C * span;       // [C][span] if GUESS

    int cols[C];
    double cb[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        int b = blockIdx.y * C + c;
        cols[c] = (b < B) ? b : -1;
        cb[c] = (b < B) ? inv_dt[b] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (cols[c] < 0) continue;
        const double* u = u_prev + (size_t)cols[c] * n;
        for (int j = lo + threadIdx.x; j < hi; j += PG_NT) s_u[c * span + j - lo] = u[j];
        if (GUESS) {
            const double* g = guess + (size_t)cols[c] * n;
            for (int j = lo + threadIdx.x; j < hi; j += PG_NT) s_g[c * span + j - lo] = g[j];
        }
    }
    __syncthreads();

    double acc[C][3];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = acc[c][2] = 0.0;

    for (int i = r0 + threadIdx.x; i < r1; i += PG_NT) {
        double mu[C], ku[C], mg[C], kg[C];
#pragma unroll
        for (int c = 0; c < C; ++c) mu[c] = ku[c] = mg[c] = kg[c] = 0.0;
        const int e0 = L.row_ptr[i], e1 = L.row_ptr[i + 1];
        for (int e = e0; e < e1; ++e) {
            const int j = ldg(L.col_idx + e) - lo;
            const double mv = ldg(L.m_val + e), kv = ldg(L.k_val + e);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const double uj = s_u[c * span + j];
                mu[c] = fma(mv, uj, mu[c]);
                ku[c] = fma(kv, uj, ku[c]);
                if (GUESS) {
                    const double gj = s_g[c * span + j];
                    mg[c] = fma(mv, gj, mg[c]);
                    kg[c] = fma(kv, gj, kg[c]);
                }
            }
        }
        const double dm = ldg(L.dM + i), dk = ldg(L.dK + i);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (cols[c] < 0) continue;
            const int b = cols[c];
            double f = 0.0;
            for (int s = 0; s < L.n_src; ++s)
                f = fma(src[b * L.n_src + s], ldg(L.shapes + (size_t)s * n + i), f);
            const double bi = fma(cb[c], mu[c], f);
            double ri, xi;
            if (GUESS) {
                ri = bi - fma(cb[c], mg[c], kg[c]);
                xi = s_g[c * span + i - lo];
            } else {
                ri = f - ku[c];          // b - A u = f - K u when x0 = u_prev
                xi = s_u[c * span + i - lo];
            }
            x[(size_t)b * n + i] = xi;
            W.r[(size_t)b * n + i] = ri;
            acc[c][0] = fma(bi, bi, acc[c][0]);
            acc[c][1] = fma(ri * ri, dinv_of(cb[c], dm, dk), acc[c][1]);
            acc[c][2] = fma(ri, ri, acc[c][2]);
        }
    }
    // per-column reductions
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (cols[c] < 0) continue;          // uniform across the CTA
        double v[3] = {acc[c][0], acc[c][1], acc[c][2]};
        block_sum<3>(v, red);
        const int b = cols[c];
        if (threadIdx.x == 0) {
            double* pp = W.partial + ((size_t)b * L.n_tiles + tile) * 3;
            pp[0] = v[0]; pp[1] = v[1]; pp[2] = v[2];
        }
        if (column_last(W.cnt, b, L.n_tiles, &s_flag) && threadIdx.x == 0) {
            double bb = 0.0, rz = 0.0, rr = 0.0;
            const double* pp = W.partial + (size_t)b * L.n_tiles * 3;
            for (int t = 0; t < L.n_tiles; ++t) {
                bb += pp[3 * t]; rz += pp[3 * t + 1]; rr += pp[3 * t + 2];
            }
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
        // all columns of this call: act[0] <- columns still active
        __shared__ int s_scan[PG_NT + 1];
        int base = 0;
        for (int off = 0; off < B; off += PG_NT) {
            int b = off + threadIdx.x;
            int keep = (b < B) && (((volatile int*)W.flag)[b] == COL_ACTIVE);
            s_scan[threadIdx.x] = keep;
            __syncthreads();
            for (int d = 1; d < PG_NT; d <<= 1) {
                int v = (threadIdx.x >= (unsigned)d) ? s_scan[threadIdx.x - d] : 0;
                __syncthreads();
                s_scan[threadIdx.x] += v;
                __syncthreads();
            }
            if (keep) W.act[0][base + s_scan[threadIdx.x] - 1] = b;
            int tot = s_scan[PG_NT - 1];
            __syncthreads();
            base += tot;
        }
        if (threadIdx.x == 0) W.nact[0] = base;
    }
}

// --- direction update + SpMV + p.q ------------------------------------------------
template <int C>
__global__ void __launch_bounds__(PG_NT)
k_pcg_dir(PcgLevel L, PcgWork W, int cur, const double* __restrict__ inv_dt) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_NT / 32) * C];
    __shared__ int s_flag;
    const int na = W.nact[cur];
    const int slot0 = blockIdx.y * C;
    if (slot0 >= na) return;
    const int n = L.n, tile = blockIdx.x;
    const int lo = L.tile_lo[tile], hi = L.tile_hi[tile], span = hi - lo;
    const int r0 = tile * L.R, r1 = min(n, r0 + L.R);
    const double* __restrict__ p_old = W.p[cur];
    double* __restrict__ p_new = W.p[cur ^ 1];

    int cols[C];
    double cb[C], beta[C];
    bool first[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const int s = slot0 + c;
        cols[c] = (s < na) ? W.act[cur][s] : -1;
        const int b = cols[c] < 0 ? 0 : cols[c];
        cb[c] = inv_dt[b];
        beta[c] = W.beta[b];
        first[c] = (W.it[b] == 0);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (cols[c] < 0) continue;
        const size_t off = (size_t)cols[c] * n;
        const double* rr = W.r + off;
        const double* po = p_old + off;
        for (int j = lo + threadIdx.x; j < hi; j += PG_NT) {
            double z = rr[j] * dinv_of(cb[c], ldg(L.dM + j), ldg(L.dK + j));
            smem[c * span + j - lo] = first[c] ? z : fma(beta[c], po[j], z);
        }
    }
    __syncthreads();

    double pq[C];
#pragma unroll
    for (int c = 0; c < C; ++c) pq[c] = 0.0;
    for (int i = r0 + threadIdx.x; i < r1; i += PG_NT) {
        double mq[C], kq[C];
#pragma unroll
        for (int c = 0; c < C; ++c) mq[c] = kq[c] = 0.0;
        const int e0 = L.row_ptr[i], e1 = L.row_ptr[i + 1];
        for (int e = e0; e < e1; ++e) {
            const int j = ldg(L.col_idx + e) - lo;
            const double mv = ldg(L.m_val + e), kv = ldg(L.k_val + e);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const double pj = smem[c * span + j];
                mq[c] = fma(mv, pj, mq[c]);
                kq[c] = fma(kv, pj, kq[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (cols[c] < 0) continue;
            const double pi = smem[c * span + i - lo];
            p_new[(size_t)cols[c] * n + i] = pi;
            pq[c] = fma(pi, fma(cb[c], mq[c], kq[c]), pq[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (cols[c] < 0) continue;
        double v[1] = {pq[c]};
        block_sum<1>(v, red);
        const int b = cols[c];
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

// --- x, r update + r.z, r.r + convergence ---------------------------------------
template <int C>
__global__ void __launch_bounds__(PG_NT)
k_pcg_upd(PcgLevel L, PcgWork W, int cur, const double* __restrict__ inv_dt,
          double* __restrict__ x, int max_iters) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_NT / 32) * 2 * C];
    __shared__ int s_flag;
    __shared__ int s_scan[PG_NT + 1];
    const int na = W.nact[cur];
    const int slot0 = blockIdx.y * C;
    const int n = L.n, tile = blockIdx.x;
    if (slot0 < na) {
        const int lo = L.tile_lo[tile], hi = L.tile_hi[tile], span = hi - lo;
        const int r0 = tile * L.R, r1 = min(n, r0 + L.R);
        const double* __restrict__ p = W.p[cur ^ 1];
        int cols[C];
        double cb[C], alpha[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int s = slot0 + c;
            cols[c] = (s < na) ? W.act[cur][s] : -1;
            const int b = cols[c] < 0 ? 0 : cols[c];
            cb[c] = inv_dt[b];
            alpha[c] = W.alpha[b];
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (cols[c] < 0) continue;
            const double* pc = p + (size_t)cols[c] * n;
            for (int j = lo + threadIdx.x; j < hi; j += PG_NT) smem[c * span + j - lo] = pc[j];
        }
        __syncthreads();
        double acc[C][2];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
        for (int i = r0 + threadIdx.x; i < r1; i += PG_NT) {
            double mq[C], kq[C];
#pragma unroll
            for (int c = 0; c < C; ++c) mq[c] = kq[c] = 0.0;
            const int e0 = L.row_ptr[i], e1 = L.row_ptr[i + 1];
            for (int e = e0; e < e1; ++e) {
                const int j = ldg(L.col_idx + e) - lo;
                const double mv = ldg(L.m_val + e), kv = ldg(L.k_val + e);
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    const double pj = smem[c * span + j];
                    mq[c] = fma(mv, pj, mq[c]);
                    kq[c] = fma(kv, pj, kq[c]);
                }
            }
            const double dm = ldg(L.dM + i), dk = ldg(L.dK + i);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if (cols[c] < 0) continue;
                const size_t k = (size_t)cols[c] * n + i;
                const double q = fma(cb[c], mq[c], kq[c]);
                const double pi = smem[c * span + i - lo];
                x[k] = fma(alpha[c], pi, x[k]);
                const double ri = fma(-alpha[c], q, W.r[k]);
                W.r[k] = ri;
                acc[c][0] = fma(ri * ri, dinv_of(cb[c], dm, dk), acc[c][0]);
                acc[c][1] = fma(ri, ri, acc[c][1]);
            }
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (cols[c] < 0) continue;
            double v[2] = {acc[c][0], acc[c][1]};
            block_sum<2>(v, red);
            const int b = cols[c];
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
    if (grid_last(W.gcnt, &s_flag)) compact_active(W.act[cur], na, W.flag, W.act[cur ^ 1],
                                                   &W.nact[cur ^ 1], s_scan);
}

// --- CTA-resident PCG for small grids (n <= PG_RES_MAX) -----------------------
// One CTA per column; x, r, p, q and D^-1 live in shared memory for the whole
// solve, so a batched Phi is a single launch with no host round trip.  The
// CSR (<= 5000 rows) streams from L1/L2.
__global__ void __launch_bounds__(PG_RES_NT)
k_pcg_resident(PcgLevel L, int B, const double* __restrict__ u_prev,
               const double* __restrict__ guess, const double* __restrict__ inv_dt,
               const double* __restrict__ src, double* __restrict__ u_out,
               const double* __restrict__ g, const int* __restrict__ g_idx,
               double rtol2, int max_iters, unsigned long long* iters, int* ictr) {
    extern __shared__ double smem[];
    __shared__ double red[(PG_RES_NT / 32) * 3];
    __shared__ double s_bc[4];
    const int n = L.n, b = blockIdx.x;
    double* s_x = smem;
    double* s_r = smem + n;
    double* s_p = smem + 2 * n;
    double* s_q = smem + 3 * n;
    double* s_d = smem + 4 * n;
    const double cb = inv_dt[b];
    const double* u = u_prev + (size_t)b * n;
    const double* gs = guess ? guess + (size_t)b * n : u;

    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        s_p[i] = u[i];
        s_x[i] = gs[i];
        s_d[i] = dinv_of(cb, ldg(L.dM + i), ldg(L.dK + i));
    }
    __syncthreads();
    double acc[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double mu = 0.0, mx = 0.0, kx = 0.0;
        for (int e = L.row_ptr[i]; e < L.row_ptr[i + 1]; ++e) {
            const int j = ldg(L.col_idx + e);
            const double mv = ldg(L.m_val + e), kv = ldg(L.k_val + e);
            mu = fma(mv, s_p[j], mu);
            mx = fma(mv, s_x[j], mx);
            kx = fma(kv, s_x[j], kx);
        }
        double f = 0.0;
        for (int s = 0; s < L.n_src; ++s)
            f = fma(src[b * L.n_src + s], ldg(L.shapes + (size_t)s * n + i), f);
        const double bi = fma(cb, mu, f);
        const double ri = guess ? bi - fma(cb, mx, kx) : f - kx;
        s_r[i] = ri;
        acc[0] = fma(bi, bi, acc[0]);
        acc[1] = fma(ri * ri, s_d[i], acc[1]);
        acc[2] = fma(ri, ri, acc[2]);
    }
    block_sum<3>(acc, red);
    if (threadIdx.x == 0) { s_bc[0] = acc[0]; s_bc[1] = acc[1]; s_bc[2] = acc[2]; }
    __syncthreads();
    const double tol2 = rtol2 * s_bc[0];
    double rho = s_bc[1], rr = s_bc[2];
    int it = 0;
    bool conv = (rr <= tol2 || rr == 0.0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_p[i] = s_r[i] * s_d[i];
    __syncthreads();
    while (!conv && it < max_iters) {
        double pq[1] = {0.0};
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double mq = 0.0, kq = 0.0;
            for (int e = L.row_ptr[i]; e < L.row_ptr[i + 1]; ++e) {
                const int j = ldg(L.col_idx + e);
                mq = fma(ldg(L.m_val + e), s_p[j], mq);
                kq = fma(ldg(L.k_val + e), s_p[j], kq);
            }
            const double q = fma(cb, mq, kq);
            s_q[i] = q;
            pq[0] = fma(s_p[i], q, pq[0]);
        }
        block_sum<1>(pq, red);
        if (threadIdx.x == 0) s_bc[3] = pq[0];
        __syncthreads();
        const double pqs = s_bc[3];
        if (!(pqs > 0.0)) break;
        const double alpha = rho / pqs;
        double a2[2] = {0.0, 0.0};
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            s_x[i] = fma(alpha, s_p[i], s_x[i]);
            const double ri = fma(-alpha, s_q[i], s_r[i]);
            s_r[i] = ri;
            a2[0] = fma(ri * ri, s_d[i], a2[0]);
            a2[1] = fma(ri, ri, a2[1]);
        }
        block_sum<2>(a2, red);
        if (threadIdx.x == 0) { s_bc[1] = a2[0]; s_bc[2] = a2[1]; }
        __syncthreads();
        const double rz = s_bc[1];
        rr = s_bc[2];
        const double beta = rz / rho;
        rho = rz;
        ++it;
        conv = (rr <= tol2 || rr == 0.0);
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            s_p[i] = fma(beta, s_p[i], s_r[i] * s_d[i]);
        __syncthreads();
    }
    const double* gg = (g && g_idx && g_idx[b] >= 0) ? g + (size_t)g_idx[b] * n : nullptr;
    double* o = u_out + (size_t)b * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) o[i] = gg ? s_x[i] + gg[i] : s_x[i];
    if (threadIdx.x == 0) {
        atomicAdd(iters, (unsigned long long)it);
        atomicAdd(iters + 1, (unsigned long long)it);
        atomicMax(ictr, it);
        if (!conv) { atomicAdd(ictr + 1, 1); atomicAdd(ictr + 2, 1); }
    }
}

// u_out[b] += g[g_idx[b]]
__global__ void k_add_g(int n, int B, double* __restrict__ u, const double* __restrict__ g,
                        const int* __restrict__ g_idx) {
    const int b = blockIdx.y;
    const int gi = g_idx[b];
    if (gi < 0) return;
    const double* gs = g + (size_t)gi * n;
    double* us = u + (size_t)b * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        us[i] += gs[i];
}
