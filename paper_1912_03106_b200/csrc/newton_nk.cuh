// Batched Newton-Krylov for the nonlinear model (inner = banded Cholesky).
//
// The reference's damped Newton (problems.py:201-244) over masked column
// sets (one column per C-interval): every step is a batched kernel over the
// active columns.  The Newton-level decisions (converged? halve?) are the
// reference's per-column rules taken on the host from per-column norms (a few
// reads per Phi call); the inner CG keeps its per-column convergence flags on
// the device (k_nk_cg_a sets flag bit 0 when |r| <= rtol |F|, every CG kernel
// skips flagged columns), so the host launches bursts of iterations and only
// reads the flags between bursts to re-pack the active list.
// The Newton system J(u) d = -F is solved by CG
// preconditioned with the banded-Cholesky factor of the linearised operator
// c M + K(nu_iron(0)) -- one per distinct dt, shared with the band-solve
// machinery (band.cuh) -- so the inner solve takes a handful of iterations
// where Jacobi-PCG needs hundreds (the iron contrast is ~1/1300).
#pragma once
#include "common.cuh"
#include "newton.cuh"

#define NK_NT 512

struct NkLevel {
    int n, n_elem, n_src;
    const int* __restrict__ row_ptr;
    const int* __restrict__ col_idx;
    const double* __restrict__ m_val;
    const double* __restrict__ k_val;      // non-iron stiffness
    const double* __restrict__ shapes;
    const int* __restrict__ edof;
    const double* __restrict__ egeo;
    const int* __restrict__ ne_ptr;
    const int* __restrict__ ne;
    double nu0, k1, k2, k3;
};

__device__ __forceinline__ double nk_sum(double v, double* red) {
    double a[1] = {v};
    block_sum<1>(a, red);
    if (threadIdx.x == 0) red[2 * (NK_NT / 32)] = a[0];
    __syncthreads();
    const double s = red[2 * (NK_NT / 32)];
    __syncthreads();
    return s;
}

// rhs = c M u_prev + f ; u = guess ; rhs2 = |rhs|^2   (CTA per column)
__global__ void __launch_bounds__(NK_NT)
k_nk_init(NkLevel L, const double* __restrict__ u_prev, const double* __restrict__ guess,
          const double* __restrict__ inv_dt, const double* __restrict__ src,
          double* __restrict__ u, double* __restrict__ rhs, double* __restrict__ rhs2) {
    __shared__ double red[2 * (NK_NT / 32) + 2];
    const int b = blockIdx.x;
    const size_t off = (size_t)b * L.n;
    const double c = inv_dt[b];
    const double* up = u_prev + off;
    const double* g0 = guess ? guess + off : up;
    double acc = 0.0;
    for (int i = threadIdx.x; i < L.n; i += blockDim.x) {
        double mv = 0.0;
        for (int k = L.row_ptr[i]; k < L.row_ptr[i + 1]; ++k)
            mv = fma(L.m_val[k], up[L.col_idx[k]], mv);
        double f = 0.0;
        for (int s = 0; s < L.n_src; ++s)
            f = fma(src[b * L.n_src + s], L.shapes[(size_t)s * L.n + i], f);
        const double r = fma(c, mv, f);
        rhs[off + i] = r;
        u[off + i] = g0[i];
        acc = fma(r, r, acc);
    }
    const double s = nk_sum(acc, red);
    if (threadIdx.x == 0) rhs2[b] = s;
}

// E[b][e] = (nu, 2 nu', gx, gy) of V[b]      grid (element chunks, active)
__global__ void k_nk_elements(NkLevel L, const int* __restrict__ act,
                              const double* __restrict__ V, double* __restrict__ E) {
    const int b = act[blockIdx.y];
    const double* v = V + (size_t)b * L.n;
    double* Eb = E + (size_t)b * L.n_elem * 4;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < L.n_elem;
         e += gridDim.x * blockDim.x) {
        const double* gq = L.egeo + (size_t)e * 7;
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int dof = L.edof[e * 3 + a];
            const double va = dof >= 0 ? v[dof] : 0.0;
            gx = fma(gq[a], va, gx);
            gy = fma(gq[3 + a], va, gy);
        }
        const double ex = exp(L.k2 * (gx * gx + gy * gy));
        double* o = Eb + (size_t)e * 4;
        o[0] = L.nu0 * (L.k1 * ex + L.k3);
        o[1] = 2.0 * L.nu0 * L.k1 * L.k2 * ex;
        o[2] = gx;
        o[3] = gy;
    }
}

// F = c M v + K v + N(v) - rhs ; f2 = |F|^2      (CTA per active column)
__global__ void __launch_bounds__(NK_NT)
k_nk_residual(NkLevel L, const int* __restrict__ act, const double* __restrict__ inv_dt,
              const double* __restrict__ V, const double* __restrict__ E,
              const double* __restrict__ rhs, double* __restrict__ F, double* __restrict__ f2) {
    __shared__ double red[2 * (NK_NT / 32) + 2];
    const int b = act[blockIdx.x];
    const size_t off = (size_t)b * L.n;
    const double c = inv_dt[b];
    const double* v = V + off;
    const double* Eb = E + (size_t)b * L.n_elem * 4;
    double acc = 0.0;
    for (int i = threadIdx.x; i < L.n; i += blockDim.x) {
        double mv = 0.0, kv = 0.0;
        for (int k = L.row_ptr[i]; k < L.row_ptr[i + 1]; ++k) {
            const double x = v[L.col_idx[k]];
            mv = fma(L.m_val[k], x, mv);
            kv = fma(L.k_val[k], x, kv);
        }
        double nl = 0.0;
        for (int k = L.ne_ptr[i]; k < L.ne_ptr[i + 1]; ++k) {
            const int ea = L.ne[k], e = ea >> 2, a = ea & 3;
            const double* gq = L.egeo + (size_t)e * 7;
            const double* q = Eb + (size_t)e * 4;
            nl = fma(gq[6] * q[0], fma(q[2], gq[a], q[3] * gq[3 + a]), nl);
        }
        const double f = fma(c, mv, kv) + nl - rhs[off + i];
        F[off + i] = f;
        acc = fma(f, f, acc);
    }
    const double s = nk_sum(acc, red);
    if (threadIdx.x == 0) f2[b] = s;
}

// Q = J(u) P over active columns                 grid (row chunks, active)
__global__ void k_nk_japply(NkLevel L, const int* __restrict__ act,
                            const int* __restrict__ flag,
                            const double* __restrict__ inv_dt, const double* __restrict__ P,
                            const double* __restrict__ E, double* __restrict__ Q) {
    const int b = act[blockIdx.y];
    if (flag[b] & 1) return;                       // CG of this column has converged
    const size_t off = (size_t)b * L.n;
    const double c = inv_dt[b];
    const double* p = P + off;
    const double* Eb = E + (size_t)b * L.n_elem * 4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += gridDim.x * blockDim.x) {
        double mv = 0.0, kv = 0.0;
        for (int k = L.row_ptr[i]; k < L.row_ptr[i + 1]; ++k) {
            const double x = p[L.col_idx[k]];
            mv = fma(L.m_val[k], x, mv);
            kv = fma(L.k_val[k], x, kv);
        }
        double nl = 0.0;
        for (int k = L.ne_ptr[i]; k < L.ne_ptr[i + 1]; ++k) {
            const int ea = L.ne[k], e = ea >> 2, a = ea & 3;
            const double* gq = L.egeo + (size_t)e * 7;
            const double* q = Eb + (size_t)e * 4;
            double tx = 0.0, ty = 0.0;
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
                const int dof = L.edof[e * 3 + bb];
                const double pb = dof >= 0 ? p[dof] : 0.0;
                tx = fma(gq[bb], pb, tx);
                ty = fma(gq[3 + bb], pb, ty);
            }
            const double ga = fma(q[2], gq[a], q[3] * gq[3 + a]);
            const double ta = fma(tx, gq[a], ty * gq[3 + a]);
            const double gt = fma(q[2], tx, q[3] * ty);
            nl = fma(gq[6], fma(q[0], ta, q[1] * ga * gt), nl);
        }
        Q[off + i] = fma(c, mv, kv) + nl;
    }
}

// Jacobian of column b's state as CSR values on the level's pattern (thread
// per row): kj = K_lin + sum over the row's iron elements of
// area [nu G^T G + 2 nu' (G^T g)(G^T g)^T] -- the matrix k_nk_japply applies
// matrix-free, minus the c M term (k_band_build adds it).  Its banded
// Cholesky factor is a frozen-Jacobian preconditioner for later Newton
// systems with a similar saturation pattern.
__global__ void k_nk_jac_assemble(NkLevel L, int b, const double* __restrict__ E,
                                  double* __restrict__ kj) {
    const double* Eb = E + (size_t)b * L.n_elem * 4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n; i += gridDim.x * blockDim.x) {
        const int r0 = L.row_ptr[i], r1 = L.row_ptr[i + 1];
        for (int k = r0; k < r1; ++k) kj[k] = L.k_val[k];
        for (int k = L.ne_ptr[i]; k < L.ne_ptr[i + 1]; ++k) {
            const int ea = L.ne[k], e = ea >> 2, a = ea & 3;
            const double* gq = L.egeo + (size_t)e * 7;
            const double* q = Eb + (size_t)e * 4;
            const double ga = fma(q[2], gq[a], q[3] * gq[3 + a]);
#pragma unroll
            for (int bb = 0; bb < 3; ++bb) {
                const int dof = L.edof[e * 3 + bb];
                if (dof < 0) continue;
                const double gg = fma(gq[a], gq[bb], gq[3 + a] * gq[3 + bb]);
                const double gb = fma(q[2], gq[bb], q[3] * gq[3 + bb]);
                const double v = gq[6] * fma(q[0], gg, q[1] * ga * gb);
                for (int m = r0; m < r1; ++m)
                    if (L.col_idx[m] == dof) { kj[m] += v; break; }
            }
        }
    }
}

// r = -F, d = 0                                   grid (row chunks, active)
__global__ void k_nk_start(int n, const int* __restrict__ act, int* __restrict__ flag,
                           const double* __restrict__ F,
                           double* __restrict__ R, double* __restrict__ D) {
    const size_t off = (size_t)act[blockIdx.y] * n;
    if (blockIdx.x == 0 && threadIdx.x == 0) flag[act[blockIdx.y]] = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        R[off + i] = -F[off + i];
        D[off + i] = 0.0;
    }
}

// alpha = rho / p.q ; d += alpha p ; r -= alpha q ; rr = |r|^2   (CTA per column)
__global__ void __launch_bounds__(NK_NT)
k_nk_cg_a(int n, const int* __restrict__ act, int* __restrict__ flag,
          const double* __restrict__ P,
          const double* __restrict__ Q, double* __restrict__ D, double* __restrict__ R,
          const double* __restrict__ rho, double* __restrict__ rr,
          const double* __restrict__ f2, double rtol) {
    __shared__ double red[2 * (NK_NT / 32) + 2];
    const int b = act[blockIdx.x];
    if (flag[b] & 1) return;
    const size_t off = (size_t)b * n;
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc = fma(P[off + i], Q[off + i], acc);
    const double pq = nk_sum(acc, red);
    const double alpha = pq > 0.0 ? rho[b] / pq : 0.0;
    acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        D[off + i] = fma(alpha, P[off + i], D[off + i]);
        const double r = fma(-alpha, Q[off + i], R[off + i]);
        R[off + i] = r;
        acc = fma(r, r, acc);
    }
    const double s = nk_sum(acc, red);
    if (threadIdx.x == 0) {
        rr[b] = s;
        // converged when |r| <= rtol |F(u)| (the host rule: rr > stop^2 continues)
        const double stop = rtol * sqrt(f2[b]);
        if (!(s > stop * stop)) flag[b] = 1;
    }
}

// rz = r.z ; beta = rz / rho (0 on the first) ; rho = rz ; p = z + beta p
__global__ void __launch_bounds__(NK_NT)
k_nk_cg_b(int n, const int* __restrict__ act, const int* __restrict__ flag,
          const double* __restrict__ R,
          const double* __restrict__ Z, double* __restrict__ P, double* __restrict__ rho,
          int first) {
    __shared__ double red[2 * (NK_NT / 32) + 2];
    const int b = act[blockIdx.x];
    if (flag[b] & 1) return;
    const size_t off = (size_t)b * n;
    // read rho before the reduction's barriers: thread 0 overwrites it below
    const double rho_old = rho[b];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc = fma(R[off + i], Z[off + i], acc);
    const double rz = nk_sum(acc, red);
    const double beta = first ? 0.0 : rz / rho_old;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        P[off + i] = first ? Z[off + i] : fma(beta, P[off + i], Z[off + i]);
    if (threadIdx.x == 0) rho[b] = rz;
}

// TR = U + alpha[b] D                             grid (row chunks, active)
__global__ void k_nk_trial(int n, const int* __restrict__ act, const double* __restrict__ alpha,
                           const double* __restrict__ U, const double* __restrict__ D,
                           double* __restrict__ TR) {
    const int b = act[blockIdx.y];
    const size_t off = (size_t)b * n;
    const double a = alpha[b];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        TR[off + i] = a == 1.0 ? U[off + i] + D[off + i] : fma(a, D[off + i], U[off + i]);
}

// U, F, E <- TR, FT, ET                           grid (chunks, active)
__global__ void k_nk_accept(int n, int n_elem, const int* __restrict__ act,
                            const double* __restrict__ TR, const double* __restrict__ FT,
                            const double* __restrict__ ET, double* __restrict__ U,
                            double* __restrict__ F, double* __restrict__ E,
                            const double* __restrict__ t2, double* __restrict__ f2) {
    const int b = act[blockIdx.y];
    if (blockIdx.x == 0 && threadIdx.x == 0) f2[b] = t2[b];       // |F(u)|^2 of the accepted iterate
    const size_t off = (size_t)b * n, eoff = (size_t)b * n_elem * 4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        U[off + i] = TR[off + i];
        F[off + i] = FT[off + i];
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_elem * 4;
         i += gridDim.x * blockDim.x)
        E[eoff + i] = ET[eoff + i];
}
