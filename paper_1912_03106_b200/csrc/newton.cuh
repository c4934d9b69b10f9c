// Batched damped Newton for the nonlinear (Brauer iron) model.
//
// One CTA per column runs the reference's control flow (problems.py:201-244)
// entirely on the device: residual F(u) = c M u + K_air u + N_iron(u) - rhs,
// convergence |F| <= tol * max(|rhs|, 1e-300), Newton step J(u) delta = -F by
// Jacobi-PCG (|r| <= rtol |F|), full step, else damping alpha = 0.5 with up
// to 8 halvings accepting the last trial, iteration accounting (it on early
// success, max_iters on late success), failure flag otherwise.
//
// The iron part is matrix-free and element based (2D P1, |B| = |grad A|):
//   N(u)_i   = sum_{(e,a) ni i} area_e nu_e  (g_e . grad phi_a),  g_e = G_e u_e
//   (J p)_i  = ... + area_e [ nu_e (G_e p_e . grad phi_a)
//                             + 2 nu'_e (g_e . grad phi_a)(g_e . G_e p_e) ]
// with nu = nu0 (k1 exp(k2 s^2) + k3), nu' = d nu / d s^2; per element and
// column (nu, 2 nu', g) is cached once per Newton iterate.  M and the
// non-iron stiffness K_air come from the level's CSR.
#pragma once
#include "common.cuh"

#define NW_NT 1024

struct NewtonWork {
    double* u;        // current iterate                 [B][n]
    double* F;        // residual F(u)                    [B][n]
    double* d;        // Newton step                      [B][n]
    double* rhs;      // c M u_prev + f                   [B][n]
    double* tr;       // trial iterate                    [B][n]
    double* pr;       // PCG residual                     [B][n]
    double* pp;       // PCG direction                    [B][n]
    double* pq;       // J p                              [B][n]
    double* dinv;     // Jacobi of J(u)                   [B][n]
    double* E;        // per iron element (nu, 2nu', gx, gy)  [B][n_elem][4]
    double* Et;       // same for the trial iterate
    int* nit;         // Newton iterations per column     [B]
    int* status;      // 0 ok, 1 failed                   [B]
    int* n_failed;    // [1]
    unsigned long long* iters;      // [0] cumulative, [1] this call: inner PCG iterations
    unsigned long long* newton;     // [1] Newton iterations this call
};

struct NewtonLevel {
    int n, n_elem, n_src;
    const int* __restrict__ row_ptr;
    const int* __restrict__ col_idx;
    const double* __restrict__ m_val;
    const double* __restrict__ k_val;
    const double* __restrict__ shapes;
    const int* __restrict__ edof;      // [n_elem][3]
    const double* __restrict__ egeo;   // [n_elem][7]
    const int* __restrict__ ne_ptr;    // [n+1]
    const int* __restrict__ ne;        // e*4 + a
    double nu0, k1, k2, k3;
    double tol, rtol;
    int max_iters, max_halvings, pcg_max;
    double damping;
};

#define NW_RED (2 * (NW_NT / 32))      // broadcast slots after the block_sum scratch

__device__ __forceinline__ double nw_sum(double v, double* red) {
    double a[1] = {v};
    block_sum<1>(a, red);
    if (threadIdx.x == 0) red[NW_RED] = a[0];
    __syncthreads();
    const double s = red[NW_RED];
    __syncthreads();
    return s;
}

// element pass: E[e] = (nu, 2 nu', gx, gy) of vector v
__device__ void nw_elements(const NewtonLevel& L, const double* v, double* E) {
    for (int e = threadIdx.x; e < L.n_elem; e += blockDim.x) {
        const double* gq = L.egeo + (size_t)e * 7;
        double gx = 0.0, gy = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int dof = L.edof[e * 3 + a];
            const double va = dof >= 0 ? v[dof] : 0.0;
            gx = fma(gq[a], va, gx);
            gy = fma(gq[3 + a], va, gy);
        }
        const double s2 = gx * gx + gy * gy;
        const double ex = exp(L.k2 * s2);
        double* o = E + (size_t)e * 4;
        o[0] = L.nu0 * (L.k1 * ex + L.k3);
        o[1] = 2.0 * L.nu0 * L.k1 * L.k2 * ex;
        o[2] = gx;
        o[3] = gy;
    }
}

// F(v) = c M v + K_air v + N(v) - rhs ; returns |F|^2 (all threads)
__device__ double nw_residual(const NewtonLevel& L, double c, const double* v, const double* E,
                              const double* rhs, double* F, double* red) {
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
            const double* q = E + (size_t)e * 4;
            nl = fma(gq[6] * q[0], fma(q[2], gq[a], q[3] * gq[3 + a]), nl);
        }
        const double f = fma(c, mv, kv) + nl - rhs[i];
        F[i] = f;
        acc = fma(f, f, acc);
    }
    return nw_sum(acc, red);
}

// y = J(u) p (E = element data of u)
__device__ void nw_japply(const NewtonLevel& L, double c, const double* p, const double* E,
                          double* y) {
    for (int i = threadIdx.x; i < L.n; i += blockDim.x) {
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
            const double* q = E + (size_t)e * 4;
            double tx = 0.0, ty = 0.0;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const int dof = L.edof[e * 3 + b];
                const double pb = dof >= 0 ? p[dof] : 0.0;
                tx = fma(gq[b], pb, tx);
                ty = fma(gq[3 + b], pb, ty);
            }
            const double ga = fma(q[2], gq[a], q[3] * gq[3 + a]);       // g . grad phi_a
            const double ta = fma(tx, gq[a], ty * gq[3 + a]);           // G p . grad phi_a
            const double gt = fma(q[2], tx, q[3] * ty);                 // g . G p
            nl = fma(gq[6], fma(q[0], ta, q[1] * ga * gt), nl);
        }
        y[i] = fma(c, mv, kv) + nl;
    }
}

// Jacobi diagonal of J(u)
__device__ void nw_diag(const NewtonLevel& L, double c, const double* E, double* dinv) {
    for (int i = threadIdx.x; i < L.n; i += blockDim.x) {
        double dm = 0.0, dk = 0.0;
        for (int k = L.row_ptr[i]; k < L.row_ptr[i + 1]; ++k)
            if (L.col_idx[k] == i) { dm += L.m_val[k]; dk += L.k_val[k]; }
        double nl = 0.0;
        for (int k = L.ne_ptr[i]; k < L.ne_ptr[i + 1]; ++k) {
            const int ea = L.ne[k], e = ea >> 2, a = ea & 3;
            const double* gq = L.egeo + (size_t)e * 7;
            const double* q = E + (size_t)e * 4;
            const double g2 = gq[a] * gq[a] + gq[3 + a] * gq[3 + a];
            const double ga = fma(q[2], gq[a], q[3] * gq[3 + a]);
            nl = fma(gq[6], fma(q[0], g2, q[1] * ga * ga), nl);
        }
        dinv[i] = 1.0 / (fma(c, dm, dk) + nl);
    }
}

__global__ void __launch_bounds__(NW_NT)
k_newton(NewtonLevel L, NewtonWork W, int B, const double* __restrict__ u_prev,
         const double* __restrict__ guess, const double* __restrict__ inv_dt,
         const double* __restrict__ src) {
    __shared__ double red[NW_RED + 2];
    const int b = blockIdx.x;
    const int n = L.n;
    const size_t off = (size_t)b * n;
    const double c = inv_dt[b];
    double* u = W.u + off;
    double* F = W.F + off;
    double* d = W.d + off;
    double* rhs = W.rhs + off;
    double* tr = W.tr + off;
    double* pr = W.pr + off;
    double* pp = W.pp + off;
    double* pq = W.pq + off;
    double* dinv = W.dinv + off;
    double* E = W.E + (size_t)b * L.n_elem * 4;
    double* Et = W.Et + (size_t)b * L.n_elem * 4;
    const double* up = u_prev + off;
    const double* g0 = guess ? guess + off : up;
    // rhs = c M u_prev + f ; u = guess
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double mv = 0.0;
        for (int k = L.row_ptr[i]; k < L.row_ptr[i + 1]; ++k)
            mv = fma(L.m_val[k], up[L.col_idx[k]], mv);
        double f = 0.0;
        for (int s = 0; s < L.n_src; ++s)
            f = fma(src[b * L.n_src + s], L.shapes[(size_t)s * n + i], f);
        const double r = fma(c, mv, f);
        rhs[i] = r;
        u[i] = g0[i];
        acc = fma(r, r, acc);
    }
    const double scale = fmax(sqrt(nw_sum(acc, red)), 1e-300);
    __syncthreads();
    nw_elements(L, u, E);
    __syncthreads();
    double rnorm = sqrt(nw_residual(L, c, u, E, rhs, F, red));
    int iters = -1;
    unsigned long long inner = 0;
    for (int it = 0; it < L.max_iters; ++it) {
        if (rnorm <= L.tol * scale) { iters = it; break; }
        // --- J(u) delta = -F by Jacobi-PCG, delta0 = 0
        nw_diag(L, c, E, dinv);
        __syncthreads();
        double rz = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double r = -F[i];
            pr[i] = r;
            d[i] = 0.0;
            const double z = r * dinv[i];
            pp[i] = z;
            rz = fma(r, z, rz);
        }
        double rho = nw_sum(rz, red);
        const double stop2 = L.rtol * L.rtol * rnorm * rnorm;
        double rr = rnorm * rnorm;
        int k = 0;
        while (rr > stop2 && k < L.pcg_max) {
            nw_japply(L, c, pp, E, pq);
            __syncthreads();
            double a = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) a = fma(pp[i], pq[i], a);
            const double pqs = nw_sum(a, red);
            if (!(pqs > 0.0)) break;
            const double alpha = rho / pqs;
            double v2[2] = {0.0, 0.0};
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                d[i] = fma(alpha, pp[i], d[i]);
                const double r = fma(-alpha, pq[i], pr[i]);
                pr[i] = r;
                v2[0] = fma(r * r, dinv[i], v2[0]);
                v2[1] = fma(r, r, v2[1]);
            }
            block_sum<2>(v2, red);
            if (threadIdx.x == 0) { red[NW_RED] = v2[0]; red[NW_RED + 1] = v2[1]; }
            __syncthreads();
            const double rzn = red[NW_RED];
            rr = red[NW_RED + 1];
            __syncthreads();
            const double beta = rzn / rho;
            rho = rzn;
            for (int i = threadIdx.x; i < n; i += blockDim.x)
                pp[i] = fma(beta, pp[i], pr[i] * dinv[i]);
            __syncthreads();
            ++k;
        }
        inner += k;
        // --- full step, else damped halvings (problems.py:223-236)
        for (int i = threadIdx.x; i < n; i += blockDim.x) tr[i] = u[i] + d[i];
        __syncthreads();
        nw_elements(L, tr, Et);
        __syncthreads();
        double tnorm = sqrt(nw_residual(L, c, tr, Et, rhs, pr, red));
        if (tnorm >= rnorm) {
            double alpha = L.damping;
            for (int h = 0; h < L.max_halvings; ++h) {
                for (int i = threadIdx.x; i < n; i += blockDim.x) tr[i] = fma(alpha, d[i], u[i]);
                __syncthreads();
                nw_elements(L, tr, Et);
                __syncthreads();
                tnorm = sqrt(nw_residual(L, c, tr, Et, rhs, pr, red));
                if (tnorm < rnorm) break;
                alpha *= 0.5;
            }
        }
        // accept: u, F, E <- trial
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            u[i] = tr[i];
            F[i] = pr[i];
        }
        for (int e = threadIdx.x; e < L.n_elem * 4; e += blockDim.x) E[e] = Et[e];
        __syncthreads();
        rnorm = tnorm;
    }
    if (iters < 0) iters = (rnorm <= L.tol * scale) ? L.max_iters : -1;
    if (threadIdx.x == 0) {
        W.nit[b] = iters < 0 ? L.max_iters : iters;
        W.status[b] = iters < 0 ? 1 : 0;
        if (iters < 0) atomicAdd(W.n_failed, 1);
        atomicAdd(W.iters, inner);
        atomicAdd(W.iters + 1, inner);
        atomicAdd(W.newton, (unsigned long long)(iters < 0 ? L.max_iters : iters));
    }
}

// u_out[b] = u[b] (+ g)
__global__ void k_newton_out(int n, int B, const double* __restrict__ u, double* __restrict__ out,
                             const double* __restrict__ g, const int* __restrict__ g_idx) {
    const int b = blockIdx.y;
    const double* gs = (g && g_idx && g_idx[b] >= 0) ? g + (size_t)g_idx[b] * n : nullptr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[(size_t)b * n + i] = gs ? u[(size_t)b * n + i] + gs[i] : u[(size_t)b * n + i];
}
