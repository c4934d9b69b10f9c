// rhs stencil microbenchmark (dev tool): b = c M u + f over B columns of a
// 127^2 7-point stencil, three thread mappings, CUDA-event timed.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
constexpr int N = 128, NI = N - 1, n = NI * NI, LDY = (n + 31) / 32 * 32, B = 1024;
__constant__ int offs[4] = {0, 1, NI, NI + 1};

// V0: copy only, thread = row, CTA = 256 rows x 32 columns
__global__ void v0(const double* __restrict__ u, double* __restrict__ Y) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    for (int j = 0; j < 32; ++j) {
        const int c = blockIdx.y * 32 + j;
        Y[(size_t)c * LDY + i] = u[(size_t)c * n + i];
    }
}
// V1: stencil, thread = row, CTA = 256 rows x 32 columns (library layout)
__global__ void v1(const double* __restrict__ u, const double* __restrict__ m, double* __restrict__ Y) {
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    double mu[4], ml[4];
    int ou[4], ol[4];
    for (int k = 0; k < 4; ++k) {
        const int o = offs[k];
        mu[k] = i + o < n ? m[k * n + i] : 0.0;
        ml[k] = (k > 0 && i - o >= 0) ? m[k * n + i - o] : 0.0;
        ou[k] = i + o < n ? o : 0;
        ol[k] = i - o >= 0 ? -o : 0;
    }
    for (int j = 0; j < 32; ++j) {
        const int c = blockIdx.y * 32 + j;
        const double* ub = u + (size_t)c * n + i;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v = fma(mu[k], ub[ou[k]], fma(ml[k], ub[ol[k]], v));
        Y[(size_t)c * LDY + i] = v;
    }
}
// V2: stencil, CTA = one column x 1024-row tile, 4 rows per thread (strided)
__global__ void v2(const double* __restrict__ u, const double* __restrict__ m, double* __restrict__ Y) {
    const int c = blockIdx.y;
    const double* uc = u + (size_t)c * n;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int i = blockIdx.x * 1024 + r * 256 + threadIdx.x;
        if (i >= n) return;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int o = offs[k];
            if (i + o < n) v = fma(m[k * n + i], uc[i + o], v);
            if (k > 0 && i - o >= 0) v = fma(m[k * n + i - o], uc[i - o], v);
        }
        Y[(size_t)c * LDY + i] = v;
    }
}
// V3: like V1 but grid x = column chunk fastest (row tile slow)
__global__ void v3(const double* __restrict__ u, const double* __restrict__ m, double* __restrict__ Y) {
    const int i = blockIdx.y * 256 + threadIdx.x;
    if (i >= n) return;
    double mu[4], ml[4];
    int ou[4], ol[4];
    for (int k = 0; k < 4; ++k) {
        const int o = offs[k];
        mu[k] = i + o < n ? m[k * n + i] : 0.0;
        ml[k] = (k > 0 && i - o >= 0) ? m[k * n + i - o] : 0.0;
        ou[k] = i + o < n ? o : 0;
        ol[k] = i - o >= 0 ? -o : 0;
    }
    for (int j = 0; j < 32; ++j) {
        const int c = blockIdx.x * 32 + j;
        const double* ub = u + (size_t)c * n + i;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v = fma(mu[k], ub[ou[k]], fma(ml[k], ub[ol[k]], v));
        Y[(size_t)c * LDY + i] = v;
    }
}
#define BD_RHS_SRC 8
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


template <int NIT>
__global__ void __launch_bounds__(256)
v12(RhsDia a0, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
               const double* __restrict__ src, const int* __restrict__ perm,
               double* __restrict__ Y) {
    RhsDia a = a0;
    a.n = NIT * NIT; a.U = 3; a.off[1] = 1; a.off[2] = NIT; a.off[3] = NIT + 1; a.off[4] = 0;
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


#define CC2 16
__global__ void __launch_bounds__(256)
v11(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
               const double* __restrict__ src, const int* __restrict__ perm,
               double* __restrict__ Y) {
    __shared__ const double* sp[CC2];
    __shared__ double sc[CC2], ss[CC2][BD_RHS_SRC];
    const int gc0 = blockIdx.y * CC2;
    const int ncol = min(CC2, a.B - gc0);
    for (int t = threadIdx.x; t < CC2 * BD_RHS_SRC; t += blockDim.x) {
        const int j = t / BD_RHS_SRC, q = t % BD_RHS_SRC;
        const int b = j < ncol ? perm[gc0 + j] : 0;
        if (q == 0) {
            sp[j] = u_prev + (size_t)b * a.n;
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
        const double* ub = sp[j] + i;
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


// V5: library kernel minus the source term
__global__ void __launch_bounds__(256)
v5(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
   const int* __restrict__ perm, double* __restrict__ Y) {
    __shared__ int sp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    if (threadIdx.x < BD_RHS_CC) { const int b = perm[gc0 + threadIdx.x]; sp[threadIdx.x] = b; sc[threadIdx.x] = inv_dt[b]; }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
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
        oup[u] = hu ? o : 0;
        olo[u] = hl ? -o : 0;
    }
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll 4
    for (int j = 0; j < ncol; ++j) {
        const double* ub = u_prev + (size_t)sp[j] * a.n + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < 4; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        yo[(size_t)j * a.ldy] = sc[j] * v;
    }
}

// V9: column pointers in smem
__global__ void __launch_bounds__(256)
v9(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
   const int* __restrict__ perm, double* __restrict__ Y) {
    __shared__ const double* spp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    if (threadIdx.x < BD_RHS_CC) { const int b = perm[gc0 + threadIdx.x]; spp[threadIdx.x] = u_prev + (size_t)b * a.n; sc[threadIdx.x] = inv_dt[b]; }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
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
        oup[u] = hu ? o : 0;
        olo[u] = hl ? -o : 0;
    }
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll 4
    for (int j = 0; j < ncol; ++j) {
        const double* ub = spp[j] + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < 4; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        yo[(size_t)j * a.ldy] = sc[j] * v;
    }
}

// V10: arithmetic columns
__global__ void __launch_bounds__(256)
v10(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
   const int* __restrict__ perm, double* __restrict__ Y) {
    __shared__ int sp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    if (threadIdx.x < BD_RHS_CC) { const int b = perm[gc0 + threadIdx.x]; sp[threadIdx.x] = b; sc[threadIdx.x] = inv_dt[b]; }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
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
        oup[u] = hu ? o : 0;
        olo[u] = hl ? -o : 0;
    }
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll 4
    for (int j = 0; j < ncol; ++j) {
        const double* ub = u_prev + (size_t)(gc0 + j) * a.n + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < 4; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        yo[(size_t)j * a.ldy] = sc[j] * v;
    }
}

// V6
__global__ void __launch_bounds__(256, 4)
v6(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
   const int* __restrict__ perm, double* __restrict__ Y) {
    __shared__ int sp[BD_RHS_CC];
    __shared__ double sc[BD_RHS_CC];
    const int gc0 = blockIdx.y * BD_RHS_CC;
    const int ncol = min(BD_RHS_CC, a.B - gc0);
    if (threadIdx.x < BD_RHS_CC) { const int b = perm[gc0 + threadIdx.x]; sp[threadIdx.x] = b; sc[threadIdx.x] = inv_dt[b]; }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
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
        oup[u] = hu ? o : 0;
        olo[u] = hl ? -o : 0;
    }
    double* yo = Y + (size_t)gc0 * a.ldy + i;
#pragma unroll 4
    for (int j = 0; j < ncol; ++j) {
        const double* ub = u_prev + (size_t)sp[j] * a.n + i;
        double v = m0 * ub[0];
#pragma unroll
        for (int u = 0; u < 4; ++u) v = fma(mup[u], ub[oup[u]], fma(mlo[u], ub[olo[u]], v));
        yo[(size_t)j * a.ldy] = sc[j] * v;
    }
}

__global__ void __launch_bounds__(256, 4)
v7(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
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


__global__ void __launch_bounds__(256, 6)
v8(RhsDia a, const double* __restrict__ u_prev, const double* __restrict__ inv_dt,
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
#pragma unroll 2
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



// v13..v16: v1's structure plus, step by step, what the library kernel needs
template <int STAGE>
__global__ void __launch_bounds__(256) vs(const double* __restrict__ u, const double* __restrict__ m,
                                         const int* __restrict__ perm, const double* __restrict__ idt,
                                         const double* __restrict__ srcv, const double* __restrict__ shp,
                                         double* __restrict__ Y) {
    __shared__ int sp[32];
    __shared__ double sc[32], ss[32][8];
    if (STAGE >= 1) {
        for (int t = threadIdx.x; t < 32 * 8; t += 256) {
            const int j = t / 8, q = t % 8;
            const int b = perm[blockIdx.y * 32 + j];
            if (q == 0) { sp[j] = b; sc[j] = idt[b]; }
            ss[j][q] = q < 6 ? srcv[b * 6 + q] : 0.0;
        }
        __syncthreads();
    }
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    double mu[4], ml[4];
    int ou[4], ol[4];
    for (int k = 0; k < 4; ++k) {
        const int o = offs[k];
        mu[k] = i + o < n ? m[k * n + i] : 0.0;
        ml[k] = (k > 0 && i - o >= 0) ? m[k * n + i - o] : 0.0;
        ou[k] = i + o < n ? o : 0;
        ol[k] = i - o >= 0 ? -o : 0;
    }
    double sh[8];
    bool has = false;
    if (STAGE >= 3) {
#pragma unroll
        for (int q = 0; q < 8; ++q) { sh[q] = q < 6 ? shp[q * n + i] : 0.0; has |= sh[q] != 0.0; }
    }
    for (int j = 0; j < 32; ++j) {
        const int c = blockIdx.y * 32 + j;
        const int b = STAGE >= 1 ? sp[j] : c;
        const double* ub = u + (size_t)b * n + i;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) v = fma(mu[k], ub[ou[k]], fma(ml[k], ub[ol[k]], v));
        if (STAGE == 2) v *= sc[j];
        if (STAGE == 4) v *= 1.5;
        if (STAGE == 5) v *= idt[b];
        if (STAGE >= 3 && has) {
            double f = 0.0;
#pragma unroll
            for (int q = 0; q < 8; ++q) f = fma(ss[j][q], sh[q], f);
            v += f;
        }
        Y[(size_t)c * LDY + i] = v;
    }
}

// vb<R>: library semantics (perm, c, sources) with R columns' stencil loads
// issued as one batch before any arithmetic
template <int R>
__global__ void __launch_bounds__(256) vb(const double* __restrict__ u, const double* __restrict__ m,
                                         const int* __restrict__ perm, const double* __restrict__ idt,
                                         const double* __restrict__ srcv, const double* __restrict__ shp,
                                         double* __restrict__ Y) {
    __shared__ int sp[32];
    __shared__ double sc[32], ss[32][8];
    for (int t = threadIdx.x; t < 32 * 8; t += 256) {
        const int j = t / 8, q = t % 8;
        const int b = perm[blockIdx.y * 32 + j];
        if (q == 0) { sp[j] = b; sc[j] = idt[b]; }
        ss[j][q] = q < 6 ? srcv[b * 6 + q] : 0.0;
    }
    __syncthreads();
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= n) return;
    double mv[8];
    int ov[8];
    for (int k = 0; k < 4; ++k) {
        const int o = offs[k];
        mv[2 * k] = i + o < n ? m[k * n + i] : 0.0;
        mv[2 * k + 1] = (k > 0 && i - o >= 0) ? m[k * n + i - o] : 0.0;
        ov[2 * k] = i + o < n ? o : 0;
        ov[2 * k + 1] = i - o >= 0 ? -o : 0;
    }
    double sh[8];
    bool has = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) { sh[q] = q < 6 ? shp[q * n + i] : 0.0; has |= sh[q] != 0.0; }
    for (int j0 = 0; j0 < 32; j0 += R) {
        double uv[R][8];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double* ub = u + (size_t)sp[j0 + r] * n + i;
#pragma unroll
            for (int q = 0; q < 8; ++q) uv[r][q] = ub[ov[q]];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int j = j0 + r;
            double v = mv[0] * uv[r][0];
#pragma unroll
            for (int q = 1; q < 8; ++q) v = fma(mv[q], uv[r][q], v);
            double f = 0.0;
            if (has) {
#pragma unroll
                for (int q = 0; q < 8; ++q) f = fma(ss[j][q], sh[q], f);
            }
            Y[(size_t)(blockIdx.y * 32 + j) * LDY + i] = fma(sc[j], v, f);
        }
    }
}
int main() {
    double *u, *m, *Y;
    cudaMalloc(&u, (size_t)B * n * 8);
    cudaMalloc(&Y, (size_t)B * LDY * 8);
    cudaMalloc(&m, (size_t)4 * n * 8);
    cudaMemset(u, 0, (size_t)B * n * 8);
    cudaMemset(m, 0, (size_t)4 * n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 2.0 * B * n * 8;
    double2* mk; cudaMalloc(&mk, (size_t)4 * n * 16); cudaMemset(mk, 0, (size_t)4 * n * 16);
    double* sh; cudaMalloc(&sh, (size_t)6 * n * 8); cudaMemset(sh, 0, (size_t)6 * n * 8);
    double *idt, *srcv; cudaMalloc(&idt, B * 8); cudaMalloc(&srcv, B * 6 * 8);
    cudaMemset(idt, 0, B * 8); cudaMemset(srcv, 0, B * 6 * 8);
    int* perm; cudaMalloc(&perm, B * 4);
    { std::vector<int> p(B); for (int b = 0; b < B; ++b) p[b] = b; cudaMemcpy(perm, p.data(), B * 4, cudaMemcpyHostToDevice); }
    RhsDia ra{n, LDY, B, 3, 6, {0, 1, NI, NI + 1, 0}, mk, sh};
    for (int v = 0; v < 22; ++v) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (v == 0) v0<<<dim3((n + 255) / 256, B / 32), 256>>>(u, Y);
            if (v == 1) v1<<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, Y);
            if (v == 2) v2<<<dim3((n + 1023) / 1024, B), 256>>>(u, m, Y);
            if (v == 3) v3<<<dim3(B / 32, (n + 255) / 256), 256>>>(u, m, Y);
            if (v == 4) k_band_rhs_dia<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, srcv, perm, Y);
            if (v == 6) v6<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, perm, Y);
            if (v == 7) v7<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, srcv, perm, Y);
            if (v == 8) v8<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, srcv, perm, Y);
            if (v == 9) v9<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, perm, Y);
            if (v == 10) v10<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, perm, Y);
            if (v == 11) v11<<<dim3((LDY + 255) / 256, B / CC2), 256>>>(ra, u, idt, srcv, perm, Y);
            if (v == 12) v12<NI><<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, srcv, perm, Y);
            if (v == 13) vs<1><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 14) vs<2><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 15) vs<3><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 16) vs<0><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 17) vs<4><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 18) vs<5><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 19) vb<1><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 20) vb<2><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 21) vb<4><<<dim3((n + 255) / 256, B / 32), 256>>>(u, m, perm, idt, srcv, sh, Y);
            if (v == 5) v5<<<dim3((LDY + 255) / 256, B / BD_RHS_CC), 256>>>(ra, u, idt, perm, Y);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("v%d: %.1f us  %.0f GB/s\n", v, best * 1e3, bytes / best / 1e6);
    }
    return 0;
}
