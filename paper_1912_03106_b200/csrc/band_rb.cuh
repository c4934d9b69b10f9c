// Register-blocked multi-column band chain (all windows W = 32 .. 512).
//
// Same recurrence as k_band_chain / k_band_pipe (band.cuh):
//     forward   y_k = D_k^-1 b_k - (D_k^-1 L_win,k) y_window
//     backward  x_k = D_k^-T y_k - (D_k^-T U_win,k) x_window
// for a group of BC columns sharing one factor, one CTA per group.  What
// changes is how a block step maps onto the SM (measured round 2,
// tools/mb/tma_mb.cu: the unicast TMA operand stream alone sustains
// ~20 TB/s into the SMs, so the old kernels -- 2.6 us per W = 512 block step
// against a 1.1 us operand-stream floor -- were bound by shared-memory
// fragment traffic and DMMA latency, not by L2):
//
//  * warp tiles.  WM x WN x WK consumer warps: warp (wm, wn, wk) owns rows
//    32/WM, columns BC/WN and every WK-th k-step of the block's 8 + W/4
//    k-steps, so one k-step is MR + NR fragment loads for MR x NR
//    independent DMMAs (m8n8k4 fp64, SASS DMMA) instead of 2 loads per DMMA.
//    The WK partial tiles are summed in a fixed order by slice 0
//    (deterministic), which writes y_k.
//  * wide groups.  BC up to 32 columns per CTA: each operand byte streamed
//    into the SM serves 32 columns (the 4,096-column level-0 batches of the
//    511^2 grid run as 128 CTAs of 32 columns).
//  * operand stream.  One producer warp streams the block operands piece by
//    piece (D^-1, then CW-column window chunks) through an NBUF-deep TMA ring
//    (cp.async.bulk + full / empty mbarriers).
//  * window ring.  NSLOT + 2 slots of 32 x BC (block b in slot b mod
//    (NSLOT + 2)); b_{k+1} is staged into its own slot during step k (that
//    slot is outside step k's window) and y_k overwrites b_k in place, so no
//    separate b buffers.  Rows are XOR-swizzled (BC >= 16) so the 4 k-rows
//    of a B fragment load hit distinct banks.  Slots of blocks outside the
//    chain start as zero (or the unit vectors of SPIKE mode), so window
//    loads need no predicates.
#pragma once
#include "band.cuh"

__device__ __forceinline__ void bar_sync_named(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int BC>
__device__ __forceinline__ int rb_swz(int row, int col) {
    // element (row, col) of a ring slot [32][BC]
    return row * BC + (BC >= 16 ? (col ^ ((row & 1) << 3)) : col);
}

__host__ __device__ constexpr int rb_nslot(int W) { return W / BD_NB + 2; }

template <int BC, int CW, int NCHK, int WM, int WN, int WK, int NBUF>
struct RbShape {
    static constexpr int NB = BD_NB;
    static constexpr int W = CW * NCHK;
    static constexpr int NSLOT = W / NB;
    static constexpr int NR = NSLOT + 2;
    static constexpr int NCW = WM * WN * WK;
    static constexpr int NCT = 32 * NCW;
    static constexpr int RW = NB / WM;
    static constexpr int MR = RW / 8;
    static constexpr int CWN = BC / WN;
    static constexpr int NRT = CWN / 8;
    static constexpr int PIECE = NB * (CW + 4) > NB * BD_PD ? NB * (CW + 4) : NB * BD_PD;
    static constexpr int NPB = 1 + NCHK;
    static constexpr int SLOT = NB * BC;
    static constexpr int NV = MR * NRT * 2;
    static constexpr size_t smem_doubles =
        (size_t)NBUF * PIECE + (size_t)NR * SLOT + (size_t)WM * WN * (WK - 1) * NV * 32;
    static_assert(WM * 8 * MR == NB, "row tiling");
    static_assert(WN * 8 * NRT == BC, "column tiling");
    static_assert(8 % WK == 0 && (CW / 4) % WK == 0, "k-slices split every piece evenly");
};

template <int BC, int CW, int NCHK, bool FWD, int WM, int WN, int WK, int NBUF>
__global__ void __launch_bounds__(32 * (WM * WN * WK + 1), 1)
k_band_rb(BandSolveArgs a) {
    using S = RbShape<BC, CW, NCHK, WM, WN, WK, NBUF>;
    constexpr int NB = S::NB, NSLOT = S::NSLOT, NR = S::NR, NCT = S::NCT;
    constexpr int MR = S::MR, NRT = S::NRT, PIECE = S::PIECE, NPB = S::NPB, SLOT = S::SLOT;
    constexpr int NV = S::NV;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF];
    double* bufs = sm;
    double* ring = bufs + (size_t)NBUF * PIECE;
    double* part = ring + (size_t)NR * SLOT;
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int col0 = ch.y, ncol = ch.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pch = a.p0 + blockIdx.y;
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const size_t blk_doubles = (size_t)NB * (BD_PD + NCHK * (CW + 4));
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };
    auto slot_of = [&](int b) { return ((b % NR) + NR) % NR; };

    if (threadIdx.x == 0) {
        for (int q = 0; q < NBUF; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], S::NCW);
        }
        mbar_fence_init();
    }
    // window ring: zero, or (SPIKE) unit vectors in the NSLOT blocks before
    // (FWD) / after (BWD) the chunk: window index wi = col0 + c
    for (int t = threadIdx.x; t < NR * SLOT; t += blockDim.x) ring[t] = 0.0;
    __syncthreads();
    if (a.spike) {
        for (int c = threadIdx.x; c < ncol; c += blockDim.x) {
            const int wi = col0 + c;
            const int b = FWD ? s0 - NSLOT + wi / NB : s1 + wi / NB;
            ring[slot_of(b) * SLOT + rb_swz<BC>(wi % NB, c)] = 1.0;
        }
    }
    __syncthreads();

    if (warp == S::NCW) {
        // ---------------- producer: the operand stream ----------------
        if (lane == 0) {
            const int total = nsteps * NPB;
            for (int P = 0; P < total; ++P) {
                const int buf = P % NBUF, use = P / NBUF;
                if (use > 0) {
                    mbar_wait(&empty[buf], (use - 1) & 1);
                    // order the consumers' generic-proxy reads of this buffer
                    // (released through the empty barrier) before the
                    // async-proxy refill: without it the TMA could overwrite
                    // operands still being read (measured round 2: 3 of 10
                    // W = 512 SPIKE runs corrupted, 0 of 20 with the fence)
                    fence_proxy_async_smem();
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

    // ---------------- consumers ----------------
    const int wk = warp % WK;
    const int wn = (warp / WK) % WN;
    const int wm = warp / (WK * WN);
    const int g = lane >> 2, q4 = lane & 3;
    const int rbase = wm * S::RW;                 // first row of this warp's tile
    const int cbase = wn * S::CWN;                // first column
    // b staging: thread t moves row t % 32 of columns t / 32 + (NCT / 32) i
    constexpr int CST = NCT / 32;
    constexpr int BPT = (BC + CST - 1) / CST;
    const int brow = threadIdx.x & 31, bcol = threadIdx.x >> 5;
    double breg[BPT];
    auto load_b = [&](int s) {
        const int rr = NB * blk_of(s) + brow;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const int cc = bcol + CST * i;
            breg[i] = (!a.spike && cc < ncol) ? a.Y[(size_t)(col0 + cc) * a.ldy + rr] : 0.0;
        }
    };
    auto store_b = [&](int s) {
        double* sl = ring + (size_t)slot_of(blk_of(s)) * SLOT;
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
            const int cc = bcol + CST * i;
            if (cc < BC) sl[rb_swz<BC>(brow, cc)] = breg[i];
        }
    };
    // fused scatter (BWD, unpartitioned chain): x straight into u_out (+ g)
    const bool fsc = !FWD && a.fz.scatter && a.P == 1 && !a.spike;
    double* fo[NRT][2];
    const double* fg[NRT][2];
#pragma unroll
    for (int ni = 0; ni < NRT; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            fo[ni][h] = nullptr;
            fg[ni][h] = nullptr;
            const int cc = cbase + 8 * ni + 2 * q4 + h;
            if (fsc && wk == 0 && cc < ncol) {
                const int b = a.fz.perm[col0 + cc];
                fo[ni][h] = a.fz.u_out + (size_t)b * a.fz.n;
                const int gi = a.fz.g ? a.fz.g_idx[b] : -1;
                fg[ni][h] = gi >= 0 ? a.fz.g + (size_t)gi * a.fz.n : nullptr;
            }
        }

    load_b(0);
    store_b(0);
    if (nsteps > 1) load_b(1);
    bar_sync_named(1, NCT);

    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        // b_{s+1} -> its slot (outside this step's window), prefetch b_{s+2}
        if (s + 1 < nsteps) {
            store_b(s + 1);
            if (s + 2 < nsteps) load_b(s + 2);
        }
        double accD[MR][NRT][2], accW[MR][NRT][2];
#pragma unroll
        for (int mi = 0; mi < MR; ++mi)
#pragma unroll
            for (int ni = 0; ni < NRT; ++ni) {
                accD[mi][ni][0] = accD[mi][ni][1] = 0.0;
                accW[mi][ni][0] = accW[mi][ni][1] = 0.0;
            }
        const double* bk = ring + (size_t)slot_of(k) * SLOT;
        const int wb0 = FWD ? k - NSLOT : k + 1;  // block of window index 0
        const int slot0 = slot_of(wb0);
#pragma unroll
        for (int j = 0; j < NPB; ++j) {
            const int P = s * NPB + j;
            const int buf = P % NBUF;
            mbar_wait(&full[buf], (P / NBUF) & 1);
            const double* pc = bufs + (size_t)buf * PIECE;
            if (j == 0) {
                // D^-1 b_k: piece 0 (row stride BD_PD), b_k in its ring slot
#pragma unroll
                for (int u = wk; u < NB / 4; u += WK) {
                    const int kk = 4 * u + q4;
                    double av[MR], bv[NRT];
#pragma unroll
                    for (int mi = 0; mi < MR; ++mi) av[mi] = pc[(rbase + 8 * mi + g) * BD_PD + kk];
#pragma unroll
                    for (int ni = 0; ni < NRT; ++ni) bv[ni] = bk[rb_swz<BC>(kk, cbase + 8 * ni + g)];
#pragma unroll
                    for (int mi = 0; mi < MR; ++mi)
#pragma unroll
                        for (int ni = 0; ni < NRT; ++ni)
                            dmma_8x8x4(accD[mi][ni][0], accD[mi][ni][1], av[mi], bv[ni]);
                }
            } else {
                // window chunk j - 1: window indices (j - 1) CW .. + CW - 1
#pragma unroll
                for (int u = wk; u < CW / 4; u += WK) {
                    const int wi = (j - 1) * CW + 4 * u;      // compile-time (+ q4)
                    const int wb = wi / NB;
                    int sl = slot0 + wb;
                    if (sl >= NR) sl -= NR;
                    const double* wsl = ring + (size_t)sl * SLOT;
                    const int kk = wi % NB + q4;
                    double av[MR], bv[NRT];
#pragma unroll
                    for (int mi = 0; mi < MR; ++mi)
                        av[mi] = pc[(rbase + 8 * mi + g) * (CW + 4) + 4 * u + q4];
#pragma unroll
                    for (int ni = 0; ni < NRT; ++ni) bv[ni] = wsl[rb_swz<BC>(kk, cbase + 8 * ni + g)];
#pragma unroll
                    for (int mi = 0; mi < MR; ++mi)
#pragma unroll
                        for (int ni = 0; ni < NRT; ++ni)
                            dmma_8x8x4(accW[mi][ni][0], accW[mi][ni][1], av[mi], bv[ni]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[buf]);
        }
        double v[NV];
#pragma unroll
        for (int mi = 0; mi < MR; ++mi)
#pragma unroll
            for (int ni = 0; ni < NRT; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    v[(mi * NRT + ni) * 2 + h] = accD[mi][ni][h] - accW[mi][ni][h];
        double* pt = part + (size_t)((wm * WN + wn) * (WK - 1 > 0 ? WK - 1 : 1)) * NV * 32;
        if constexpr (WK > 1) {
            if (wk > 0) {
#pragma unroll
                for (int e = 0; e < NV; ++e) pt[((wk - 1) * NV + e) * 32 + lane] = v[e];
            }
            bar_sync_named(1, NCT);
        }
        if (wk == 0) {
            double* yk = ring + (size_t)slot_of(k) * SLOT;       // overwrites b_k
#pragma unroll
            for (int mi = 0; mi < MR; ++mi)
#pragma unroll
                for (int ni = 0; ni < NRT; ++ni)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int e = (mi * NRT + ni) * 2 + h;
                        double y = v[e];
#pragma unroll
                        for (int q = 0; q < WK - 1; ++q) y += pt[(q * NV + e) * 32 + lane];
                        const int r = rbase + 8 * mi + g;
                        const int cc = cbase + 8 * ni + 2 * q4 + h;
                        yk[rb_swz<BC>(r, cc)] = y;
                        const int row = NB * k + r;
                        if (fsc) {
                            if (fo[ni][h] && row < a.fz.n)
                                fo[ni][h][row] = fg[ni][h] ? y + fg[ni][h][row] : y;
                        } else if (cc < ncol) {
                            a.Y[(size_t)(col0 + cc) * a.ldy + row] = y;
                        }
                    }
        }
        bar_sync_named(1, NCT);   // y_k and b_{k+1} visible; partials free
    }
}

// smem bytes of one k_band_rb instantiation
template <int BC, int CW, int NCHK, int WM, int WN, int WK, int NBUF>
constexpr size_t rb_smem_bytes() {
    return RbShape<BC, CW, NCHK, WM, WN, WK, NBUF>::smem_doubles * sizeof(double);
}

// ---------------------------------------------------------------------------
// Warp-per-column-group chain for narrow windows (the strip systems of
// strips.cuh: W = h + 1 <= 64) -- the same recurrence and operand layout as
// k_band_rb, mapped for chains whose block step is too short to amortise
// CTA-wide barriers (k_band_rb spends 2.0 us per W = 64 step against a
// 0.8 us DMMA floor).  A CTA is NWC consumer warps + one producer warp; every
// consumer warp owns its own NCW columns and all 32 rows of the block
// (4 x NCW/8 DMMA tiles), with a private window ring, so the consumer warps
// never synchronise with each other: they only share the operand stream (one
// TMA ring of pieces, full / empty mbarriers with NWC arrivals), which
// therefore serves NCW NWC columns per byte; two warps per SM sub-partition
// hide each other's fragment-load latency.  Ring slots are [column][36]
// (rows contiguous, stride 4 mod 16: conflict-free B-fragment loads), so
// b_{k+1} goes into its slot as 16-byte cp.async pieces straight from the
// column-major Y while step k runs; y_k overwrites b_k.  One accumulator per
// tile: acc = D^-1 b_k + (-(D^-1 L_win)) y_win.
#define BD_WLD 36
template <int CW, int NCHK, bool FWD, int NWC, int NCW, int NBUF>
__global__ void __launch_bounds__(32 * (NWC + 1), 1)
k_band_wcol(BandSolveArgs a) {
    constexpr int NB = BD_NB, NRT = NCW / 8, LDR = BD_WLD;
    constexpr int W = CW * NCHK, NSLOT = W / NB, NR = NSLOT + 2;
    constexpr int PIECE = NB * (CW + 4) > NB * BD_PD ? NB * (CW + 4) : NB * BD_PD;
    constexpr int NPB = 1 + NCHK, SLOT = NCW * LDR;
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t full[NBUF], empty[NBUF];
    double* bufs = sm;
    double* rings = bufs + (size_t)NBUF * PIECE;
    const int4 ch = a.chunks[blockIdx.x];
    const double* F = a.F[ch.x];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pch = a.p0 + blockIdx.y;
    const int s0 = pch * a.q;
    const int s1 = pch + 1 == a.P ? a.nblk : s0 + a.q;
    const int nsteps = s1 - s0;
    const size_t blk_doubles = (size_t)NB * (BD_PD + NCHK * (CW + 4));
    auto blk_of = [&](int s) { return FWD ? s0 + s : s1 - 1 - s; };
    auto slot_of = [&](int b) { return ((b % NR) + NR) % NR; };
    if (threadIdx.x == 0) {
        for (int q = 0; q < NBUF; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], NWC);
        }
        mbar_fence_init();
    }
    for (int t = threadIdx.x; t < NWC * NR * SLOT; t += blockDim.x) rings[t] = 0.0;
    __syncthreads();
    if (warp == NWC) {
        if (lane == 0) {
            const int total = nsteps * NPB;
            for (int P = 0; P < total; ++P) {
                const int buf = P % NBUF, use = P / NBUF;
                if (use > 0) {
                    mbar_wait(&empty[buf], (use - 1) & 1);
                    fence_proxy_async_smem();
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
    // ---------------- consumer warp: columns col0 .. col0 + NCW - 1 ----------------
    double* ring = rings + (size_t)warp * NR * SLOT;
    const int col0 = ch.y + NCW * warp;
    const int ncol = max(0, min(NCW, ch.z - NCW * warp));
    const int g = lane >> 2, q4 = lane & 3;
    // b_s -> its ring slot: 16 lanes per column (16 bytes = 2 rows each), two
    // columns per instruction
    constexpr int NST = NCW / 2;
    auto stage_b = [&](int s) {
        const uint32_t dst = smem_u32(ring + (size_t)slot_of(blk_of(s)) * SLOT);
        const size_t row = (size_t)NB * blk_of(s) + 2 * (lane & 15);
#pragma unroll
        for (int i = 0; i < NST; ++i) {
            const int c = 2 * i + (lane >> 4);
            const bool ok = c < ncol;
            const double* srcp = a.Y + (size_t)(col0 + (ok ? c : 0)) * a.ldy + row;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                             dst + 8u * (uint32_t)(c * LDR + 2 * (lane & 15))),
                         "l"(srcp), "r"(ok ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage_b(0);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    for (int s = 0; s < nsteps; ++s) {
        const int k = blk_of(s);
        if (s + 1 < nsteps) stage_b(s + 1);
        double acc[4][NRT][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < NRT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        double* bk = ring + (size_t)slot_of(k) * SLOT;
        const int slot0 = slot_of(FWD ? k - NSLOT : k + 1);
#pragma unroll
        for (int j = 0; j < NPB; ++j) {
            const int P = s * NPB + j;
            const int buf = P % NBUF;
            mbar_wait(&full[buf], (P / NBUF) & 1);
            const double* pc = bufs + (size_t)buf * PIECE;
            if (j == 0) {
                // D^-1 is lower (D^-T upper) triangular with exact zeros in
                // the other half: the 8 x 4 operand tiles that lie entirely in
                // it are skipped at compile time (12 of 32: an eighth of the
                // step's DMMAs), the result is bit-identical
#pragma unroll
                for (int u = 0; u < NB / 4; ++u) {
                    const int kk = 4 * u + q4;
                    double bv[NRT];
#pragma unroll
                    for (int ni = 0; ni < NRT; ++ni) bv[ni] = bk[(8 * ni + g) * LDR + kk];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) {
                        if (FWD ? (u > 2 * mi + 1) : (u < 2 * mi)) continue;
                        const double av = pc[(8 * mi + g) * BD_PD + kk];
#pragma unroll
                        for (int ni = 0; ni < NRT; ++ni)
                            dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av, bv[ni]);
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < CW / 4; ++u) {
                    const int wi = (j - 1) * CW + 4 * u;
                    int sl = slot0 + wi / NB;
                    if (sl >= NR) sl -= NR;
                    const double* wsl = ring + (size_t)sl * SLOT;
                    const int kk = wi % NB + q4;
                    double av[4], bv[NRT];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) av[mi] = -pc[(8 * mi + g) * (CW + 4) + 4 * u + q4];
#pragma unroll
                    for (int ni = 0; ni < NRT; ++ni) bv[ni] = wsl[(8 * ni + g) * LDR + kk];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int ni = 0; ni < NRT; ++ni)
                            dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[buf]);
        }
        // y_k: over b_k in the ring, and out to Y
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < NRT; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int r = 8 * mi + g, cc = 8 * ni + 2 * q4 + h;
                    const double y = acc[mi][ni][h];
                    bk[cc * LDR + r] = y;
                    if (cc < ncol) a.Y[(size_t)(col0 + cc) * a.ldy + NB * k + r] = y;
                }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
    }
}

template <int CW, int NCHK, int NWC, int NCW, int NBUF>
constexpr size_t wcol_smem_bytes() {
    constexpr int PIECE = BD_NB * (CW + 4) > BD_NB * BD_PD ? BD_NB * (CW + 4) : BD_NB * BD_PD;
    return ((size_t)NBUF * PIECE + (size_t)NWC * (CW * NCHK / BD_NB + 2) * NCW * BD_WLD) * sizeof(double);
}
