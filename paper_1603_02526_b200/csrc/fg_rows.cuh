// Class-L rows (packing: one row of ~5,000 edges per disk variable) on a
// 2-CTA cluster, unit-weight form.
//
// The reduceat segment of a row is a[0] + pairwise(a[1:]), and NumPy's
// pairwise tree splits its root at h = n/2 - (n/2)%8: the root is exactly
// pairwise(left h items) + pairwise(right n-h items).  CTA rank 0 of the
// cluster owns element 0 and the left subtree, rank 1 the right subtree:
//   1. one elected thread bulk-copies (cp.async.bulk, SASS UBLKCP) the CTA's
//      x and u range into shared memory -- all bytes in flight at once;
//   2. leaf sums from shared memory (8 lanes per leaf, NumPy's 8
//      accumulators and xor butterfly), then the subtree's level-ordered
//      top on warp 0;
//   3. the two subtree sums are exchanged through distributed shared
//      memory (one cluster barrier); both CTAs form the same z;
//   4. each CTA updates u of its range from shared memory.
// Every payload value crosses HBM once per iteration (x, u read; u
// written); the two CTAs of a row and the second CTA on the SM overlap
// their load, tree and update phases.  Same arithmetic order as
// k_var_large_vec, so bitwise equal to it.
#pragma once

#include <cooperative_groups.h>

#include "fg_tma.cuh"

namespace fg {

constexpr int kRowThreads = 256;

// Per row: the two subtree programs and the split.
struct Row2 { int32_t var, prog_l, prog_r, h; };

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kRowThreads, 2)
k_var_row2(PassB b, const Row2* rows, const int32_t* prog, const LExc* exc, int64_t part_off) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double row_smem[];
    __shared__ double sv[D][2 * kMaxUnits];
    __shared__ double sm[2 * (kRowThreads / 32)];
    __shared__ double s_half[2][D];                    // [rank][c] subtree sums
    __shared__ __align__(8) uint64_t s_bar;
    const int rank = (int)cluster.block_rank();
    if (b.ctrl->stop) return;                           // uniform over the grid
    const int64_t it = b.ctrl->iter;
    const Row2 R = rows[blockIdx.x >> 1];
    const int32_t v = R.var;
    const int64_t pb = b.vt.pbase[v];
    const int64_t zb = b.vt.zbase[v];
    const int deg = b.vt.deg[v];
    const LExc xe = exc[blockIdx.x >> 1];
    // element ranges: rank 0 owns [0, 1 + h) (element 0 + left subtree),
    // rank 1 owns [1 + h, deg)
    const int64_t e_lo = rank == 0 ? 0 : 1 + (int64_t)R.h;
    const int64_t e_hi = rank == 0 ? 1 + (int64_t)R.h : deg;
    const int64_t ne = e_hi - e_lo;
    const Span sx = span16(pb + e_lo * D, pb + e_hi * D);
    double* xs = row_smem;                              // aligned span of x
    double* us = row_smem + ((sx.n + 1) & ~int64_t(1));
    if (threadIdx.x == 0) {
        mbar_init(&s_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // split cluster barrier: arrive now, wait before the first write into
    // the peer's shared memory (the peer CTA must have started)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    if (threadIdx.x == 0) {
        const unsigned bytes = (unsigned)(sx.n * 8);
        mbar_expect_tx(&s_bar, 2 * bytes);
        bulk_g2s(xs, b.x + sx.lo, bytes, &s_bar);
        bulk_g2s(us, b.uin + sx.lo, bytes, &s_bar);
    }
    // what z needs besides the tree: element 0 (m checked by rank 0, whose
    // range holds it), z weights, previous z
    double a0[D], zw0[D], zo0[D];
    bool bm = false, bu = false;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double m0 = b.x[pb + c] + b.uin[pb + c];
            if (rank == 0) bm |= !finite(m0);
            a0[c] = xe.rank == 0 ? m0 * xe.rho : m0;
            zw0[c] = b.zw[zb + c];
            zo0[c] = b.zin[zb + c];
        }
    }
    mbar_wait(&s_bar, 0);
    const double* xr = xs + sx.off;                     // element e at (e - e_lo) * D
    const double* ur = us + sx.off;
    auto mval = [&](int64_t e, int c) {                 // (x + u) * rho of element e
        const int64_t q = (e - e_lo) * D + c;
        const double m = xr[q] + ur[q];
        bm |= !finite(m);
        return e == xe.rank ? m * xe.rho : m;
    };
    // ---- leaf sums of this CTA's subtree (elements from 1 + base) ----
    const int32_t* P = prog + (rank == 0 ? R.prog_l : R.prog_r);
    const int64_t base = rank == 0 ? 1 : 1 + (int64_t)R.h;
    const int nu = P[0], nlev = P[1];
    const int32_t* units = P + 2;
    const int32_t* lev = units + 2 * nu;
    const int32_t* ops = lev + nlev;
    const int g = threadIdx.x >> 3, j = threadIdx.x & 7;
    constexpr int NG = kRowThreads / 8;
    for (int r0 = 0; r0 < nu; r0 += NG) {
        const int L = r0 + g;
        int64_t s = 0, len = 0;
        if (L < nu) { s = units[2 * L]; len = units[2 * L + 1]; }
        const int64_t e0 = base + s;
        const bool small = len < kUnroll;
        const int64_t top = len - len % kUnroll;
        double acc[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        if (small) {
            if (j == 0)
                for (int64_t i = 0; i < len; ++i)
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
        } else {
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] = mval(e0 + j, c);
            for (int64_t i = kUnroll; i < top; i += kUnroll)
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i + j, c);
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double bsum = acc[c] + __shfl_xor_sync(kFull, acc[c], 1);
            bsum = bsum + __shfl_xor_sync(kFull, bsum, 2);
            bsum = bsum + __shfl_xor_sync(kFull, bsum, 4);
            if (!small) acc[c] = bsum;
        }
        if (!small && j == 0)
            for (int64_t i = top; i < len; ++i)
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
        if (L < nu && j == 0) {
#pragma unroll
            for (int c = 0; c < D; ++c) sv[c][L] = acc[c];
        }
    }
    __syncthreads();
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (threadIdx.x < 32) {                             // subtree top on warp 0
        int node = nu, op = 0;
        for (int l = 0; l < nlev; ++l) {
            const int cnt = lev[l];
            for (int o = threadIdx.x; o < cnt * D; o += 32) {
                const int c = o / cnt, oo = o - c * cnt;
                sv[c][node + oo] = sv[c][ops[2 * (op + oo)]] + sv[c][ops[2 * (op + oo) + 1]];
            }
            __syncwarp();
            node += cnt;
            op += cnt;
        }
        if (threadIdx.x < D) {                          // publish to both CTAs
            const double hs = sv[threadIdx.x][node - 1];
            s_half[rank][threadIdx.x] = hs;
            double* peer = cluster.map_shared_rank(&s_half[0][0], rank ^ 1);
            peer[rank * D + threadIdx.x] = hs;
        }
    }
    cluster.sync();                                     // both subtree sums landed
    __shared__ double s_z[2][D];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double T = s_half[0][c] + s_half[1][c];   // the root: left + right
            const double zn = ddiv(a0[c] + T, zw0[c]);
            s_z[0][c] = zn;
            s_z[1][c] = zo0[c];
            if (rank == 0) {
                b.z[zb + c] = zn;
                if (!finite(zn)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
            }
        }
    }
    __syncthreads();
    // ---- u update of this CTA's range from shared memory ----
    double zn[D], dz[D];
#pragma unroll
    for (int c = 0; c < D; ++c) { zn[c] = s_z[0][c]; dz[c] = zn[c] - s_z[1][c]; }
    double pp = 0.0, dd = 0.0;
    for (int64_t q = threadIdx.x; q < ne * D; q += kRowThreads) {
        const int64_t e = e_lo + q / D;
        const int c = (int)(q - (e - e_lo) * D);
        const bool ex = e == xe.rank;
        const double t = xr[q] - zn[c];
        pp += t * t;
        const double rd = ex ? xe.rho * dz[c] : dz[c];
        dd += rd * rd;
        const double un = ur[q] + (ex ? t * xe.alpha : t);
        b.uout[pb + e * D + c] = un;
        bu |= !finite(un);
    }
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kRowThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
}

// ---------------------------------------------------------------------------
// Class-L rows, unit-weight form, one CTA per row with a TMA ring.
//
// The row is streamed through NS shared-memory stages as a sequence of
// jobs: phase-1 chunks (consecutive whole leaves of the reduceat tree,
// <= CH elements) then phase-2 chunks (CH consecutive elements).  One
// elected thread issues the two bulk copies (x, u) of a job into a free
// stage; consumers wait on the stage's mbarrier.  The phase-2 copies of
// the first NS chunks are issued while phase 1 ends and warp 0 evaluates
// the top of the tree and z, so the load stream never stops: NS stages of
// up to 2 x 10 KB are in flight per CTA.  Same arithmetic order as
// k_var_large_vec (unit form): bitwise equal.
//
// Row plan (int32, per distinct degree): J1, J2, CH, then J1 x (elo, ehi,
// leaf_lo, leaf_hi) for the phase-1 chunks; phase-2 chunk k is elements
// [k*CH, min(deg, (k+1)*CH)).
// Per class-L row, everything a CTA needs before its first bulk copy in
// one 48-byte load (built at plan creation): payload and z base, degree,
// its TMA plan (offset, J1 phase-1 jobs, J2 phase-2 jobs, CH) and its
// tree program.
struct __align__(16) RowDesc {
    int64_t pb, zb;
    int32_t deg, planoff, progoff, J1, J2, CH;
    int32_t pad[2];
};

constexpr int kPipeMidDoubles = 2048;             // mid stage form (3 CTAs/SM at 2 stages)
constexpr int kPipeStages = 3;
constexpr int kPipeStageDoubles = 1280;             // per array per stage

template <int D, int NS = kPipeStages, int SDB = kPipeStageDoubles, bool L2HINT = false>
__global__ void __launch_bounds__(kRowThreads, NS == 3 ? 3 : (NS == 2 && SDB <= kPipeStageDoubles ? 4
                                                    : (NS == 2 && SDB <= kPipeMidDoubles ? 3 : 2)))
k_var_row_pipe(PassB b, const RowDesc* rdesc, const int32_t* prog, const int32_t* plans,
               const LExc* exc, int64_t part_off) {
    extern __shared__ __align__(16) double pipe_smem[];
    __shared__ double sv[D][2 * kMaxUnits];
    __shared__ double sm[2 * (kRowThreads / 32)];
    __shared__ double s_z[2][D];
    __shared__ __align__(8) uint64_t full[NS];
    if (b.ctrl->stop) return;
    const int64_t it = b.ctrl->iter;
    const RowDesc rd = rdesc[blockIdx.x];
    const int64_t pb = rd.pb;
    const int64_t zb = rd.zb;
    const int deg = rd.deg;
    const LExc xe = exc[blockIdx.x];
    const int J1 = rd.J1, J2 = rd.J2, CH = rd.CH;
    const int32_t* chunks = plans + rd.planoff + 3;
    const int NJ = J1 + J2;
    constexpr int SD = SDB + 4;           // array slot (span slack)
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto job_range = [&](int j, int64_t& lo, int64_t& hi) {
        if (j < J1) { lo = chunks[4 * j]; hi = chunks[4 * j + 1]; }
        else { lo = (int64_t)(j - J1) * CH; hi = lo + CH < (int64_t)deg ? lo + CH : (int64_t)deg; }
    };
    auto issue = [&](int j, int s) {
        int64_t lo, hi;
        job_range(j, lo, hi);
        const Span sx = span16(pb + lo * D, pb + hi * D);
        double* base = pipe_smem + (int64_t)s * 2 * SD;
        const unsigned bytes = (unsigned)(sx.n * 8);
        mbar_expect_tx(&full[s], 2 * bytes);
        if (L2HINT) {
            // phase-1 bytes are read again by phase 2: keep them in L2
            const uint64_t pol = j < J1 ? l2_policy_evict_last() : l2_policy_evict_first();
            bulk_g2s_hint(base, b.x + sx.lo, bytes, &full[s], pol);
            bulk_g2s_hint(base + SD, b.uin + sx.lo, bytes, &full[s], pol);
        } else {
            bulk_g2s(base, b.x + sx.lo, bytes, &full[s]);
            bulk_g2s(base + SD, b.uin + sx.lo, bytes, &full[s]);
        }
    };
    if (threadIdx.x == 0)
        for (int k = 0; k < NS && k < NJ; ++k) issue(k, k);
    // z needs element 0 (the reduceat initial value), z weights, previous z
    double a0[D], zw0[D], zo0[D];
    bool bm = false, bu = false;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double m0 = b.x[pb + c] + b.uin[pb + c];
            bm |= !finite(m0);
            a0[c] = xe.rank == 0 ? m0 * xe.rho : m0;
            zw0[c] = b.zw[zb + c];
            zo0[c] = b.zin[zb + c];
        }
    }
    const int32_t* P = prog + rd.progoff;
    const int nu = P[0], nlev = P[1];
    const int32_t* units = P + 2;
    const int32_t* lev = units + 2 * nu;
    const int32_t* ops = lev + nlev;
    // the tree top's program, staged while the first jobs load
    __shared__ int32_t s_prog[2 * kMaxUnits + 64];
    const int nops = 2 * (nu - 1);
    for (int i = threadIdx.x; i < nops + nlev; i += kRowThreads) s_prog[i] = i < nops ? ops[i] : lev[i - nops];
    const int g = threadIdx.x >> 3, j8 = threadIdx.x & 7;
    constexpr int NG = kRowThreads / 8;
    double zn[D], dz[D];
    double pp = 0.0, dd = 0.0;
    for (int j = 0; j < NJ; ++j) {
        const int s = j % NS;
        if (j == J1) {
            // all leaf sums are in: top of the tree on warp 0, z on thread 0
            __syncthreads();
            if (threadIdx.x < 32) {
                int node = nu, op = 0;
                for (int l = 0; l < nlev; ++l) {
                    const int cnt = s_prog[nops + l];
                    for (int o = threadIdx.x; o < cnt * D; o += 32) {
                        const int c = o / cnt, oo = o - c * cnt;
                        sv[c][node + oo] = sv[c][s_prog[2 * (op + oo)]] + sv[c][s_prog[2 * (op + oo) + 1]];
                    }
                    __syncwarp();
                    node += cnt;
                    op += cnt;
                }
                if (threadIdx.x == 0) {
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        const double z = ddiv(a0[c] + sv[c][node - 1], zw0[c]);
                        s_z[0][c] = z;
                        s_z[1][c] = zo0[c];
                        b.z[zb + c] = z;
                        if (!finite(z)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
                    }
                }
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < D; ++c) { zn[c] = s_z[0][c]; dz[c] = zn[c] - s_z[1][c]; }
        }
        mbar_wait(&full[s], (unsigned)((j / NS) & 1));
        int64_t lo, hi;
        job_range(j, lo, hi);
        const Span sx = span16(pb + lo * D, pb + hi * D);
        const double* X = pipe_smem + (int64_t)s * 2 * SD + sx.off;
        const double* U = X + SD;
        if (j < J1) {
            // leaves [L0, L1) of this chunk; leaf elements are 1 + unit start
            const int L0 = chunks[4 * j + 2], L1 = chunks[4 * j + 3];
            auto mval = [&](int64_t e, int c) {
                const int64_t q = (e - lo) * D + c;
                const double m = X[q] + U[q];
                bm |= !finite(m);
                return e == xe.rank ? m * xe.rho : m;
            };
            for (int L = L0 + g; L < L1; L += NG) {
                const int64_t e0 = 1 + (int64_t)units[2 * L], len = units[2 * L + 1];
                const bool small = len < kUnroll;
                const int64_t top = len - len % kUnroll;
                double acc[D];
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] = 0.0;
                const bool exl = xe.rank >= e0 && xe.rank < e0 + len;
                if (!small && !exl) {
                    // fast path: fixed strides from shared memory; a finite
                    // accumulator proves every m finite (NaN/inf propagate),
                    // only a non-finite one pays for the per-value check
                    const double* xp = X + (e0 + j8 - lo) * D;
                    const double* up = U + (e0 + j8 - lo) * D;
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = xp[c] + up[c];
                    const int nst = (int)(top / kUnroll);
                    for (int i = 1; i < nst; ++i)
#pragma unroll
                        for (int c = 0; c < D; ++c)
                            acc[c] += xp[i * kUnroll * D + c] + up[i * kUnroll * D + c];
#pragma unroll
                    for (int c = 0; c < D; ++c)
                        if (!finite(acc[c]))
                            for (int i = 0; i < nst; ++i)
                                bm |= !finite(xp[i * kUnroll * D + c] + up[i * kUnroll * D + c]);
                } else if (small) {
                    if (j8 == 0)
                        for (int64_t i = 0; i < len; ++i)
#pragma unroll
                            for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
                } else {                                   // leaf with the exception edge
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = mval(e0 + j8, c);
                    for (int64_t i = kUnroll; i < top; i += kUnroll)
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i + j8, c);
                }
                // leaf groups are warp-aligned octets: the butterfly stays
                // inside the group (all 8 lanes take the same branch)
                const unsigned gmask = 0xFFu << (threadIdx.x & 24);
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    double bs = acc[c] + __shfl_xor_sync(gmask, acc[c], 1);
                    bs = bs + __shfl_xor_sync(gmask, bs, 2);
                    bs = bs + __shfl_xor_sync(gmask, bs, 4);
                    if (!small) acc[c] = bs;
                }
                if (!small && j8 == 0)
                    for (int64_t i = top; i < len; ++i)
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
                if (j8 == 0) {
#pragma unroll
                    for (int c = 0; c < D; ++c) sv[c][L] = acc[c];
                }
            }
        } else {
            const int64_t nq = (hi - lo) * D;
            for (int64_t q = threadIdx.x; q < nq; q += kRowThreads) {
                const int64_t e = lo + q / D;
                const int c = (int)(q - (e - lo) * D);
                const bool ex = e == xe.rank;
                const double t = X[q] - zn[c];
                pp += t * t;
                const double rd = ex ? xe.rho * dz[c] : dz[c];
                dd += rd * rd;
                const double un = U[q] + (ex ? t * xe.alpha : t);
                b.uout[pb + lo * D + q] = un;
                bu |= !finite(un);
            }
        }
        __syncthreads();                               // stage s consumed
        if (threadIdx.x == 0 && j + NS < NJ) issue(j + NS, s);
    }
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kRowThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
}

// ---------------------------------------------------------------------------
// Class-L rows, unit-weight form, persistent: a grid of resident CTAs walks
// the rows (row slot blockIdx.x, + gridDim.x, ...) through ONE job ring.
// The producer thread keeps issuing the next jobs of the CTA's row sequence
// -- past the end of the current row into the next row's phase-1 chunks --
// so HBM reads continue while a row finishes its tree top, z and phase-2
// update, and no CTA start-up gap opens between rows.  Per row the jobs and
// arithmetic are k_var_row_pipe's (bitwise equal); residual partials
// accumulate per CTA (slot blockIdx.x; the class's other slots are zeroed).
template <int D, int NS, int SDB>
__global__ void __launch_bounds__(kRowThreads, NS >= 3 ? 3 : 2)
k_var_row_ring(PassB b, const RowDesc* rdesc, const int32_t* prog, const int32_t* plans,
               const LExc* exc, int64_t part_off, int32_t nrows) {
    extern __shared__ __align__(16) double pipe_smem[];
    __shared__ double sv[D][2 * kMaxUnits];
    __shared__ double sm[2 * (kRowThreads / 32)];
    __shared__ double s_z[2][D];
    __shared__ __align__(8) uint64_t full[NS];
    __shared__ int32_t s_prog[2 * kMaxUnits + 64];
    if (b.ctrl->stop) return;
    const int64_t it = b.ctrl->iter;
    const int G = gridDim.x;
    constexpr int SD = SDB + 4;           // array slot (span slack)
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // producer cursor (thread 0): row slot, job index, that row's plan
    int prs = blockIdx.x, pj = 0, pJ1 = 0, pNJ = 0, pCH = 0, pdeg = 0;
    int64_t ppb = 0;
    const int32_t* pch = nullptr;
    auto prow = [&](int rs) {
        prs = rs;
        pj = 0;
        if (rs >= nrows) return;
        const RowDesc rd = rdesc[rs];
        ppb = rd.pb;
        pdeg = rd.deg;
        pJ1 = rd.J1;
        pNJ = rd.J1 + rd.J2;
        pCH = rd.CH;
        pch = plans + rd.planoff + 3;
    };
    auto issue_next = [&](int s) {
        if (prs >= nrows) return;
        int64_t lo, hi;
        if (pj < pJ1) { lo = pch[4 * pj]; hi = pch[4 * pj + 1]; }
        else { lo = (int64_t)(pj - pJ1) * pCH; hi = lo + pCH < (int64_t)pdeg ? lo + pCH : (int64_t)pdeg; }
        const Span sx = span16(ppb + lo * D, ppb + hi * D);
        double* base = pipe_smem + (int64_t)s * 2 * SD;
        const unsigned bytes = (unsigned)(sx.n * 8);
        mbar_expect_tx(&full[s], 2 * bytes);
        bulk_g2s(base, b.x + sx.lo, bytes, &full[s]);
        bulk_g2s(base + SD, b.uin + sx.lo, bytes, &full[s]);
        if (++pj == pNJ) prow(prs + G);
    };
    if (threadIdx.x == 0) {
        prow(blockIdx.x);
        for (int k = 0; k < NS; ++k) issue_next(k);
    }
    const int g = threadIdx.x >> 3, j8 = threadIdx.x & 7;
    constexpr int NG = kRowThreads / 8;
    double pp = 0.0, dd = 0.0;
    bool bm = false, bu = false;
    int64_t gj = 0;                       // jobs consumed by this CTA
    for (int rs = blockIdx.x; rs < nrows; rs += G) {
        const RowDesc rd = rdesc[rs];
        const int64_t pb = rd.pb;
        const int64_t zb = rd.zb;
        const int deg = rd.deg;
        const LExc xe = exc[rs];
        const int J1 = rd.J1, J2 = rd.J2, CH = rd.CH;
        const int32_t* chunks = plans + rd.planoff + 3;
        const int NJ = J1 + J2;
        double a0[D], zw0[D], zo0[D];
        if (threadIdx.x == 0) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double m0 = b.x[pb + c] + b.uin[pb + c];
                bm |= !finite(m0);
                a0[c] = xe.rank == 0 ? m0 * xe.rho : m0;
                zw0[c] = b.zw[zb + c];
                zo0[c] = b.zin[zb + c];
            }
        }
        const int32_t* P = prog + rd.progoff;
        const int nu = P[0], nlev = P[1];
        const int32_t* units = P + 2;
        const int32_t* lev = units + 2 * nu;
        const int32_t* ops = lev + nlev;
        // this row's tree-top program (the previous row's top finished
        // before its phase-2 jobs, each closed by a barrier)
        const int nops = 2 * (nu - 1);
        for (int i = threadIdx.x; i < nops + nlev; i += kRowThreads) s_prog[i] = i < nops ? ops[i] : lev[i - nops];
        double zn[D], dz[D];
        for (int j = 0; j < NJ; ++j, ++gj) {
            const int s = (int)(gj % NS);
            if (j == J1) {
                __syncthreads();
                if (threadIdx.x < 32) {
                    int node = nu, op = 0;
                    for (int l = 0; l < nlev; ++l) {
                        const int cnt = s_prog[nops + l];
                        for (int o = threadIdx.x; o < cnt * D; o += 32) {
                            const int c = o / cnt, oo = o - c * cnt;
                            sv[c][node + oo] = sv[c][s_prog[2 * (op + oo)]] + sv[c][s_prog[2 * (op + oo) + 1]];
                        }
                        __syncwarp();
                        node += cnt;
                        op += cnt;
                    }
                    if (threadIdx.x == 0) {
#pragma unroll
                        for (int c = 0; c < D; ++c) {
                            const double z = ddiv(a0[c] + sv[c][node - 1], zw0[c]);
                            s_z[0][c] = z;
                            s_z[1][c] = zo0[c];
                            b.z[zb + c] = z;
                            if (!finite(z)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
                        }
                    }
                }
                __syncthreads();
#pragma unroll
                for (int c = 0; c < D; ++c) { zn[c] = s_z[0][c]; dz[c] = zn[c] - s_z[1][c]; }
            }
            mbar_wait(&full[s], (unsigned)((gj / NS) & 1));
            int64_t lo, hi;
            if (j < J1) { lo = chunks[4 * j]; hi = chunks[4 * j + 1]; }
            else { lo = (int64_t)(j - J1) * CH; hi = lo + CH < (int64_t)deg ? lo + CH : (int64_t)deg; }
            const Span sx = span16(pb + lo * D, pb + hi * D);
            const double* X = pipe_smem + (int64_t)s * 2 * SD + sx.off;
            const double* U = X + SD;
            if (j < J1) {
                const int L0 = chunks[4 * j + 2], L1 = chunks[4 * j + 3];
                auto mval = [&](int64_t e, int c) {
                    const int64_t q = (e - lo) * D + c;
                    const double m = X[q] + U[q];
                    bm |= !finite(m);
                    return e == xe.rank ? m * xe.rho : m;
                };
                for (int L = L0 + g; L < L1; L += NG) {
                    const int64_t e0 = 1 + (int64_t)units[2 * L], len = units[2 * L + 1];
                    const bool small = len < kUnroll;
                    const int64_t top = len - len % kUnroll;
                    double acc[D];
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] = 0.0;
                    const bool exl = xe.rank >= e0 && xe.rank < e0 + len;
                    if (!small && !exl) {
                        const double* xp = X + (e0 + j8 - lo) * D;
                        const double* up = U + (e0 + j8 - lo) * D;
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] = xp[c] + up[c];
                        const int nst = (int)(top / kUnroll);
                        for (int i = 1; i < nst; ++i)
#pragma unroll
                            for (int c = 0; c < D; ++c)
                                acc[c] += xp[i * kUnroll * D + c] + up[i * kUnroll * D + c];
#pragma unroll
                        for (int c = 0; c < D; ++c)
                            if (!finite(acc[c]))
                                for (int i = 0; i < nst; ++i)
                                    bm |= !finite(xp[i * kUnroll * D + c] + up[i * kUnroll * D + c]);
                    } else if (small) {
                        if (j8 == 0)
                            for (int64_t i = 0; i < len; ++i)
#pragma unroll
                                for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
                    } else {
#pragma unroll
                        for (int c = 0; c < D; ++c) acc[c] = mval(e0 + j8, c);
                        for (int64_t i = kUnroll; i < top; i += kUnroll)
#pragma unroll
                            for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i + j8, c);
                    }
                    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        double bs = acc[c] + __shfl_xor_sync(gmask, acc[c], 1);
                        bs = bs + __shfl_xor_sync(gmask, bs, 2);
                        bs = bs + __shfl_xor_sync(gmask, bs, 4);
                        if (!small) acc[c] = bs;
                    }
                    if (!small && j8 == 0)
                        for (int64_t i = top; i < len; ++i)
#pragma unroll
                            for (int c = 0; c < D; ++c) acc[c] += mval(e0 + i, c);
                    if (j8 == 0) {
#pragma unroll
                        for (int c = 0; c < D; ++c) sv[c][L] = acc[c];
                    }
                }
            } else {
                const int64_t nq = (hi - lo) * D;
                for (int64_t q = threadIdx.x; q < nq; q += kRowThreads) {
                    const int64_t e = lo + q / D;
                    const int c = (int)(q - (e - lo) * D);
                    const bool ex = e == xe.rank;
                    const double t = X[q] - zn[c];
                    pp += t * t;
                    const double rd = ex ? xe.rho * dz[c] : dz[c];
                    dd += rd * rd;
                    const double un = U[q] + (ex ? t * xe.alpha : t);
                    b.uout[pb + lo * D + q] = un;
                    bu |= !finite(un);
                }
            }
            __syncthreads();                               // stage s consumed
            if (threadIdx.x == 0) issue_next(s);
        }
    }
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kRowThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
    for (int64_t k = blockIdx.x + G + threadIdx.x * (int64_t)G; k < nrows; k += (int64_t)G * kRowThreads) {
        b.part[2 * (part_off + k)] = 0.0;
        b.part[2 * (part_off + k) + 1] = 0.0;
    }
}

inline size_t row_pipe_smem(int ns = kPipeStages, int sdb = kPipeStageDoubles) {
    return (size_t)ns * 2 * (sdb + 4) * sizeof(double);
}

}  // namespace fg
