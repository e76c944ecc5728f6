// Class-L rows (packing: one row of ~5,000 edges per disk variable),
// unit-weight form: one CTA per row streaming the row through a TMA ring
// (k_var_row_pipe below).  Every payload value crosses HBM once per
// iteration for the sums and once for the update (x, u read; u written).
// Same arithmetic order as k_var_large_vec, so bitwise equal to it.
//
// Two other forms were built, tested bitwise and measured slower on pack
// N=5000 (profiles/r01_rows_ab.md), then removed: a 2-CTA cluster per row
// exchanging the two subtree sums through distributed shared memory (d1
// 0.257 vs 0.192 ms), and a persistent ring streaming the next row during
// a row's tree top and update (equal at best).
#pragma once


#include "fg_tma.cuh"

namespace fg {

constexpr int kRowThreads = 256;
#ifndef FG_ROW_FIXC
#define FG_ROW_FIXC 1
#endif

// ---------------------------------------------------------------------------
// Class-L rows, unit-weight form, one CTA per row with a TMA ring.
//
// The row is streamed through NS = 2 shared-memory stages as a sequence of
// jobs: phase-1 chunks (consecutive whole leaves of the reduceat tree,
// <= CH elements) then phase-2 chunks (CH consecutive elements).  One
// elected thread issues the two bulk copies (x, u) of a job into a free
// stage; consumers wait on the stage's mbarrier.  The phase-2 copies of
// the first NS chunks are issued while phase 1 ends and warp 0 evaluates
// the top of the tree and z, so the load stream never stops.  Stage size
// SDB (doubles per array): 1280 at 5 CTAs/SM for dim-1 rows (48 registers;
// pack N=5000 radius rows 0.130 ms, 0.133 at 4 CTAs/SM, 0.157 with three
// stages at 3), 2048 at 3 CTAs/SM for
// dim >= 2 rows (center rows 0.254 vs 0.264 ms with 2 x 2560 at 2 CTAs/SM;
// profiles/r01_rows_ab.md).  L2HINT: phase-1 copies are marked L2
// evict_last (phase 2 reads the same bytes again), phase-2 copies
// evict_first (HBM re-reads 924 -> 816 MB against 800 MB algorithmic).
// Same arithmetic order as k_var_large_vec (unit form): bitwise equal.
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

constexpr int kPipeMidDoubles = 2048;               // dim >= 2 rows: 3 CTAs/SM
constexpr int kPipeStageDoubles = 1280;             // dim-1 rows: 5 CTAs/SM
constexpr int kPipeNS = 2;                          // stages

template <int D, int SDB, bool L2HINT>
__global__ void __launch_bounds__(kRowThreads, SDB <= kPipeStageDoubles ? 5 : 3)
k_var_row_pipe(PassB b, const RowDesc* rdesc, const int32_t* prog, const int32_t* plans,
               const LExc* exc, int64_t part_off) {
    extern __shared__ __align__(16) double pipe_smem[];
    __shared__ double sv[D][2 * kMaxUnits];
    __shared__ double sm[2 * (kRowThreads / 32)];
    __shared__ double s_z[2][D];
    constexpr int NS = kPipeNS;
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
            if (D == 1) {
                // 32-bit job-local indices (dim-1 rows: 2% faster); the
                // exception edge, if in this job, as a job-local index
                const int nq = (int)(hi - lo);
                const int exl = (xe.rank >= lo && xe.rank < hi) ? (int)(xe.rank - lo) : -1;
                double* __restrict__ uo = b.uout + pb + lo;
                for (int q = threadIdx.x; q < nq; q += kRowThreads) {
                    const bool ex = q == exl;
                    const double t = X[q] - zn[0];
                    pp += t * t;
                    const double rd = ex ? xe.rho * dz[0] : dz[0];
                    dd += rd * rd;
                    const double un = U[q] + (ex ? t * xe.alpha : t);
                    uo[q] = un;
                    bu |= !finite(un);
                }
            } else if (FG_ROW_FIXC && kRowThreads % D == 0) {
                // D divides the block: thread t always meets component
                // t % D, so z, dz and the exception edge's element are
                // per-thread constants (no division, 32-bit indices)
                const int nq = (int)((hi - lo) * D);
                const int c = threadIdx.x % D;
                double znc = zn[0], dzc = dz[0];
#pragma unroll
                for (int k = 1; k < D; ++k)
                    if (c == k) { znc = zn[k]; dzc = dz[k]; }
                const int exq = (xe.rank >= lo && xe.rank < hi) ? (int)(xe.rank - lo) * D + c : -1;
                double* __restrict__ uo = b.uout + pb + lo * D;
                for (int q = threadIdx.x; q < nq; q += kRowThreads) {
                    const bool ex = q == exq;
                    const double t = X[q] - znc;
                    pp += t * t;
                    const double rd = ex ? xe.rho * dzc : dzc;
                    dd += rd * rd;
                    const double un = U[q] + (ex ? t * xe.alpha : t);
                    uo[q] = un;
                    bu |= !finite(un);
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

inline size_t row_pipe_smem(int sdb) {
    return (size_t)kPipeNS * 2 * (sdb + 4) * sizeof(double);
}

}  // namespace fg
