// Variable-pass kernels for regular layouts (the hot path of every
// benchmark family).
//
// * k_var_small_run: class S (degree <= 32) organised in runs of
//   consecutive variables with one (dim, degree): addresses are affine in
//   the component index, so a thread goes straight from its index to its
//   segment.  For degree <= 8 the whole segment (x, u, rho, alpha) is
//   loaded into registers up front (4*deg independent loads in flight),
//   summed, and updated without a second read.
// * k_var_large_vec<D>: class L, one CTA per VARIABLE (all D components
//   together): an element's D payload values are contiguous, so the 8
//   lanes of a leaf group read 8*D*8 contiguous bytes, and rho/alpha are
//   read once per element instead of once per component.
// Both replay the NumPy reduceat tree exactly (see fg_device.cuh).
#pragma once

#include "fg_kernels.cuh"

namespace fg {

struct SRun {
    int64_t pb0, zb0;        // payload / z base of the run's first variable
    int32_t eb0, nv, d, deg; // edge base, variables, dim, degree
};
struct SBlock { int32_t run, c0, c1, pad; };   // CTA -> run components [c0, c1)

constexpr int kSmallRegDeg = 8;
constexpr int kSmallTinyDeg = 4;
constexpr int kSmallCompsPerCta = 4 * 256;
constexpr int kLargeThreads = 512;   // CTA of the one-variable large kernel

template <int DMAX, int MODE>
__global__ void __launch_bounds__(256, 4) k_var_small_run(PassB b, const SRun* runs,
                                                       const SBlock* blocks,
                                                       int64_t part_off) {
    __shared__ double sm[16];
    const SBlock bk = blocks[blockIdx.x];
    const SRun R = runs[bk.run];
    if (b.ctrl->stop) return;                // uniform: set only between kernels
    const int64_t it = b.ctrl->iter;
    double pp = 0.0, dd = 0.0;
    for (int32_t q = bk.c0 + (int32_t)threadIdx.x; q < bk.c1; q += 256) {
        const int32_t vl = (int32_t)((uint32_t)q / (uint32_t)R.d);
        const int c = q - vl * R.d;
        const int d = R.d, deg = R.deg;
        const int64_t pb = R.pb0 + (int64_t)vl * deg * d + c;
        const int64_t eb = R.eb0 + (int64_t)vl * deg;
        const int64_t k = R.zb0 + q;
        const double* msrc = (MODE == MODE_FUSED) ? b.uin : b.msrc;
        bool bm = false, bu = false;
        if (DMAX > 0) {
            constexpr int NR = DMAX > 0 ? DMAX : 1;
            double xv[NR], uv[NR], rv[NR], av[NR];
            // z_old and z_weights are issued with the segment loads so the
            // whole component costs one memory round trip
            const double zo = (MODE == MODE_FUSED) ? b.zin[k] : 0.0;
            const double zw = b.zw[k];
#pragma unroll
            for (int e = 0; e < DMAX; ++e) {
                if (e < deg) {
                    uv[e] = msrc[pb + (int64_t)e * d];
                    rv[e] = b.rho[eb + e];
                    if (MODE == MODE_FUSED) {
                        xv[e] = b.x[pb + (int64_t)e * d];
                        av[e] = b.alpha[eb + e];
                    }
                }
            }
            double S = 0.0, res = 0.0;
#pragma unroll
            for (int e = 0; e < DMAX; ++e) {
                if (e < deg) {
                    double m = uv[e];
                    if (MODE == MODE_FUSED) {
                        m = xv[e] + uv[e];                   // phase m
                        bm |= !finite(m);
                    }
                    const double val = m * rv[e];
                    if (e == 0) S = val;
                    else res += val;                         // leaf, n < 8
                }
            }
            if (deg > 1) S = S + res;                        // a[0] + tree
            const double zn = ddiv(S, zw);
            if (MODE == MODE_FUSED) {
                b.z[k] = zn;
                const double dz = zn - zo;
#pragma unroll
                for (int e = 0; e < DMAX; ++e) {
                    if (e < deg) {
                        const double t = xv[e] - zn;
                        pp += t * t;
                        const double rd = rv[e] * dz;
                        dd += rd * rd;
                        const double un = uv[e] + t * av[e];
                        b.uout[pb + (int64_t)e * d] = un;
                        bu |= !finite(un);
                    }
                }
                if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
                if (!finite(zn)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
                if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
            } else {
                b.z[k] = zn;
            }
        } else {
            CompRef r;
            r.pb = pb - c;
            r.eb = (int32_t)eb;
            r.deg = deg;
            r.d = d;
            r.c = c;
            ValFn<MODE> val(b, r, &bm);
            double S = val(0);
            if (deg > 1) S = S + leaf_seq(val, 1, deg - 1);
            const double zn = ddiv(S, b.zw[k]);
            if (MODE == MODE_FUSED) {
                const double zo = b.zin[k];
                b.z[k] = zn;
                update_range(b, r, 0, deg, 1, zn, zo, pp, dd, bu);
                if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
                if (!finite(zn)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
                if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
            } else {
                b.z[k] = zn;
            }
        }
    }
    if (MODE == MODE_FUSED) {
        block_sum2<256>(pp, dd, sm);
        if (threadIdx.x == 0) {
            b.part[2 * (part_off + blockIdx.x)] = pp;
            b.part[2 * (part_off + blockIdx.x) + 1] = dd;
        }
    }
}

// Class L, one CTA per variable with D components.
// Unit-weight rows: at most one edge per row has rho or alpha != 1 (its
// rank and weights in the row's LExc, k_unit_rows; rank -1 for none).
// UNIT: rows in unit-weight form: every other weight is exactly 1, and
// m*1, rho*dz and t*1 are exact identities, so no rho/alpha loads.
template <int D, int MODE, bool UNIT = false, int NT = kLargeThreads>
__global__ void __launch_bounds__(NT, 1024 / NT) k_var_large_vec(
    PassB b, const int32_t* vlist, const int32_t* progoff, const int32_t* prog,
    int64_t part_off, const LExc* exc = nullptr) {
    __shared__ double sv[D][2 * kMaxUnits];
    __shared__ double sm[2 * (NT / 32)];
    __shared__ double s_z[2][D];
    __shared__ int s_stop;
    if (threadIdx.x == 0) s_stop = b.ctrl->stop;
    __syncthreads();
    if (s_stop) return;
    const int64_t it = b.ctrl->iter;
    const int32_t v = vlist[blockIdx.x];
    const int64_t pb = b.vt.pbase[v];
    const int64_t eb = b.vt.ebase[v];
    const int64_t zb = b.vt.zbase[v];
    const int deg = b.vt.deg[v];
    const double* msrc = (MODE == MODE_FUSED) ? b.uin : b.msrc;
    bool bm = false, bu = false;
    LExc xe{-1, 0, 1.0, 1.0};
    if (UNIT) xe = exc[blockIdx.x];
    // element e -> D values of m*rho
    auto vals = [&](int64_t e, double* out) {
        const double r = UNIT ? (e == xe.rank ? xe.rho : 1.0) : b.rho[eb + e];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double m = msrc[pb + e * D + c];
            if (MODE == MODE_FUSED) {
                m = b.x[pb + e * D + c] + m;
                bm |= !finite(m);
            }
            out[c] = m * r;
        }
    };
    const int32_t* P = prog + progoff[blockIdx.x];
    const int nu = P[0], nlev = P[1];
    const int32_t* units = P + 2;
    const int32_t* lev = units + 2 * nu;
    const int32_t* ops = lev + nlev;
    // thread 0 prefetches what z needs besides the tree: a[0], z weights and
    // the previous z (independent loads, issued before the leaf phase)
    double a0[D], zw0[D], zo0[D];
    if (threadIdx.x == 0) {
        vals(0, a0);
#pragma unroll
        for (int c = 0; c < D; ++c) {
            zw0[c] = b.zw[zb + c];
            zo0[c] = (MODE == MODE_FUSED) ? b.zin[zb + c] : 0.0;
        }
    }
    const int g = threadIdx.x >> 3, j = threadIdx.x & 7;
    constexpr int NG = NT / 8;
    for (int r0 = 0; r0 < nu; r0 += NG) {
        const int L = r0 + g;
        int64_t s = 0, len = 0;
        if (L < nu) { s = units[2 * L]; len = units[2 * L + 1]; }
        const int64_t base = 1 + s;
        const bool small = len < kUnroll;
        const int64_t top = len - len % kUnroll;
        double acc[D], tmp[D];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        if (small) {
            if (j == 0)
                for (int64_t i = 0; i < len; ++i) {
                    vals(base + i, tmp);
#pragma unroll
                    for (int c = 0; c < D; ++c) acc[c] += tmp[c];
                }
        } else {
            vals(base + j, acc);
#pragma unroll 8
            for (int64_t i = kUnroll; i < top; i += kUnroll) {
                vals(base + i + j, tmp);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] += tmp[c];
            }
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double bsum = acc[c] + __shfl_xor_sync(kFull, acc[c], 1);
            bsum = bsum + __shfl_xor_sync(kFull, bsum, 2);
            bsum = bsum + __shfl_xor_sync(kFull, bsum, 4);
            if (!small) acc[c] = bsum;
        }
        if (!small && j == 0)
            for (int64_t i = top; i < len; ++i) {
                vals(base + i, tmp);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[c] += tmp[c];
            }
        if (L < nu && j == 0) {
#pragma unroll
            for (int c = 0; c < D; ++c) sv[c][L] = acc[c];
        }
    }
    __syncthreads();
    // The top of the tree is small (~2 nodes per leaf): warp 0 evaluates it
    // level by level with warp barriers, then thread 0 forms z with the
    // element-0 value and z weights it prefetched above.
    if (threadIdx.x < 32) {
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
        if (threadIdx.x == 0) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double zn = ddiv(a0[c] + sv[c][node - 1], zw0[c]);
                s_z[0][c] = zn;
                s_z[1][c] = zo0[c];
                b.z[zb + c] = zn;
                if (MODE == MODE_FUSED && !finite(zn)) flag_error(b.ctrl, it, FG_PHASE_Z, false);
            }
        }
    }
    __syncthreads();
    if (MODE == MODE_FUSED) {
        double zn[D], dz[D];
#pragma unroll
        for (int c = 0; c < D; ++c) { zn[c] = s_z[0][c]; dz[c] = zn[c] - s_z[1][c]; }
        double pp = 0.0, dd = 0.0;
        // batches of kUB elements per thread: all loads of a batch are issued
        // before its stores (the compiler cannot prove uout aliases nothing
        // read here), one memory round trip per batch
        constexpr int kUB = D == 1 ? 4 : 2;
        for (int64_t e0 = threadIdx.x; e0 < deg; e0 += kUB * NT) {
            double xr[kUB][D], ur[kUB][D], rr[kUB], ar[kUB];
#pragma unroll
            for (int k = 0; k < kUB; ++k) {
                const int64_t e = e0 + (int64_t)k * NT;
                if (e < deg) {
                    rr[k] = UNIT ? (e == xe.rank ? xe.rho : 1.0) : b.rho[eb + e];
                    ar[k] = UNIT ? (e == xe.rank ? xe.alpha : 1.0) : b.alpha[eb + e];
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        xr[k][c] = b.x[pb + e * D + c];
                        ur[k][c] = b.uin[pb + e * D + c];
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kUB; ++k) {
                const int64_t e = e0 + (int64_t)k * NT;
                if (e < deg) {
#pragma unroll
                    for (int c = 0; c < D; ++c) {
                        const double t = xr[k][c] - zn[c];
                        pp += t * t;
                        const double rd = rr[k] * dz[c];
                        dd += rd * rd;
                        const double un = ur[k][c] + t * ar[k];
                        b.uout[pb + e * D + c] = un;
                        bu |= !finite(un);
                    }
                }
            }
        }
        if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
        if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
        block_sum2<NT>(pp, dd, sm);
        if (threadIdx.x == 0) {
            b.part[2 * (part_off + blockIdx.x)] = pp;
            b.part[2 * (part_off + blockIdx.x) + 1] = dd;
        }
    }
}

}  // namespace fg
