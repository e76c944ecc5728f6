// Fused SVM-chain iteration: the edge pass AND the variable pass of every
// point's weight copy w_i and slack xi_i in ONE kernel.
//
// Topology (reference problems.py:218-239, build_svm): per point i a norm
// factor on w_i, a slack factor on xi_i, a margin factor on (w_i, b, xi_i)
// and an equality factor on (w_i, w_{i+1}).  Every factor that touches w_i
// or xi_i is local to points i-1, i, i+1, so one warp per point can:
//   1. form n = z - u for all edges of its factors (phase n of the previous
//      iteration, engine.py:292-298), reading the neighbours' equality
//      edges (their u and z of the previous iteration: u and z are
//      ping-ponged, so nothing a neighbour writes is read here);
//   2. evaluate the four proxes (operators.py:439-441, 477-479, 515-525,
//      560-564) -- the equality on (w_{i-1}, w_i) and (w_i, w_{i+1}) is
//      evaluated by both neighbouring warps with identical arithmetic, and
//      an equality gives both slots the same value;
//   3. finish phases m, z, u for w_i (degree 3-4) and xi_i (degree 2) from
//      registers: x never goes to memory for these edges.
// Only the bias b (degree N) needs a global reduction: the kernel writes
// x at b's N margin edges and the ordinary giant/large kernels finish b.
//
// Per point and iteration this moves u (read+write) and z (read+write)
// once plus the point's data, instead of the two-pass schedule's separate
// x write/read and four z reads.  The arithmetic is that of the per-kind
// kernels operation by operation (same dot-product order as k_svm_margin's
// 8-lane groups, same reduceat order as k_var_small_run), so the fused path
// is bitwise equal to the generic one.
#pragma once

#include "fg_kernels.cuh"

namespace fg {

// Addresses are affine in the point index (verified on the host): w_i's
// segment starts at element offw(i) = (i ? 4i - 1 : 0) of the w block, so
// w_{i-1}'s eq(i-1, i) edge is the element right before it and w_{i+1}'s
// eq(i, i+1) edge is element offw(i) + deg_i + 2.
struct ChainDev {
    int32_t n, D;                 // points, weight dimension (<= 32)
    int64_t pW, zW, pX, zX, pB, zB;   // payload / z bases: w block, xi block, b
    int32_t eW, eX, eB, pad;          // edge bases
    int32_t st_norm, st_slack, st_margin;
    const double* fp_norm;        // per point: scale
    const double* fp_slack;       // per point: lam
    const double* fp_margin;      // per point: x (D), y
};

constexpr int kChainThreads = 256;

// Per-point scalars are spread over the lanes of the point's warp (one
// load per lane, fetched with shuffles where used) so a lane holds only its
// own component's values: low register pressure, many warps in flight.
enum : int {
    kSR = 0,        // lanes 0..3: rho of w_i's edges k
    kSA = 4,        // lanes 4..7: alpha of w_i's edges k
    kSRP = 8, kSRN = 9, kSY = 10, kSScale = 11, kSLam = 12,
    kSZX = 13, kSUX0 = 14, kSUX1 = 15, kSRX0 = 16, kSRX1 = 17, kSAX0 = 18, kSAX1 = 19,
    kSZB = 20, kSUB = 21, kSRB = 22
};

template <int MINB>
__global__ void __launch_bounds__(kChainThreads, MINB) k_svm_chain(PassB b, ChainDev c,
                                                                double* xb_out,
                                                                int64_t part_off) {
    __shared__ double sm[16];
    if (b.ctrl->stop) return;                        // uniform
    const int64_t it = b.ctrl->iter;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int D = c.D;
    const bool act = lane < D;
    const int cl = act ? lane : 0;                   // clamped component
    const int32_t per_cta = (c.n + gridDim.x - 1) / gridDim.x;
    const int32_t i0 = blockIdx.x * per_cta;
    const int32_t i1 = min(c.n, i0 + per_cta);
    double pp = 0.0, dd = 0.0;
    bool bn = false, bx = false, bm = false, bz = false, bu = false;
    auto S = [&](double v, int src) { return __shfl_sync(kFull, v, src); };
    // this lane's scalar: base pointer and per-point stride (lanes < 10
    // address w_i's edges through ow instead)
    const double* sb = nullptr;
    int64_t ss = 0;
    switch (lane) {
        case kSY: sb = c.fp_margin + D; ss = c.st_margin; break;
        case kSScale: sb = c.fp_norm; ss = c.st_norm; break;
        case kSLam: sb = c.fp_slack; ss = c.st_slack; break;
        case kSZX: sb = b.zin + c.zX; ss = 1; break;
        case kSUX0: sb = b.uin + c.pX; ss = 2; break;
        case kSUX1: sb = b.uin + c.pX + 1; ss = 2; break;
        case kSRX0: sb = b.rho + c.eX; ss = 2; break;
        case kSRX1: sb = b.rho + c.eX + 1; ss = 2; break;
        case kSAX0: sb = b.alpha + c.eX; ss = 2; break;
        case kSAX1: sb = b.alpha + c.eX + 1; ss = 2; break;
        case kSZB: sb = b.zin + c.zB; ss = 0; break;
        case kSUB: sb = b.uin + c.pB; ss = 1; break;
        case kSRB: sb = b.rho + c.eB; ss = 1; break;
        default:
            if (lane < kSA || lane == kSRP || lane == kSRN) sb = b.rho + c.eW;
            else if (lane < kSRP) sb = b.alpha + c.eW;
            break;
    }
    for (int32_t i = i0 + warp; i < i1; i += kChainThreads / 32) {
        const bool hasP = i > 0, hasN = i + 1 < c.n;
        const int32_t ow = i ? 4 * i - 1 : 0;        // first element of w_i
        const int64_t pw = c.pW + (int64_t)ow * D, zwi = c.zW + (int64_t)i * D + cl;
        const int deg = 2 + (int)hasP + (int)hasN;
        const int64_t px = c.pX + 2 * (int64_t)i;
        // ---- loads (addresses affine in i: one memory round trip) ----
        const double zi = b.zin[zwi];
        double u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = (k < deg) ? b.uin[pw + (int64_t)k * D + cl] : 0.0;
        const double up = hasP ? b.uin[pw - D + cl] : 0.0;                 // w_{i-1}'s eq
        const double zp = hasP ? b.zin[zwi - D] : 0.0;
        const double un_ = hasN ? b.uin[pw + (int64_t)(deg + 2) * D + cl] : 0.0;  // w_{i+1}'s
        const double zn_ = hasN ? b.zin[zwi + D] : 0.0;
        const double zwv = b.zw[zwi];                 // z weights (phase z)
        const double zwx = b.zw[c.zX + i];
        const double* PM = c.fp_margin + (int64_t)i * c.st_margin;
        const double X = act ? PM[lane] : 0.0;
        const double* sp = nullptr;
        double sv = 0.0;
        if (lane < kSRP) {
            const int k = lane & 3;
            if (k < deg) sp = sb + ow + k;
            else sv = (lane < kSA) ? 1.0 : 0.0;
        } else if (lane == kSRP) {
            if (hasP) sp = sb + ow - 1; else sv = 1.0;
        } else if (lane == kSRN) {
            if (hasN) sp = sb + ow + deg + 2; else sv = 1.0;
        } else if (sb) {
            sp = sb + (int64_t)i * ss;
        }
        if (sp) sv = *sp;
        // ---- phase n (previous iteration) ----
        double nv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) nv[k] = zi - u[k];
        const double np_ = zp - up, nn_ = zn_ - un_;
        const double zxi = S(sv, kSZX), ux0 = S(sv, kSUX0), ux1 = S(sv, kSUX1);
        const double nb = S(sv, kSZB) - S(sv, kSUB), nx0 = zxi - ux0, nx1 = zxi - ux1;
        if (act) {
            bool f = finite(nv[0]) && finite(nv[1]);
            if (deg > 2) f = f && finite(nv[2]);
            if (deg > 3) f = f && finite(nv[3]);
            if (hasP) f = f && finite(np_);
            if (hasN) f = f && finite(nn_);
            bn |= !f;
        }
        bn |= !(finite(nb) && finite(nx0) && finite(nx1));
        // ---- phase x ----
        double rho[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) rho[k] = S(sv, kSR + k);
        double x[4];
        x[0] = prox_svm_norm(nv[0], rho[0], S(sv, kSScale));
        // margin: k_svm_margin's order -- lane l of an 8-lane group sums
        // components l, l+8, l+16, l+24 from 0.0, then a xor-1/2/4 butterfly
        const double n1 = act ? nv[1] : 0.0;
        const double pr = n1 * X, xq = X * X;
        const int g = lane & 7;
        double dot = 0.0, xx = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            dot += S(pr, g + 8 * k);
            xx += S(xq, g + 8 * k);
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            dot += __shfl_xor_sync(kFull, dot, o);
            xx += __shfl_xor_sync(kFull, xx, o);
        }
        const double Y = S(sv, kSY), rb = S(sv, kSRB);
        const double R1 = rho[1], R3 = S(sv, kSRX1), rx0 = S(sv, kSRX0);
        const double slack = (1.0 - nx1) - Y * (dot + nb);
        const double denom = (ddiv(xx, R1) + ddiv(1.0, rb)) + ddiv(1.0, R3);
        const double mu = ddiv(np_max0(slack), denom);
        const double tw = ddiv(mu, R1) * Y;
        x[1] = n1 + tw * X;
        const double xbv = nb + ddiv(mu, rb) * Y;
        const double xx1 = nx1 + ddiv(mu, R3);
        const double xx0 = prox_svm_slack(nx0, rx0, S(sv, kSLam));
        // eq(i, i+1) sits at rank 3 after eq(i-1, i), else at rank 2
        const double rp = S(sv, kSRP), rn = S(sv, kSRN);
        const double nvN = hasP ? nv[3] : nv[2], rhoN = hasP ? rho[3] : rho[2];
        const double xe = hasN ? prox_equality(nvN, nn_, rhoN, rn) : 0.0;
        const double xp = hasP ? prox_equality(np_, nv[2], rp, rho[2]) : 0.0;
        x[2] = hasP ? xp : xe;
        x[3] = hasP ? xe : 0.0;
        if (act) {
            bool f = finite(x[0]) && finite(x[1]);
            if (deg > 2) f = f && finite(x[2]);
            if (deg > 3) f = f && finite(x[3]);
            bx |= !f;
        }
        bx |= !(finite(xbv) && finite(xx0) && finite(xx1));
        // ---- phases m, z, u of w_i (k_var_small_run<4> arithmetic) ----
        double al[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) al[k] = S(sv, kSA + k);
        const double ax0 = S(sv, kSAX0), ax1 = S(sv, kSAX1);
        if (act) {
            double Ssum = 0.0, res = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < deg) {
                    const double m = x[k] + u[k];
                    bm |= !finite(m);
                    const double v = m * rho[k];
                    if (k == 0) Ssum = v;
                    else res += v;
                }
            }
            Ssum = Ssum + res;
            const double zn = ddiv(Ssum, zwv);
            bz |= !finite(zn);
            b.z[zwi] = zn;
            const double dz = zn - zi;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (k < deg) {
                    const double t = x[k] - zn;
                    pp += t * t;
                    const double rd = rho[k] * dz;
                    dd += rd * rd;
                    const double un = u[k] + t * al[k];
                    b.uout[pw + (int64_t)k * D + cl] = un;
                    bu |= !finite(un);
                }
            }
        }
        // ---- phases m, z, u of xi_i (degree 2: slack, margin) ----
        if (lane == 0) {
            const int64_t zx = c.zX + i;
            const double m0 = xx0 + ux0, m1 = xx1 + ux1;
            bm |= !(finite(m0) && finite(m1));
            double Ssum = m0 * rx0;
            double res = 0.0;
            res += m1 * R3;
            Ssum = Ssum + res;
            const double zn = ddiv(Ssum, zwx);
            bz |= !finite(zn);
            b.z[zx] = zn;
            const double dz = zn - zxi;
            const double t0 = xx0 - zn, t1 = xx1 - zn;
            pp += t0 * t0;
            const double rd0 = rx0 * dz;
            dd += rd0 * rd0;
            pp += t1 * t1;
            const double rd1 = R3 * dz;
            dd += rd1 * rd1;
            const double v0 = ux0 + t0 * ax0, v1 = ux1 + t1 * ax1;
            b.uout[px] = v0;
            b.uout[px + 1] = v1;
            bu |= !(finite(v0) && finite(v1));
            xb_out[c.pB + i] = xbv;
        }
    }
    if (bn) flag_error(b.ctrl, it - 1, FG_PHASE_N, true);
    if (bx) flag_error(b.ctrl, it, FG_PHASE_X, true);
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bz) flag_error(b.ctrl, it, FG_PHASE_Z, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kChainThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
}

}  // namespace fg
