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
    // partitioned plans: w_0 is a cut variable (its x goes to memory for the
    // cut exchange instead of a local z update), and w_{n-1}'s equality
    // partner is the next rank's first weight copy, a cut variable whose
    // single local edge follows w_{n-1}'s segment
    int32_t w0_cut, has_extra;
    int32_t st_norm, st_slack, st_margin;
    const double* fp_norm;        // per point: scale
    const double* fp_slack;       // per point: lam
    const double* fp_margin;      // per point: x (D), y
    const double* xx;             // per point: x.x (plan-time, margin order)
    const double* fnorm;          // per point: 1/(1+scale) (unit-weight form)
    const double* wtab;           // per point: 3 tables of the weighted form
};

// Weighted form with uniform weights (every rho one value r, every alpha one
// value a, so every interior w_i / xi_i z weight one value): the weights are
// kernel arguments instead of per-point lane scalars, and each division by
// a constant divisor carries its exact power-of-two inverse (0: none).
struct WUni {
    double r, a, zww, zwx;        // rho, alpha, z weight of w_i, of xi_i
    double inv2r, invr, invzww, invzwx;   // exact power-of-two inverses (0: none)
    double rcp2r, rcpr, rcpzww, rcpzwx;   // refined reciprocals qdiv_rcp (0: none)
};

// x / y for a run-constant divisor: the exact power-of-two inverse (ddivq's
// test made once per run), else the quotient from y's refined reciprocal
// computed once per run (qdiv_r), else the full inline division: bitwise
// ddivq(x, y) in every case
template <bool SC = false>
__device__ __forceinline__ double dq_c(double x, double y, double inv, double rcp) {
    if (inv != 0.0) return x * inv;
    if (rcp != 0.0) return qdiv_r<SC>(x, y, rcp);
    return qdiv<SC>(x, y);
}

// Constant-divisor mode of the uniform form (template argument CM):
// kCmAny -- power-of-two inverse when given, else the inline division;
// kCmRcp -- ... else the refined reciprocal; kCmPow2 -- every divisor has
// its power-of-two inverse (rho a power of two: z weights 4r, 2r, 2r and r
// all are), so the kernel carries no division code at these sites.
enum : int { kCmAny = 0, kCmRcp = 1, kCmPow2 = 2 };
template <int CM>
__device__ __forceinline__ double dq_m(double x, double y, double inv, double rcp) {
    if (CM == kCmPow2) return x * inv;
    return dq_c<true>(x, y, inv, CM == kCmRcp ? rcp : 0.0);
}

// refined reciprocals of the uniform form's constant divisors (one thread;
// run at parameter sync): out[k] = qdiv_rcp(y[k]) for y within qdiv_r's
// range, else 0
__global__ void k_wuni_rcp(double y0, double y1, double y2, double y3, double* out) {
    const double y[4] = {y0, y1, y2, y3};
    for (int k = 0; k < 4; ++k) {
        const int e = (int)((__double_as_longlong(y[k]) >> 52) & 0x7ff);
        out[k] = (y[k] > 0.0 && (unsigned)(e - 128) <= 1792u) ? qdiv_rcp(y[k]) : 0.0;
    }
}

constexpr int kChainThreads = 256;
#ifndef FG_CHAIN_W_MINB
#define FG_CHAIN_W_MINB 4        // CTAs/SM of the weighted form (3: 0.83 vs 0.79 ms, SVM 1M)
#endif

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

// Generic form (any D <= 32, end points): handles points ilo, ilo + istep,
// ... < ihi, spread over the grid.
template <int MINB>
__global__ void __launch_bounds__(kChainThreads, MINB) k_svm_chain(PassB b, ChainDev c,
                                                                double* xb_out,
                                                                int64_t part_off,
                                                                int32_t ilo, int32_t ihi,
                                                                int32_t istep) {
    __shared__ double sm[16];
    if (b.ctrl->stop) return;                        // uniform
    const int64_t it = b.ctrl->iter;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int D = c.D;
    const bool act = lane < D;
    const int cl = act ? lane : 0;                   // clamped component
    const int32_t npts = (ihi - ilo + istep - 1) / istep;
    const int32_t per_cta = (npts + gridDim.x - 1) / gridDim.x;
    const int32_t j0 = blockIdx.x * per_cta;
    const int32_t j1 = min(npts, j0 + per_cta);
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
    for (int32_t jj = j0 + warp; jj < j1; jj += kChainThreads / 32) {
        const int32_t i = ilo + jj * istep;
        const bool hasP = i > 0;
        const bool toExtra = c.has_extra && i == c.n - 1;   // partner: next rank's w
        const bool hasN = i + 1 < c.n || toExtra;
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
        const double un_ = hasN ? b.uin[pw + (int64_t)(toExtra ? deg : deg + 2) * D + cl] : 0.0;  // w_{i+1}'s
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
            if (hasN) sp = sb + ow + (toExtra ? deg : deg + 2); else sv = 1.0;
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
        if (toExtra && act) xb_out[pw + (int64_t)deg * D + cl] = xe;   // partner's x
        // ---- phases m, z, u of w_i (k_var_small_run<4> arithmetic) ----
        double al[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) al[k] = S(sv, kSA + k);
        const double ax0 = S(sv, kSAX0), ax1 = S(sv, kSAX1);
        if (act && c.w0_cut && i == 0) {
            // cut w_0: x goes to memory; the cut exchange finishes z and u
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < deg) xb_out[pw + (int64_t)k * D + cl] = x[k];
        } else if (act) {
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

// ---------------------------------------------------------------------------
// Weighted form: D = 32 (one lane per component) and interior points
// 1 <= i <= n-2 (degree 4: norm, margin, eq(i-1,i), eq(i,i+1)), any edge
// weights.  Same arithmetic as the generic form operation by operation,
// organised like the unit-weight form below (per-warp scalar slots in
// shared memory, 64 registers, 4 CTAs/SM):
//  * the per-point weights (rho/alpha of the point's 8 edges, the
//    neighbours' equality rho, b's margin rho, xi's z weight, w_i's z
//    weight) are one load per lane; the z weight of w_i is the same for all
//    D components (z_weights sums the per-edge rho_flat, graph.py:216-222;
//    checked at sync), so it is a per-point scalar, not a per-lane row;
//  * the iteration-invariant divisions are per-point tables built at every
//    parameter sync with the same operations (k_chain_wtab): the norm
//    factor rho0/(rho0+scale), the slack threshold lam/rho_x0 and the
//    margin denominator (x.x/rho1 + 1/rho_b) + 1/rho_x1;
//  * the three divisions of the margin multiplier mu (mu/rho1, mu/rho_b,
//    mu/rho_x1) run as ONE warp-wide division, lane k dividing by the k-th
//    weight, then shuffled back: a warp issues a division sequence once
//    whatever each lane divides;
//  * every division is the inline qdiv (fg_device.cuh), bitwise the
//    runtime's `x / y`: with the runtime's slow-path call, ptxas saved the
//    live registers around every division site.
// Six division sequences per point instead of thirteen.
enum : int {
    kWR = 0,        // lanes 0..3: rho of w_i's edges k
    kWA = 4,        // lanes 4..7: alpha of w_i's edges k
    kWRP = 8, kWRN = 9, kWY = 10, kWFN = 11, kWLR = 12, kWZX = 13, kWUX0 = 14, kWUX1 = 15,
    kWRX0 = 16, kWRX1 = 17, kWAX0 = 18, kWAX1 = 19, kWZB = 20, kWUB = 21, kWRB = 22,
    kWZWX = 23, kWDEN = 24, kWZWW = 25
};

// One interior point of the weighted form.
// The point's loads (u rows, z of w_{i-1..i+1}, margin data, the lane
// scalar) are issued together by the caller before the warp barrier, so a
// point costs one memory round trip (the lane scalar used to be a second,
// dependent one).
struct ChainWLoads {
    double u0, u1, u2, u3, up, un_, zi, zp, zn_, X;
};

template <int D>
__device__ __forceinline__ ChainWLoads chain_w_load(const PassB& b, const ChainDev& c,
                                                   int32_t i, int lane) {
    const double* __restrict__ U = b.uin + c.pW + (int64_t)(4 * i - 1) * D + lane;
    const double* __restrict__ Z = b.zin + c.zW + (int64_t)i * D + lane;
    ChainWLoads L;
    L.u0 = U[0]; L.u1 = U[D]; L.u2 = U[2 * D]; L.u3 = U[3 * D];
    L.up = U[-D]; L.un_ = U[6 * D];
    L.zi = Z[0]; L.zp = Z[-D]; L.zn_ = Z[D];
    L.X = c.fp_margin[(int64_t)i * c.st_margin + lane];
    return L;
}

template <int D, bool UNI, int CM>
__device__ __forceinline__ void chain_w_point(const PassB& b, const ChainDev& c, int32_t i,
                                              int lane, double* sc, double* su,
                                              const ChainWLoads& L, const WUni& W,
                                              double* xb_out, double& pp, double& dd,
                                              unsigned& bad) {
    // weights: kernel arguments (UNI) or the point's lane scalars
    auto WR = [&](int k) { return UNI ? W.r : sc[kWR + k]; };
    auto WA = [&](int k) { return UNI ? W.a : sc[kWA + k]; };
    auto WS = [&](int slot) { return UNI ? (slot == kWZWW ? W.zww : slot == kWZWX ? W.zwx
                                            : (slot == kWAX0 || slot == kWAX1) ? W.a : W.r)
                                         : sc[slot]; };
    const int64_t wo = c.pW + (int64_t)(4 * i - 1) * D + lane;
    const int64_t zo = c.zW + (int64_t)i * D + lane;
    double u0 = L.u0, u1 = L.u1, u2 = L.u2, u3 = L.u3;
    const double up = L.up, un_ = L.un_;
    const double zi = L.zi, zp = L.zp, zn_ = L.zn_;
    const double X = L.X;
    // u rows parked in shared memory across the divisions (registers)
    su[0] = u0; su[32] = u1; su[64] = u2; su[96] = u3;
    // ---- phase n ----
    const double n0 = zi - u0, n1 = zi - u1, n2 = zi - u2, n3 = zi - u3;
    const double np_ = zp - up, nn_ = zn_ - un_;
    const double zxi = sc[kWZX], ux0 = sc[kWUX0], ux1 = sc[kWUX1];
    const double nb = sc[kWZB] - sc[kWUB], nx0 = zxi - ux0, nx1 = zxi - ux1;
    {
        const double sn = ((n0 + n1) + (n2 + n3)) + ((np_ + nn_) + ((nb + nx0) + nx1));
        if (!finite(sn) &&
            !(finite(n0) && finite(n1) && finite(n2) && finite(n3) && finite(np_) &&
              finite(nn_) && finite(nb) && finite(nx0) && finite(nx1)))
            bad |= 1u;
    }
    // ---- phase x (equalities first: their inputs die early) ----
    double x2, x3;
    if (UNI) {                                                    // prox_equality
        x2 = dq_m<CM>(W.r * np_ + W.r * n2, W.r + W.r, W.inv2r, W.rcp2r);
        x3 = dq_m<CM>(W.r * n3 + W.r * nn_, W.r + W.r, W.inv2r, W.rcp2r);
    } else {
        x2 = ddivq<true>(sc[kWRP] * np_ + sc[kWR + 2] * n2, sc[kWRP] + sc[kWR + 2]);
        x3 = ddivq<true>(sc[kWR + 3] * n3 + sc[kWRN] * nn_, sc[kWR + 3] + sc[kWRN]);
    }
    const double x0 = sc[kWFN] * n0;                              // prox_svm_norm
    const double pr = n1 * X;
    const int g = lane & 7;
    double dot = 0.0;
    dot += __shfl_sync(kFull, pr, g);
    dot += __shfl_sync(kFull, pr, g + 8);
    dot += __shfl_sync(kFull, pr, g + 16);
    dot += __shfl_sync(kFull, pr, g + 24);
    dot += __shfl_xor_sync(kFull, dot, 1);
    dot += __shfl_xor_sync(kFull, dot, 2);
    dot += __shfl_xor_sync(kFull, dot, 4);
    const double Y = sc[kWY];
    const double slack = (1.0 - nx1) - Y * (dot + nb);
    const double mu = ddivq<true>(np_max0(slack), sc[kWDEN]);
    double x1, xbv, xx1;
    if (UNI) {                         // mu / rho: one divisor for all three
        const double q = dq_m<CM>(mu, W.r, W.invr, W.rcpr);
        x1 = n1 + (q * Y) * X;
        xbv = nb + q * Y;
        xx1 = nx1 + q;
    } else {
        // mu/rho1, mu/rho_b, mu/rho_x1 on lanes 0, 1, 2 (one division for all)
        const double q = ddivq<true>(mu, sc[lane == 1 ? kWRB : (lane == 2 ? kWRX1 : kWR + 1)]);
        x1 = n1 + (__shfl_sync(kFull, q, 0) * Y) * X;
        xbv = nb + __shfl_sync(kFull, q, 1) * Y;
        xx1 = nx1 + __shfl_sync(kFull, q, 2);
    }
    const double xx0 = np_max0(nx0 - sc[kWLR]);                  // prox_svm_slack
    // ---- phases m, z, u of w_i ----
    {
        const double r0 = WR(0), r1 = WR(1), r2 = WR(2), r3 = WR(3);
        u0 = su[0]; u1 = su[32]; u2 = su[64]; u3 = su[96];
        const double m0 = x0 + u0, m1 = x1 + u1, m2 = x2 + u2, m3 = x3 + u3;
        double res = 0.0;
        res += m1 * r1;
        res += m2 * r2;
        res += m3 * r3;
        const double zn = UNI ? dq_m<CM>(m0 * r0 + res, W.zww, W.invzww, W.rcpzww)
                              : ddivq<true>(m0 * r0 + res, sc[kWZWW]);
        b.z[zo] = zn;
        const double dz = zn - zi;
        const double t0 = x0 - zn, t1 = x1 - zn, t2 = x2 - zn, t3 = x3 - zn;
        const double v0 = u0 + t0 * WA(0), v1 = u1 + t1 * WA(1);
        const double v2 = u2 + t2 * WA(2), v3 = u3 + t3 * WA(3);
        double* __restrict__ UO = b.uout + wo;
        UO[0] = v0; UO[D] = v1; UO[2 * D] = v2; UO[3 * D] = v3;
        const double d0 = r0 * dz, d1 = r1 * dz, d2 = r2 * dz, d3 = r3 * dz;
        pp += t0 * t0; dd += d0 * d0;
        pp += t1 * t1; dd += d1 * d1;
        pp += t2 * t2; dd += d2 * d2;
        pp += t3 * t3; dd += d3 * d3;
        if (!finite((m0 + m1) + (m2 + m3))) {
            const bool mbad = !(finite(m0) && finite(m1) && finite(m2) && finite(m3));
            if (mbad && !(finite(x0) && finite(x1) && finite(x2) && finite(x3))) bad |= 2u;
            if (mbad) bad |= 4u;
        }
        if (!finite(zn)) bad |= 8u;
        if (!finite((v0 + v1) + (v2 + v3)) &&
            !(finite(v0) && finite(v1) && finite(v2) && finite(v3)))
            bad |= 16u;
    }
    // ---- xi_i (slack, margin) and b's margin x ----
    if (lane == 0) {
        const double rx0 = WS(kWRX0), R3 = WS(kWRX1);
        const double mx0 = xx0 + ux0, mx1 = xx1 + ux1;
        double rs = 0.0;
        rs += mx1 * R3;
        const double zx = UNI ? dq_m<CM>(mx0 * rx0 + rs, W.zwx, W.invzwx, W.rcpzwx)
                              : ddivq<true>(mx0 * rx0 + rs, sc[kWZWX]);
        {
            b.z[c.zX + i] = zx;
            const double dzx = zx - zxi;
            const double s0 = xx0 - zx, s1 = xx1 - zx;
            const double e0 = rx0 * dzx, e1 = R3 * dzx;
            pp += s0 * s0; dd += e0 * e0;
            pp += s1 * s1; dd += e1 * e1;
            const double w0 = ux0 + s0 * WS(kWAX0), w1 = ux1 + s1 * WS(kWAX1);
            b.uout[c.pX + 2 * (int64_t)i] = w0;
            b.uout[c.pX + 2 * (int64_t)i + 1] = w1;
            xb_out[c.pB + i] = xbv;
            if (!(finite(xbv) && finite(xx0) && finite(xx1))) bad |= 2u;
            if (!(finite(mx0) && finite(mx1))) bad |= 4u;
            if (!finite(zx)) bad |= 8u;
            if (!(finite(w0) && finite(w1))) bad |= 16u;
        }
    }
}

// CM (uniform weights): kCmPow2 when every constant divisor is a power of
// two (no division code), kCmRcp when one is not and has a refined
// reciprocal, else kCmAny (registers: 64 at the cap)
template <int D, bool UNI, int CM = kCmAny>
__global__ void __launch_bounds__(kChainThreads, FG_CHAIN_W_MINB) k_svm_chain_w(PassB b, ChainDev c,
                                                                double* xb_out,
                                                                int64_t part_off, WUni W) {
    static_assert(D == 32, "one lane per component");
    __shared__ double sm[16];
    __shared__ double s_sc[kChainThreads / 32][32];     // per-warp point scalars
    __shared__ const double* s_sb[32];                 // lane scalar: s_sb + i * s_ss
    __shared__ int32_t s_ss[32];
    __shared__ double s_u[kChainThreads / 32][4][32];   // per-warp u rows of the point
    if (b.ctrl->stop) return;
    const int64_t it = b.ctrl->iter;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t nin = c.n - 2;
    const int32_t per_cta = (nin + gridDim.x - 1) / gridDim.x;
    const int32_t i0 = 1 + blockIdx.x * per_cta;
    const int32_t i1 = min(c.n - 1, i0 + per_cta);
    // lane scalar: sb + i * ss (w_i's edges start at 4i - 1); kept in shared
    // memory, not registers (the loop body needs all 64)
    if (warp == 0) {
        const double* sb = c.xx;
        int32_t ss = 0;
        switch (lane) {
            case 0: case 1: case 2: case 3: sb = b.rho + c.eW - 1 + lane; ss = 4; break;
            case 4: case 5: case 6: case 7: sb = b.alpha + c.eW - 1 + (lane - 4); ss = 4; break;
            case kWRP: sb = b.rho + c.eW - 2; ss = 4; break;        // w_{i-1}'s eq
            case kWRN: sb = b.rho + c.eW - 1 + 6; ss = 4; break;    // w_{i+1}'s eq
            case kWY: sb = c.fp_margin + D; ss = c.st_margin; break;
            case kWFN: sb = c.wtab; ss = 1; break;
            case kWLR: sb = c.wtab + c.n; ss = 1; break;
            case kWZX: sb = b.zin + c.zX; ss = 1; break;
            case kWUX0: sb = b.uin + c.pX; ss = 2; break;
            case kWUX1: sb = b.uin + c.pX + 1; ss = 2; break;
            case kWRX0: sb = b.rho + c.eX; ss = 2; break;
            case kWRX1: sb = b.rho + c.eX + 1; ss = 2; break;
            case kWAX0: sb = b.alpha + c.eX; ss = 2; break;
            case kWAX1: sb = b.alpha + c.eX + 1; ss = 2; break;
            case kWZB: sb = b.zin + c.zB; ss = 0; break;
            case kWUB: sb = b.uin + c.pB; ss = 1; break;
            case kWRB: sb = b.rho + c.eB; ss = 1; break;
            case kWZWX: sb = b.zw + c.zX; ss = 1; break;
            case kWDEN: sb = c.wtab + 2 * (int64_t)c.n; ss = 1; break;
            case kWZWW: sb = b.zw + c.zW; ss = D; break;
            default: break;
        }
        if (UNI) {
            // the weights are kernel arguments: their lanes read one cached
            // double (stride 0) instead of streaming the per-edge arrays
            switch (lane) {
                case 0: case 1: case 2: case 3: case 4: case 5: case 6: case 7:
                case kWRP: case kWRN: case kWRX0: case kWRX1: case kWAX0: case kWAX1:
                case kWRB: case kWZWX: case kWZWW: sb = c.xx; ss = 0; break;
                default: break;
            }
        }
        s_sb[lane] = sb;
        s_ss[lane] = ss;
    }
    __syncthreads();
    double pp = 0.0, dd = 0.0;
    unsigned bad = 0;                                   // 1 n, 2 x, 4 m, 8 z, 16 u
    double* sc = s_sc[warp];
    constexpr int32_t NW = kChainThreads / 32;
#pragma unroll 1
    for (int32_t i = i0 + warp; i < i1; i += NW) {
        const ChainWLoads L = chain_w_load<D>(b, c, i, lane);
        const double sv = s_sb[lane][(int64_t)i * s_ss[lane]];
        __syncwarp();                                  // previous point's reads done
        sc[lane] = sv;
        __syncwarp();
        chain_w_point<D, UNI, CM>(b, c, i, lane, sc, &s_u[warp][0][lane], L, W, xb_out, pp, dd, bad);
    }
    if (bad & 1u) flag_error(b.ctrl, it - 1, FG_PHASE_N, true);
    if (bad & 2u) flag_error(b.ctrl, it, FG_PHASE_X, true);
    if (bad & 4u) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bad & 8u) flag_error(b.ctrl, it, FG_PHASE_Z, false);
    if (bad & 16u) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kChainThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
}

// ---------------------------------------------------------------------------
// Unit-weight form: every edge weight rho and relaxation alpha of the graph
// is exactly 1.0 and the z weights are the degrees (4 for interior w_i, 2
// for xi_i) -- checked on the host at every parameter sync.  Then each
// IEEE operation involving a weight is an exact identity (r * 1.0 == r,
// r / 1.0 == r, r / 4.0 == r * 0.25, (1*a + 1*b) / 2 == (a + b) * 0.5), so
// the kernel drops them, reads no rho/alpha/z weights, and stays bitwise
// equal to the general forms.  The norm factor 1 / (1 + scale_i) is a
// per-point table built at sync time with the same division.
enum : int { kUY = 0, kUFN = 1, kULam = 2, kUZX = 3, kUUX0 = 4, kUUX1 = 5, kUZB = 6,
             kUUB = 7, kUXX = 8 };

template <int D>
__global__ void __launch_bounds__(kChainThreads, 4) k_svm_chain_unit(PassB b, ChainDev c,
                                                                    double* xb_out,
                                                                    int64_t part_off) {
    static_assert(D == 32, "one lane per component");
    __shared__ double sm[16];
    __shared__ double s_sc[kChainThreads / 32][32];     // per-warp point scalars
    if (b.ctrl->stop) return;
    const int64_t it = b.ctrl->iter;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int32_t nin = c.n - 2;
    const int32_t per_cta = (nin + gridDim.x - 1) / gridDim.x;
    const int32_t i0 = 1 + blockIdx.x * per_cta;
    const int32_t i1 = min(c.n - 1, i0 + per_cta);
    const double* sb = c.xx;
    int32_t ss = 0;
    switch (lane) {
        case kUY: sb = c.fp_margin + D; ss = c.st_margin; break;
        case kUFN: sb = c.fnorm; ss = 1; break;
        case kULam: sb = c.fp_slack; ss = c.st_slack; break;
        case kUZX: sb = b.zin + c.zX; ss = 1; break;
        case kUUX0: sb = b.uin + c.pX; ss = 2; break;
        case kUUX1: sb = b.uin + c.pX + 1; ss = 2; break;
        case kUZB: sb = b.zin + c.zB; ss = 0; break;
        case kUUB: sb = b.uin + c.pB; ss = 1; break;
        case kUXX: sb = c.xx; ss = 1; break;
        default: break;
    }
    double pp = 0.0, dd = 0.0;
    bool bn = false, bx = false, bm = false, bz = false, bu = false;
    auto S = [&](double v, int src) { return __shfl_sync(kFull, v, src); };
    double* sc = s_sc[warp];
#pragma unroll 1
    for (int32_t i = i0 + warp; i < i1; i += kChainThreads / 32) {
        const int64_t wo = c.pW + (int64_t)(4 * i - 1) * D + lane;
        const double* __restrict__ U = b.uin + wo;
        const int64_t zo = c.zW + (int64_t)i * D + lane;
        const double* __restrict__ Z = b.zin + zo;
        const double u0 = U[0], u1 = U[D], u2 = U[2 * D], u3 = U[3 * D];
        const double up = U[-D], un_ = U[6 * D];
        const double zi = Z[0], zp = Z[-D], zn_ = Z[D];
        const double X = c.fp_margin[(int64_t)i * c.st_margin + lane];
        const double sv = sb[(int64_t)i * ss];
        __syncwarp();                                  // previous point's reads done
        sc[lane] = sv;
        __syncwarp();
        // ---- phase n ----
        const double n0 = zi - u0, n1 = zi - u1, n2 = zi - u2, n3 = zi - u3;
        const double np_ = zp - up, nn_ = zn_ - un_;
        const double zxi = sc[kUZX], ux0 = sc[kUUX0], ux1 = sc[kUUX1];
        const double nb = sc[kUZB] - sc[kUUB], nx0 = zxi - ux0, nx1 = zxi - ux1;
        // a finite sum proves every term finite (NaN and inf propagate);
        // only a non-finite sum pays for the per-value check
        const double sn = ((n0 + n1) + (n2 + n3)) + ((np_ + nn_) + ((nb + nx0) + nx1));
        if (!finite(sn))
            bn |= !(finite(n0) && finite(n1) && finite(n2) && finite(n3) && finite(np_) &&
                    finite(nn_) && finite(nb) && finite(nx0) && finite(nx1));
        // ---- phase x ----
        const double x0 = sc[kUFN] * n0;                    // prox_svm_norm
        const double pr = n1 * X;
        const int g = lane & 7;
        double dot = 0.0;
        dot += S(pr, g);
        dot += S(pr, g + 8);
        dot += S(pr, g + 16);
        dot += S(pr, g + 24);
        dot += __shfl_xor_sync(kFull, dot, 1);
        dot += __shfl_xor_sync(kFull, dot, 2);
        dot += __shfl_xor_sync(kFull, dot, 4);
        const double Y = sc[kUY];
        const double slack = (1.0 - nx1) - Y * (dot + nb);
        const double denom = (sc[kUXX] + 1.0) + 1.0;
        const double mu = ddiv(np_max0(slack), denom);
        const double x1 = n1 + (mu * Y) * X;
        const double xbv = nb + mu * Y;
        const double xx1 = nx1 + mu;
        const double xx0 = np_max0(nx0 - sc[kULam]);       // prox_svm_slack
        const double x2 = (np_ + n2) * 0.5;                    // prox_equality
        const double x3 = (n3 + nn_) * 0.5;
        // ---- phases m, z, u of w_i: z weight 4 ----
        const double m0 = x0 + u0, m1 = x1 + u1, m2 = x2 + u2, m3 = x3 + u3;
        double res = 0.0;
        res += m1;
        res += m2;
        res += m3;
        const double zn = (m0 + res) * 0.25;
        b.z[zo] = zn;
        const double dz = zn - zi;
        const double t0 = x0 - zn, t1 = x1 - zn, t2 = x2 - zn, t3 = x3 - zn;
        const double v0 = u0 + t0, v1 = u1 + t1, v2 = u2 + t2, v3 = u3 + t3;
        double* __restrict__ UO = b.uout + wo;
        UO[0] = v0; UO[D] = v1; UO[2 * D] = v2; UO[3 * D] = v3;
        pp += t0 * t0; pp += t1 * t1; pp += t2 * t2; pp += t3 * t3;
        const double dz2 = dz * dz;
        dd += dz2; dd += dz2; dd += dz2; dd += dz2;
        // x non-finite => m non-finite (u is finite: it passed last
        // iteration's check), so x is only inspected when m is bad
        if (!finite((m0 + m1) + (m2 + m3))) {
            const bool mbad = !(finite(m0) && finite(m1) && finite(m2) && finite(m3));
            if (mbad) bx |= !(finite(x0) && finite(x1) && finite(x2) && finite(x3));
            bm |= mbad;
        }
        bz |= !finite(zn);
        if (!finite((v0 + v1) + (v2 + v3)))
            bu |= !(finite(v0) && finite(v1) && finite(v2) && finite(v3));
        // ---- xi_i (slack, margin; z weight 2) and b's margin x ----
        if (lane == 0) {
            const double mx0 = xx0 + ux0, mx1 = xx1 + ux1;
            double rs = 0.0;
            rs += mx1;
            const double zx = (mx0 + rs) * 0.5;
            b.z[c.zX + i] = zx;
            const double dzx = zx - zxi;
            const double s0 = xx0 - zx, s1 = xx1 - zx;
            const double w0 = ux0 + s0, w1 = ux1 + s1;
            b.uout[c.pX + 2 * (int64_t)i] = w0;
            b.uout[c.pX + 2 * (int64_t)i + 1] = w1;
            xb_out[c.pB + i] = xbv;
            pp += s0 * s0; pp += s1 * s1;
            dd += dzx * dzx; dd += dzx * dzx;
            bx |= !(finite(xbv) && finite(xx0) && finite(xx1));
            bm |= !(finite(mx0) && finite(mx1));
            bz |= !finite(zx);
            bu |= !(finite(w0) && finite(w1));
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

// Per-point tables of the weighted form (fg_chain.cuh k_svm_chain_w), rebuilt
// at every parameter sync with the generic form's operations:
//   wtab[i]       = rho0 / (rho0 + scale_i)                 (prox_svm_norm)
//   wtab[n + i]   = lam_i / rho_x0                          (prox_svm_slack)
//   wtab[2n + i]  = (x.x / rho1 + 1 / rho_b) + 1 / rho_x1  (margin denominator)
__global__ void k_chain_wtab(ChainDev c, const double* __restrict__ rho, double* wtab) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.n || i == 0 || i == c.n - 1) return;     // interior points only
    const double* r = rho + c.eW - 1 + 4 * i;
    const double rx0 = rho[c.eX + 2 * i], rx1 = rho[c.eX + 2 * i + 1], rb = rho[c.eB + i];
    wtab[i] = ddiv(r[0], r[0] + c.fp_norm[i * c.st_norm]);
    wtab[c.n + i] = ddiv(c.fp_slack[i * c.st_slack], rx0);
    wtab[2 * c.n + i] = (ddiv(c.xx[i], r[1]) + ddiv(1.0, rb)) + ddiv(1.0, rx1);
}

// 1 / (1 + scale_i): prox_svm_norm's factor at unit edge weight
// (ddiv(R, R + scale) with R = 1.0, the same IEEE division)
__global__ void k_chain_fnorm(ChainDev c, double* fnorm) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.n) return;
    fnorm[i] = ddiv(1.0, 1.0 + c.fp_norm[i * c.st_norm]);
}

// x.x of every point's margin data in k_svm_margin's order (8-lane groups,
// lane l summing components l, l+8, l+16, l+24 from 0.0, then xor 1/2/4).
__global__ void k_chain_xx(ChainDev c, double* xx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.n) return;
    const double* P = c.fp_margin + i * c.st_margin;
    double r[8];
    for (int g = 0; g < 8; ++g) {
        double a = 0.0;
        for (int k = 0; k < 4; ++k) {
            const int cc = g + 8 * k;
            const double v = cc < c.D ? P[cc] : 0.0;
            a += v * v;
        }
        r[g] = a;
    }
    xx[i] = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

}  // namespace fg
