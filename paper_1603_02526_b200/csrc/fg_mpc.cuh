// mpc_dyn edge kernel, 8 lanes per factor (operators.py:86-96, 390-404).
//
// Weighted projection of nv = [q_t, u_t, q_t1] onto {M v = 0},
// M = [I+A, B, -I] (d x cols, cols = 2d+k), W = diag(rho0 on slot 0,
// rho1 on the first d of slot 1):
//     lambda = S^-1 M nv,  S = M W^-1 M^T = G/rho0 + I/rho1,
//     v = nv - W^-1 M^T lambda,
// with G = Q L Q^T precomputed per system on the host, so
// S^-1 = Q diag(1 / (L/rho0 + 1/rho1)) Q^T (no per-factor LAPACK solve;
// parity with the reference's gesv is ~1e-13 relative, gated at 1e-9).
//
// Mapping: an aligned group of 8 lanes per factor, 32 factors per CTA
// pass.  When the group has one system its tables (M, Q, L) are staged in
// shared memory once per CTA; the factor's vectors live in shared memory
// and every lane owns rows/columns l, l+8, ...  (~1.7 kflop per factor).
#pragma once

#include "fg_edge.cuh"

namespace fg {

constexpr int kDynLanes = 8;
constexpr int kDynSlots = kEdgeThreads / kDynLanes;      // factors per CTA pass
constexpr int kDynTab = kDynMaxD * kDynMaxCols + kDynMaxD * kDynMaxD + kDynMaxD;

template <bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads) k_mpc_dyn8(PassA a, GroupDev g) {
    extern __shared__ double dyn_smem[];
    double* s_tab = dyn_smem;                                  // [tstride] if shared
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    const int n0 = g.dim[0];
    const int d = g.ip;
    const int cols = n0 + d;
    const bool shared_tab = (g.fsys == nullptr);
    double* s_nv = dyn_smem + (shared_tab ? g.tstride : 0);    // [slots][cols + 2d]
    if (shared_tab) {
        for (int i = threadIdx.x; i < g.tstride; i += blockDim.x) s_tab[i] = g.tab[i];
        __syncthreads();
    }
    const int slot = threadIdx.x / kDynLanes;
    double* nv = s_nv + slot * (cols + 2 * d);
    double* v1 = nv + cols;                                    // M nv, then lambda
    double* v2 = v1 + d;                                       // y
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int l) {               // group-uniform
        const SlotLoc s0 = locate(a.vt, g, 0, r), s1 = locate(a.vt, g, 1, r);
        const double* T = shared_tab ? s_tab : g.tab + (int64_t)g.fsys[r.f] * g.tstride;
        const double* M = T;
        const double* Q = T + d * cols;
        const double* Lam = Q + d * d;
        for (int c = l; c < cols; c += kDynLanes)
            nv[c] = (c < n0) ? nval<FIRST>(a, s0, c, bn) : nval<FIRST>(a, s1, c - n0, bn);
        const double R0 = a.rho[s0.q], R1 = a.rho[s1.q];
        __syncwarp(gmask);
        for (int q = l; q < d; q += kDynLanes) {               // M nv
            const double* Mr = M + q * cols;
            double acc = 0.0;
            for (int c = 0; c < cols; ++c) acc += Mr[c] * nv[c];
            v1[q] = acc;
        }
        __syncwarp(gmask);
        for (int i = l; i < d; i += kDynLanes) {               // y = diag Q^T (M nv)
            double acc = 0.0;
            for (int q = 0; q < d; ++q) acc += Q[q * d + i] * v1[q];
            v2[i] = ddiv(acc, ddiv(Lam[i], R0) + ddiv(1.0, R1));
        }
        __syncwarp(gmask);
        for (int q = l; q < d; q += kDynLanes) {               // lambda = Q y
            double acc = 0.0;
            for (int i = 0; i < d; ++i) acc += Q[q * d + i] * v2[i];
            v1[q] = acc;
        }
        __syncwarp(gmask);
        for (int c = l; c < cols; c += kDynLanes) {            // v = nv - W^-1 M^T lambda
            double acc = 0.0;
            for (int q = 0; q < d; ++q) acc += M[q * cols + c] * v1[q];
            const double winv = ddiv(1.0, (c < n0) ? R0 : R1);
            const double vv = nv[c] - winv * acc;
            if (c < n0) xput(a, s0.pos + c, vv, bx);
            else xput(a, s1.pos + (c - n0), vv, bx);
        }
        for (int c = d + l; c < n0; c += kDynLanes)            // slot-1 control passes
            xput(a, s1.pos + c, nval<FIRST>(a, s1, c, bn), bx);
        __syncwarp(gmask);
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

inline size_t mpc_dyn8_smem(int tstride, int cols, int d, bool shared_tab) {
    return ((shared_tab ? (size_t)tstride : 0) + (size_t)kDynSlots * (cols + 2 * d)) *
           sizeof(double);
}

}  // namespace fg
