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

// ---------------------------------------------------------------------------
// Matrix form (uniform weights, one system; decided at every parameter
// sync).  With rho0 and rho1 the same for every factor of the group, the
// projection is one linear map of the stacked n values:
//     v = K nv,   K = I - W^-1 M^T Q diag(1/(L/rho0 + 1/rho1)) Q^T M,
// (cols x cols, built on the host in double at sync time), so the group is
// a batched matrix product: a CTA stages the n values of the <= 128 factors
// of one run block in shared memory (coalesced, contiguous per slot),
// multiplies by K (also in shared memory) with 18 independent accumulators
// per thread, and writes x back contiguously per slot.  Parity with the
// reference's LAPACK solve stays ~1e-13 relative (gated at 1e-9).
constexpr int kDynGemmF = 128;                      // factors per CTA (one run block)
constexpr int kDynGemmMaxCols = 40;

__host__ __device__ inline size_t mpc_dyn_gemm_smem(int n0, int d) {
    const size_t cols = (size_t)(n0 + d);
    return (cols * kDynGemmMaxCols + (size_t)kDynGemmF * (cols + 1) +
            (size_t)kDynGemmF * (2 * n0 + 1)) * sizeof(double);
}

template <bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads, 2) k_mpc_dyn_gemm(PassA a, GroupDev g) {
    extern __shared__ double gsm[];
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    const int n0 = g.dim[0], d = g.ip, cols = n0 + d, ld = cols + 1, ldo = 2 * n0 + 1;
    double* Ks = gsm;                                   // [cols][cols]
    double* nvs = Ks + cols * kDynGemmMaxCols;          // [F][ld]
    double* outs = nvs + kDynGemmF * ld;                // [F][2 n0 + 1]: x of both slots
    const BlockRef bk = g.blocks[blockIdx.x];
    const RunHdr h = g.runs[bk.run];
    const SlotRun* sr = g.sruns + (int64_t)bk.run * g.nslots;
    const int64_t fl0 = bk.item0 / g.tpf;               // first factor (run-local)
    const int nf = (bk.item1 - bk.item0) / g.tpf;
    bool bn = false, bx = false;
    // K stored as [c][r0][k] for row r = r0 + 2k: a thread's 20 rows of one
    // column are contiguous (16-byte loads)
    constexpr int KH = kDynGemmMaxCols / 2;
    for (int i = threadIdx.x; i < cols * cols; i += blockDim.x) {
        const int r = i / cols, c = i - r * cols;
        Ks[(c * 2 + (r & 1)) * KH + (r >> 1)] = g.kmat[i];
    }
    // stage n: factor f's slot 0 (n0 values) and slot 1 (n0 values, the
    // first d enter the projection, the rest pass through to x).  The
    // addresses are affine in the factor (run mode), and the loop holds no
    // global store, so its loads pipeline.
    const SlotRun R0 = sr[0], R1 = sr[1];
    const double* __restrict__ src = FIRST ? a.nsrc : a.uin;
    const double* __restrict__ zz = a.z;
    const int per = 2 * n0;
    for (int idx = threadIdx.x; idx < nf * per; idx += blockDim.x) {
        const int f = idx / per, c = idx - f * per;
        const int j = c < n0 ? 0 : 1, cc = c - j * n0;
        const SlotRun& RR = j ? R1 : R0;
        const int64_t fl = fl0 + f;
        const int64_t pos = RR.pos0 + fl * RR.pos_s + cc;
        double n;
        if (FIRST) {
            n = src[pos];
        } else {
            n = zz[RR.z0 + fl * RR.z_s + cc] - src[pos];
            bn |= !finite(n);
        }
        if (j == 0) nvs[f * ld + cc] = n;
        else if (cc < d) nvs[f * ld + n0 + cc] = n;
        else outs[f * ldo + n0 + cc] = n;                  // control of t+1 passes
    }
    __syncthreads();
    // out[f][r] = sum_c K[r][c] nv[f][c]: thread -> factor f, rows r0 + 2k
    {
        const int f = threadIdx.x & (kDynGemmF - 1), r0 = threadIdx.x >> 7;
        if (f < nf) {
            double acc[kDynGemmMaxCols / 2];
#pragma unroll
            for (int k = 0; k < kDynGemmMaxCols / 2; ++k) acc[k] = 0.0;
            const double* nvf = nvs + f * ld;
            // explicit fma: this form is gated at 1e-9, not bitwise, and a
            // fused multiply-add is the more accurate product-sum
            for (int c = 0; c < cols; ++c) {
                const double v = nvf[c];
                const double2* kc = reinterpret_cast<const double2*>(Ks + (c * 2 + r0) * KH);
#pragma unroll
                for (int k2 = 0; k2 < KH / 2; ++k2) {
                    const double2 kk = kc[k2];
                    acc[2 * k2] = __fma_rn(kk.x, v, acc[2 * k2]);
                    acc[2 * k2 + 1] = __fma_rn(kk.y, v, acc[2 * k2 + 1]);
                }
            }
#pragma unroll
            for (int k = 0; k < kDynGemmMaxCols / 2; ++k) {
                const int r = r0 + 2 * k;
                if (r < cols) outs[f * ldo + r] = acc[k];
            }
        }
    }
    __syncthreads();
    double* __restrict__ xo = a.x;
    for (int idx = threadIdx.x; idx < nf * per; idx += blockDim.x) {
        const int f = idx / per, c = idx - f * per;
        const int j = c < n0 ? 0 : 1, cc = c - j * n0;
        const SlotRun& RR = j ? R1 : R0;
        const double v = outs[f * ldo + c];
        xo[RR.pos0 + (fl0 + f) * RR.pos_s + cc] = v;
        bx |= !finite(v);
    }
    passa_flags<FIRST>(a, it, bn, bx);
}

}  // namespace fg
