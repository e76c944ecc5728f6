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
    const SlotRun* sr = g.sruns + (int64_t)bk.run * g.nslots;
    const int64_t fl0 = bk.item0 / g.tpf;               // first factor (run-local)
    const int nf = (bk.item1 - bk.item0) / g.tpf;
    bool bn = false, bx = false;
    // K stored as [c][r0][k] for row r = r0 + 2k: a thread's 20 rows of one
    // column are contiguous (16-byte loads)
    constexpr int KH = kDynGemmMaxCols / 2;
    // cols a multiple of 4 (the 16/4 systems): K row-major for the f64 MMA
    const bool mma = (cols & 3) == 0;
    for (int i = threadIdx.x; i < cols * cols; i += blockDim.x) {
        const int r = i / cols, c = i - r * cols;
        if (mma) Ks[i] = g.kmat[i];
        else Ks[(c * 2 + (r & 1)) * KH + (r >> 1)] = g.kmat[i];
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
    if (mma) {
        // out^T = K . nv^T as mma.sync.m8n8k4 f64 tiles (k_mpc_block's form):
        // warp w owns the factor tiles w and w + 8; every output is the
        // same fma chain over the columns as the scalar form below (bitwise)
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, kq = lane & 3;
        const int C4 = cols >> 2;
        for (int nt = w; nt < kDynGemmF / 8; nt += kEdgeThreads / 32) {
            const int fb = 8 * nt + (lane >> 2);
            double bf[kDynGemmMaxCols / 4];
#pragma unroll
            for (int ks = 0; ks < kDynGemmMaxCols / 4; ++ks)
                bf[ks] = ks < C4 ? nvs[fb * ld + 4 * ks + kq] : 0.0;
            const int f0 = 8 * nt + 2 * kq;
            for (int m = 0; m < (cols + 7) / 8; ++m) {
                const double* ka = Ks + min(8 * m + (lane >> 2), cols - 1) * cols + kq;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < kDynGemmMaxCols / 4; ++ks) {
                    if (ks < C4) {
                        const double av = ka[4 * ks];
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                     : "+d"(d0), "+d"(d1) : "d"(av), "d"(bf[ks]));
                    }
                }
                const int r = 8 * m + (lane >> 2);
                if (r < cols) {
                    if (f0 < nf) outs[f0 * ldo + r] = d0;
                    if (f0 + 1 < nf) outs[(f0 + 1) * ldo + r] = d1;
                }
            }
        }
    } else {
    // out[f][r] = sum_c K[r][c] nv[f][c]: thread -> factor f, rows r0 + 2k
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



// ===========================================================================
// Fused MPC chain (build_mpc's graph, problems.py:200-215): one kernel per
// iteration instead of the cost, dynamics, init and variable-pass kernels.
//
// Node t (state+control, dim n0) has edges [cost_t, dyn_{t-1} slot 1,
// dyn_t slot 0] (node 0: [cost_0, dyn_0 slot 0, init], node T: [cost_T,
// dyn_{T-1} slot 1]).  A CTA owns up to kMpcTile consecutive nodes: it
// stages the n values of every dynamics factor touching them (<= 128,
// one shared with each neighbouring tile and evaluated by both with
// identical arithmetic), applies the matrix form v = K nv, then finishes
// each node from registers: cost and init proxes, m, z (NumPy's reduceat
// order), u and the residual partials.  x of the nodes never goes to
// memory (it is recomputed on download, as for the SVM chain).  Unit-weight
// form only (every rho, alpha = 1; checked at sync): the arithmetic is the
// per-kind path's operation by operation, so bitwise equal to it.
// ===========================================================================
constexpr int kMpcTile = 63;                        // nodes per CTA (<= 64 factors)
constexpr int kMpcF = kMpcTile + 1;                 // factor slots per CTA
constexpr int kMpcRG = kEdgeThreads / kMpcF;        // row groups: thread rows r0 + RG k
constexpr int kMpcKH = (kDynGemmMaxCols + kMpcRG - 1) / kMpcRG;

inline size_t mpc_chain_smem(int n0, int d) {
    const size_t cols = (size_t)(n0 + d);
    return (cols * kMpcRG * kMpcKH + (size_t)kMpcF * (cols + 1) + (size_t)kMpcF * (2 * n0 + 1)) *
           sizeof(double);
}

struct MpcChainDev {
    int32_t T, n0, d, pad;
    int64_t pN, zN;                                 // node 0 payload / z base
    int32_t eN, cost_st;                            // node 0 edge base, cost fstride
    const double* cost_fp;                          // per node: diag (n0)
    const double* init_fp;                          // q0 (d)
    const double* kmat;                             // K (cols x cols)
};

// N0/DD > 0: the state/input sizes as compile-time constants (the index
// arithmetic -- divisions by n0, 2 n0, cols -- folds to multiplies; the
// generic form divides at run time).  Same operations on the doubles.
template <bool FIRST_UNUSED = false, int N0 = 0, int DD = 0>
__global__ void __launch_bounds__(kEdgeThreads, N0 > 0 ? 4 : 3) k_mpc_chain(PassB b, MpcChainDev c,
                                                               int64_t part_off,
                                                               FusedReduce fr) {
    extern __shared__ double gsm[];
    __shared__ double sm[2 * (kEdgeThreads / 32)];
    __shared__ int s_last;
    if (b.ctrl->stop) return;
    const int64_t it = b.ctrl->iter;
    const double r3 = qdiv_rcp(3.0);                    // z = S / 3 without the runtime call
    const int n0 = N0 > 0 ? N0 : c.n0, d = N0 > 0 ? DD : c.d;
    const int cols = n0 + d, ld = cols + 1, ldo = 2 * n0 + 1;
    constexpr int KH = kMpcKH, RG = kMpcRG;
    double* Ks = gsm;                                   // [c][r0][k], row r = r0 + RG k
    double* nvs = Ks + cols * RG * KH;                  // [F][ld]
    double* outs = nvs + kMpcF * ld;                    // [F][ldo]
    const int t0 = blockIdx.x * kMpcTile;
    const int t1 = min(c.T + 1, t0 + kMpcTile);         // nodes [t0, t1)
    const int fA = max(0, t0 - 1), fB = min(c.T, t1);   // factors [fA, fB)
    const int nf = fB - fA;
    bool bn = false, bx = false, bm = false, bz = false, bu = false;
    // compile-time sizes: K row-major for the f64 MMA (fits the same space)
    for (int i = threadIdx.x; i < cols * cols; i += blockDim.x) {
        const int r = i / cols, cc = i - r * cols;
        if (N0 > 0) Ks[i] = c.kmat[i];
        else Ks[(cc * RG + r % RG) * KH + r / RG] = c.kmat[i];
    }
    const double* __restrict__ uin = b.uin;
    const double* __restrict__ zin = b.zin;
    // node t: payload pN + 3 t n0 (rank k at + k n0), z zN + t n0
    auto upos = [&](int t, int rank) { return c.pN + ((int64_t)3 * t + rank) * n0; };
    // ---- stage n of the dynamics factors: slot 0 at node f (rank 2, or 1
    // for f = 0), slot 1 at node f+1 (rank 1) ----
    const int per = 2 * n0;
    constexpr int SB = 4;                               // loads in flight per thread
    for (int base = threadIdx.x; base < nf * per; base += SB * kEdgeThreads) {
        double zv[SB], uv[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int idx = base + k * kEdgeThreads;
            zv[k] = 0.0; uv[k] = 0.0;
            if (idx < nf * per) {
                const int fl = idx / per, cc = idx - fl * per;
                const int f = fA + fl;
                const int j = cc < n0 ? 0 : 1, q = cc - j * n0;
                const int node = f + j;
                const int rank = j ? 1 : (f == 0 ? 1 : 2);
                zv[k] = zin[c.zN + (int64_t)node * n0 + q];
                uv[k] = uin[upos(node, rank) + q];
            }
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
            const int idx = base + k * kEdgeThreads;
            if (idx < nf * per) {
                const int fl = idx / per, cc = idx - fl * per;
                const int j = cc < n0 ? 0 : 1, q = cc - j * n0;
                const double n = zv[k] - uv[k];
                bn |= !finite(n);
                if (j == 0) nvs[fl * ld + q] = n;
                else if (q < d) nvs[fl * ld + n0 + q] = n;
                else outs[fl * ldo + n0 + q] = n;   // control of t+1 passes
            }
        }
    }
    __syncthreads();
    if (N0 > 0) {
        // v = K nv on the fp64 tensor cores (as k_mpc_block): warp w owns
        // factor slots 8w..8w+7, B fragments in registers, A from K; each
        // output is the same fma chain over the columns (bitwise)
        static_assert(N0 == 0 || ((N0 + DD) % 4 == 0 && kMpcF == 8 * (kEdgeThreads / 32)), "tiles");
        constexpr int C4 = N0 > 0 ? (N0 + DD) / 4 : 1;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const int fb = 8 * w + (lane >> 2), kq = lane & 3;
        double bf[C4];
#pragma unroll
        for (int ks = 0; ks < C4; ++ks) bf[ks] = nvs[fb * ld + 4 * ks + kq];
        const int f0 = 8 * w + 2 * kq;
#pragma unroll 1
        for (int m = 0; m < (4 * C4 + 7) / 8; ++m) {
            const double* ka = Ks + min(8 * m + (lane >> 2), cols - 1) * cols + kq;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < C4; ++ks) {
                const double av = ka[4 * ks];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(d0), "+d"(d1) : "d"(av), "d"(bf[ks]));
            }
            const int r = 8 * m + (lane >> 2);
            if (r < cols) {
                if (f0 < nf) outs[f0 * ldo + r] = d0;
                if (f0 + 1 < nf) outs[(f0 + 1) * ldo + r] = d1;
            }
        }
    } else {   // v = K nv: thread -> factor slot fl, rows r0 + RG k; every output is
        // the fma chain over columns 0..cols-1 of k_mpc_dyn_gemm (bitwise)
        const int fl = threadIdx.x % kMpcF, r0 = threadIdx.x / kMpcF;
        if (fl < nf) {
            double acc[KH];
#pragma unroll
            for (int k = 0; k < KH; ++k) acc[k] = 0.0;
            const double* nvf = nvs + fl * ld;
            for (int cc = 0; cc < cols; ++cc) {
                const double v = nvf[cc];
                const double2* kc = reinterpret_cast<const double2*>(Ks + (cc * RG + r0) * KH);
#pragma unroll
                for (int k2 = 0; k2 < KH / 2; ++k2) {
                    const double2 kk = kc[k2];
                    acc[2 * k2] = __fma_rn(kk.x, v, acc[2 * k2]);
                    acc[2 * k2 + 1] = __fma_rn(kk.y, v, acc[2 * k2 + 1]);
                }
            }
#pragma unroll
            for (int k = 0; k < KH; ++k) {
                const int r = r0 + RG * k;
                if (r < cols) outs[fl * ldo + r] = acc[k];
            }
        }
    }
    __syncthreads();
    // ---- nodes: cost / init proxes, m, z, u ----
    double pp = 0.0, dd = 0.0;
    const int nn = t1 - t0;
    double* __restrict__ uout = b.uout;
    double* __restrict__ zout = b.z;
    const double* __restrict__ cfp = c.cost_fp;
    constexpr int NB = 2;                               // nodes' loads in flight per thread
    for (int ib = threadIdx.x; ib < nn * n0; ib += NB * kEdgeThreads) {
      double zl[NB], ul[NB][3], dl[NB];
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const int idx = ib + k * kEdgeThreads;
        if (idx < nn * n0) {
            const int tl = idx / n0, q = idx - tl * n0;
            const int t = t0 + tl;
            zl[k] = zin[c.zN + (int64_t)t * n0 + q];
            ul[k][0] = uin[upos(t, 0) + q];
            ul[k][1] = uin[upos(t, 1) + q];
            ul[k][2] = t < c.T ? uin[upos(t, 2) + q] : 0.0;
            dl[k] = cfp[(int64_t)t * c.cost_st + q];
        }
      }
#pragma unroll
      for (int k = 0; k < NB; ++k) {
        const int idx = ib + k * kEdgeThreads;
        if (idx >= nn * n0) continue;
        const int tl = idx / n0, q = idx - tl * n0;
        const int t = t0 + tl;
        const int deg = t == c.T ? 2 : 3;
        const int64_t zo = c.zN + (int64_t)t * n0 + q;
        const double zi = zl[k];
        double u[3], x[3];
        u[0] = ul[k][0];
        u[1] = ul[k][1];
        u[2] = ul[k][2];
        // cost (rank 0): prox_mpc_cost with rho = 1
        const double n_c = zi - u[0];
        bn |= !finite(n_c);
        x[0] = prox_mpc_cost(n_c, 1.0, dl[k]);
        // rank 1: dyn_{t-1} slot 1 (node 0: dyn_0 slot 0)
        x[1] = t == 0 ? outs[(0 - fA) * ldo + q] : outs[(t - 1 - fA) * ldo + n0 + q];
        // rank 2: dyn_t slot 0 (node 0: init)
        x[2] = 0.0;
        if (deg == 3) {
            if (t == 0) {
                const double n_i = zi - u[2];
                bn |= !finite(n_i);
                x[2] = q < d ? c.init_fp[q] : n_i;
            } else {
                x[2] = outs[(t - fA) * ldo + q];
            }
        }
        bx |= !(finite(x[0]) && finite(x[1]) && (deg == 2 || finite(x[2])));
        // phases m, z, u (k_var_small_run<4> order, weights 1)
        double S = 0.0, res = 0.0;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
            if (kk < deg) {
                const double m = x[kk] + u[kk];
                bm |= !finite(m);
                if (kk == 0) S = m;
                else res += m;
            }
        }
        S = S + res;
        const double zn = deg == 3 ? qdiv_r(S, 3.0, r3) : S * 0.5;   // z weights 3 / 2
        bz |= !finite(zn);
        zout[zo] = zn;
        const double dz = zn - zi;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
            if (kk < deg) {
                const double tt = x[kk] - zn;
                pp += tt * tt;
                dd += dz * dz;
                const double un = u[kk] + tt;
                uout[upos(t, kk) + q] = un;
                bu |= !finite(un);
            }
        }
      }
    }
    if (bn) flag_error(b.ctrl, it - 1, FG_PHASE_N, true);
    if (bx) flag_error(b.ctrl, it, FG_PHASE_X, true);
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bz) flag_error(b.ctrl, it, FG_PHASE_Z, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kEdgeThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
    if (fr.counter) {                 // the last CTA runs the residual reduction
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(fr.counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            reduce_body<kEdgeThreads>(b.ctrl, b.part, fr.npart, fr.hist, fr.skip_lo, fr.skip_hi, sm);
            if (threadIdx.x == 0) *fr.counter = 0u;
        }
    }
}

}  // namespace fg
