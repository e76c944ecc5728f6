// Temporally blocked MPC chain: KB iterations of build_mpc's graph per
// launch (problems.py:200-215; the per-iteration kernel is k_mpc_chain in
// fg_mpc.cuh).
//
// The graph is a chain: one iteration of node t reads only nodes t-1, t,
// t+1 (the dynamics factors t-1 and t).  A CTA owning nodes [t0, t1) loads
// the state (z and the three u slots) of [t0-KB, t1+KB) into shared memory
// once, runs KB iterations there -- the halo shrinks by one node per side
// per iteration, so after KB iterations [t0, t1) is exact -- and writes
// its own nodes back.  HBM traffic per iteration drops KB-fold; the halo
// (2 KB nodes) is recomputed with identical arithmetic by both tiles.
//
// Every operation is k_mpc_chain's, in the same order (cost prox, the
// matrix-form dynamics v = K nv as the same fma chain, init, m, z in
// NumPy's reduceat order, u), so the state is bitwise the per-iteration
// chain's and therefore the per-kind path's.  Residual partials of the
// owned nodes are written per iteration (the last CTA turns them
// into the history rows).  Any non-finite value of an owned node stops the
// run and records the block (Ctrl::blk_err); the host then replays that
// block iteration by iteration with the ordinary kernels, which raise the
// reference's exact (iteration, phase) error.  Used without tolerances
// only (fixed iteration budgets): a tolerance stop must see every
// iteration's residuals before the next one runs.
#pragma once

#include "fg_mpc.cuh"
#include "fg_edge.cuh"

namespace fg {

#ifndef FG_MPC_KB
#define FG_MPC_KB 3
#endif
constexpr int kMpcKB = FG_MPC_KB;                      // iterations per launch (odd)
constexpr int kMpcKBTail = 3;                          // shorter block for a run's tail
constexpr int kMbF = 64;                               // factor slots
constexpr int kMbThreads = kEdgeThreads;               // 256
// v = K nv on the fp64 tensor cores: V^T (rows x factors) = K (rows x
// cols) . NV^T (cols x factors) as mma.sync.m8n8k4 f64 tiles, warp w owning
// the 8 factors 8w.. (its 9 B fragments stay in registers) and looping over
// the 5 row tiles of K (A fragments from shared memory).  The f64 MMA
// accumulates each output as the sequential fma chain over k within a
// k-step, and the k-steps run in column order, so every output is the SAME
// fma chain over the columns as k_mpc_chain / k_mpc_dyn_gemm, bit for bit
// (checked on the B200 against the scalar chain, including subnormal, inf,
// NaN and signed-zero operands: tools/probe/dmma_check.cu).  ncu: the
// scalar form was bound by shared-memory wavefronts (12 per 10 FMAs).
constexpr int kMbMT = (kDynGemmMaxCols + 7) / 8;       // row tiles of K (last one clamped)
constexpr int kMbLD = 44;                              // factor row stride: nv, then v (aliased)
constexpr int kMbNN = kMbF + 1;                        // nodes staged per CTA (tile + 2 KB)
constexpr int kMbEPT = (kMbNN * 20 + kMbThreads - 1) / kMbThreads;   // node components per thread (n0 <= 20)

// K (cols x cols), z and the three u slots of the staged nodes, and one
// factor row buffer holding nv (staging) and then v (K nv) in place: ~74 KB
// at the 16/4 sizes, three CTAs per SM
inline size_t mpc_block_smem(int n0, int d) {
    const size_t cols = (size_t)(n0 + d);
    return (cols * cols + (size_t)kMbNN * 4 * n0 + (size_t)kMbF * kMbLD) * sizeof(double);
}

// The KB iterations' residual reductions (history rows, iteration counter,
// stop) in one CTA of NT threads: every iteration's tile partials loaded in
// one pass (each accumulator sums its tiles in index order), then the block
// sums and commits back to back.
template <int NT>
__device__ void mpc_block_commit(Ctrl* c, const double* bpart, int64_t ntiles, int kb,
                                 double* hist, double* sm) {
    double a[kMpcKB], bs[kMpcKB];
#pragma unroll
    for (int k = 0; k < kMpcKB; ++k) a[k] = bs[k] = 0.0;
    for (int64_t i = threadIdx.x; i < ntiles; i += NT) {
#pragma unroll
        for (int k = 0; k < kMpcKB; ++k) {
            if (k < kb) {
                a[k] += __ldcg(bpart + 2 * ((int64_t)k * ntiles + i));
                bs[k] += __ldcg(bpart + 2 * ((int64_t)k * ntiles + i) + 1);
            }
        }
    }
    // thread 0 keeps the control block in registers across the KB commits
    CtrlIn in{};
    if (threadIdx.x == 0) in = ctrl_in(c);
#pragma unroll
    for (int k = 0; k < kMpcKB; ++k) {
        if (k < kb) {
            block_sum2<NT>(a[k], bs[k], sm);
            if (threadIdx.x == 0) {
                reduce_commit(c, in, a[k], bs[k], hist);
                ++in.it;
            }
        }
    }
}

// `counter` non-null: the last CTA to finish runs the block's reductions
// (mpc_block_commit) -- no separate reduction launch.  Every CTA that got
// past the stop check counts itself, a faulting one included, and the last
// one resets the counter; nothing is committed when a CTA stopped the run.
template <int KB, int N0, int DD>
__global__ void __launch_bounds__(kMbThreads, 3) k_mpc_block(PassB b, MpcChainDev c,
                                                             int32_t tile, double* bpart,
                                                             int64_t ntiles,
                                                             int64_t fault_it = 0,
                                                             unsigned* counter = nullptr,
                                                             double* hist = nullptr) {
    static_assert(KB % 2 == 1, "a block must flip the ping-pong slot");
    extern __shared__ double gsm[];
    if (b.ctrl->stop) return;
    constexpr int n0 = N0, d = DD, cols = N0 + DD, ld = kMbLD, ldo = kMbLD;
    static_assert(cols % 4 == 0 && cols <= 8 * kMbMT && 2 * n0 <= kMbLD && n0 <= 20, "tile sizes");
    static_assert(kMbF == 8 * (kMbThreads / 32), "one 8-factor tile per warp");
    double* Ks = gsm;                                   // [cols][cols] row-major
    double* zs = Ks + cols * cols;                      // [NN][n0]
    double* us = zs + kMbNN * n0;                       // [NN][3][n0]
    // factor rows: nv of the two slots (cols 0 .. cols-1) and the control
    // passed through to node t+1 (cols n0+d .. 2 n0-1); the MMA overwrites
    // cols 0 .. cols-1 of the warp's own rows with v = K nv after reading nv
    // into its fragments, so nv and v share the buffer
    double* nvs = us + kMbNN * 3 * n0;                  // [F][ld]
    double* outs = nvs;
    // per-iteration warp sums of the residual partials live in the unused
    // columns 2 n0 .. ld-1 of the factor rows (KB x warps x 2 doubles)
    static_assert(KB * (kMbThreads / 32) * 2 <= kMbF * (kMbLD - 2 * N0), "warp-sum slots");
    auto wsum = [&](int i, int w, int k) -> double& {
        const int f = (i * (kMbThreads / 32) + w) * 2 + k;
        constexpr int per = kMbLD - 2 * N0;
        return nvs[(f / per) * ld + 2 * n0 + f % per];
    };
    const int T = c.T;
    const int t0 = blockIdx.x * tile;
    const int t1 = min(T + 1, t0 + tile);               // owned nodes [t0, t1)
    const int a = max(0, t0 - KB);
    const int bnd = min(T + 1, t1 + KB);                // staged nodes [a, bnd)
    const int NN = bnd - a;
    const int nf = NN - 1;                              // factors [a, bnd - 1)
    // ---- stage K and the state of [a, bnd) with
    // asynchronous copies (every load in flight at once): node t's payload
    // is 3 n0 contiguous doubles at pN + 3 t n0 (node T has two slots), z
    // n0 at zN + t n0 ----
    for (int i = threadIdx.x; i < cols * cols; i += blockDim.x) {
        const int r = i / cols, cc = i - r * cols;
        cp_async8(&Ks[r * cols + cc], c.kmat + i);
    }
    {
        const double* __restrict__ uin = b.uin + c.pN + (int64_t)3 * a * n0;
        const double* __restrict__ zin = b.zin + c.zN + (int64_t)a * n0;
        const int nu = NN * 3 * n0 - (bnd == T + 1 ? n0 : 0);
        for (int i = threadIdx.x; i < nu; i += blockDim.x) cp_async8(us + i, uin + i);
        for (int i = threadIdx.x; i < NN * n0; i += blockDim.x) cp_async8(zs + i, zin + i);
        if (bnd == T + 1)
            for (int q = threadIdx.x; q < n0; q += blockDim.x) us[(NN - 1) * 3 * n0 + 2 * n0 + q] = 0.0;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int64_t it0 = b.ctrl->iter;
    const double r3 = qdiv_rcp(3.0);                    // z = S / 3 without the runtime call
    bool bad = false;
    // the cost diagonal of this thread's node components (the same ones in
    // every iteration), held in registers across the KB iterations
    double cst[kMbEPT];
#pragma unroll
    for (int jj = 0; jj < kMbEPT; ++jj) {
        const int idx = threadIdx.x + jj * kMbThreads;
        const int tl = idx / n0, q = idx - tl * n0;
        cst[jj] = idx < NN * n0 ? __ldg(c.cost_fp + (int64_t)(a + tl) * c.cost_st + q) : 0.0;
    }
    for (int i = 0; i < KB; ++i) {
        // ---- n of the dynamics factors (k_mpc_chain's staging): the first
        // iteration here, later ones written by the previous node pass ----
        if (i == 0)
        for (int idx = threadIdx.x; idx < nf * 2 * n0; idx += blockDim.x) {
            const int fl = idx / (2 * n0), cc = idx - fl * (2 * n0);
            const int f = a + fl;
            const int j = cc < n0 ? 0 : 1, q = cc - j * n0;
            const int node = fl + j;                    // local index
            const int rank = j ? 1 : (f == 0 ? 1 : 2);
            const double n = zs[node * n0 + q] - us[(node * 3 + rank) * n0 + q];
            const int tg = a + node;
            bad |= (tg >= t0 && tg < t1) && !finite(n);
            if (j == 0) nvs[fl * ld + q] = n;
            else if (q < d) nvs[fl * ld + n0 + q] = n;
            else outs[fl * ldo + n0 + q] = n;           // control of t+1 passes
        }
        __syncthreads();
        {   // v = K nv: the fma chain of k_mpc_chain / k_mpc_dyn_gemm, as f64 MMAs
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            const int fb = 8 * w + (lane >> 2), kq = lane & 3;
            double bf[cols / 4];
#pragma unroll
            for (int ks = 0; ks < cols / 4; ++ks) bf[ks] = nvs[fb * ld + 4 * ks + kq];
            // every lane's nv reads precede any lane's v writes into the
            // same (aliased) rows of this warp
            __syncwarp();
            const int f0 = 8 * w + 2 * kq;
#pragma unroll 1
            for (int m = 0; m < kMbMT; ++m) {
                // rows past cols (the last tile) reuse row cols-1: their
                // outputs are discarded and each output row depends only
                // on its own A row
                const double* ka = Ks + min(8 * m + (lane >> 2), cols - 1) * cols + kq;
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < cols / 4; ++ks) {
                    const double a = ka[4 * ks];
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(bf[ks]));
                }
                const int r = 8 * m + (lane >> 2);
                if (r < cols) {
                    if (f0 < nf) outs[f0 * ldo + r] = d0;
                    if (f0 + 1 < nf) outs[(f0 + 1) * ldo + r] = d1;
                }
            }
        }
        __syncthreads();
        // ---- nodes: cost / init proxes, m, z, u (in place) ----
        double pp = 0.0, dd = 0.0;
#pragma unroll
        for (int jj = 0; jj < kMbEPT; ++jj) {
            const int idx = threadIdx.x + jj * kMbThreads;
            if (idx >= NN * n0) break;
            const int tl = idx / n0, q = idx - tl * n0;
            const int t = a + tl;
            const bool own = t >= t0 && t < t1;
            const int deg = t == T ? 2 : 3;
            const double zi = zs[tl * n0 + q];
            double u[3], x[3];
            u[0] = us[(tl * 3 + 0) * n0 + q];
            u[1] = us[(tl * 3 + 1) * n0 + q];
            u[2] = us[(tl * 3 + 2) * n0 + q];
            const double n_c = zi - u[0];
            x[0] = prox_mpc_cost(n_c, 1.0, cst[jj]);
            bool bn = !finite(n_c);
            // rank 1: dyn_{t-1} slot 1 (node 0: dyn_0 slot 0); a halo node
            // without its factor computes a placeholder (never owned)
            if (t == 0) x[1] = outs[0 * ldo + q];
            else x[1] = tl >= 1 ? outs[(tl - 1) * ldo + n0 + q] : 0.0;
            x[2] = 0.0;
            if (deg == 3) {
                if (t == 0) {
                    const double n_i = zi - u[2];
                    bn |= !finite(n_i);
                    x[2] = q < d ? c.init_fp[q] : n_i;
                } else {
                    x[2] = tl < nf ? outs[tl * ldo + q] : 0.0;
                }
            }
            bool bb = bn || !(finite(x[0]) && finite(x[1]) && (deg == 2 || finite(x[2])));
            double S = 0.0, res = 0.0;
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                if (kk < deg) {
                    const double m = x[kk] + u[kk];
                    bb |= !finite(m);
                    if (kk == 0) S = m;
                    else res += m;
                }
            }
            S = S + res;
            const double zn = deg == 3 ? qdiv_r(S, 3.0, r3) : S * 0.5;   // z weights 3 / 2
            bb |= !finite(zn);
            zs[tl * n0 + q] = zn;
            const double dz = zn - zi;
            double un3[3];
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                un3[kk] = 0.0;
                if (kk < deg) {
                    const double tt = x[kk] - zn;
                    const double un = u[kk] + tt;
                    un3[kk] = un;
                    us[(tl * 3 + kk) * n0 + q] = un;
                    bb |= !finite(un);
                    if (own) {
                        pp += tt * tt;
                        dd += dz * dz;
                    }
                }
            }
            // the next iteration's staging of this node's dynamics slots
            // (same values the staging loop would read after the pass; each
            // factor-row position is read above and rewritten here by the
            // same thread, so the pass needs no extra barrier)
            if (i + 1 < KB) {
                if (tl < nf) {                          // slot 0 of factor tl
                    const double n = zn - un3[t == 0 ? 1 : 2];
                    bb |= !finite(n);
                    nvs[tl * ld + q] = n;
                }
                if (tl >= 1) {                          // slot 1 of factor tl-1
                    const double n = zn - un3[1];
                    bb |= !finite(n);
                    if (q < d) nvs[(tl - 1) * ld + n0 + q] = n;
                    else outs[(tl - 1) * ldo + n0 + q] = n;   // control of t+1
                }
            }
            bad |= own && bb;
        }
        // residual partials: block_sum2's warp stage now, its cross-warp
        // stage for all KB iterations after the loop (same order, one
        // barrier per iteration instead of three)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            pp += __shfl_xor_sync(kFull, pp, o);
            dd += __shfl_xor_sync(kFull, dd, o);
        }
        if ((threadIdx.x & 31) == 0) {
            wsum(i, threadIdx.x >> 5, 0) = pp;
            wsum(i, threadIdx.x >> 5, 1) = dd;
        }
        __syncthreads();                                // node pass done: next GEMM
    }
    if (threadIdx.x < 32) {
        const int l = threadIdx.x;
        for (int i = 0; i < KB; ++i) {
            double pa = l < kMbThreads / 32 ? wsum(i, l, 0) : 0.0;
            double da = l < kMbThreads / 32 ? wsum(i, l, 1) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                pa += __shfl_xor_sync(kFull, pa, o);
                da += __shfl_xor_sync(kFull, da, o);
            }
            if (l == 0) {
                bpart[2 * ((int64_t)i * ntiles + blockIdx.x)] = pa;
                bpart[2 * ((int64_t)i * ntiles + blockIdx.x) + 1] = da;
            }
        }
    }
    // fault injection for the replay test (FGADMM_MPC_BLOCK_FAULT=<iteration>)
    bad |= fault_it >= it0 && fault_it < it0 + KB;
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) {
            b.ctrl->blk_err = it0;
            b.ctrl->stop = 1;
        }
    } else {
        // ---- owned nodes back to the output slot ----
        const int lo = t0 - a, nown = t1 - t0;
        double* __restrict__ uout = b.uout + c.pN + (int64_t)3 * t0 * n0;
        double* __restrict__ zout = b.z + c.zN + (int64_t)t0 * n0;
        const int nu = nown * 3 * n0 - (t1 == T + 1 ? n0 : 0);
        for (int i = threadIdx.x; i < nu; i += blockDim.x) uout[i] = us[lo * 3 * n0 + i];
        for (int i = threadIdx.x; i < nown * n0; i += blockDim.x) zout[i] = zs[lo * n0 + i];
    }
    if (counter) {
        __shared__ int s_last;
        __shared__ double s_red[2 * (kMbThreads / 32)];
        if (threadIdx.x == 0) {
            __threadfence();                           // bpart / stop before the count
            s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (threadIdx.x == 0) *counter = 0u;
            if (!*(volatile int32_t*)&b.ctrl->stop)
                mpc_block_commit<kMbThreads>(b.ctrl, bpart, ntiles, KB, hist, s_red);
        }
    }
}

}  // namespace fg
