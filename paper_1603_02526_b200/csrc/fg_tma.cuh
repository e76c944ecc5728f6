// TMA bulk-copy pipelines for the streaming classes of the variable pass.
//
// A run of consecutive variables with one (dim, degree) keeps every array a
// tile needs in six CONTIGUOUS ranges: x and u (deg*d per variable), rho
// and alpha (deg per variable), z and z_weights (d per variable).  A
// persistent CTA walks its tiles through a ring of shared-memory stages;
// one elected thread arms the stage's mbarrier with the byte count and
// issues six 1-D `cp.async.bulk` copies (SASS UBLKCP) that complete on it,
// so several tiles per SM are in flight without holding registers, while
// the CTA computes the tile that has landed.  Results go out with plain
// coalesced stores (the ranges are not 16-byte aligned, and a bulk store of
// the aligned superset would overwrite neighbouring tiles).
#pragma once

#include "fg_var_fast.cuh"

namespace fg {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared, completing `bytes` on the mbarrier.
// L2 eviction-priority policies for bulk copies (createpolicy)
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}

// bulk copy with an L2 cache hint (data a CTA reads again soon: evict_last;
// read for the last time: evict_first)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes,
                                              uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// A tile: `nv` consecutive variables of one small run starting at v0 (run-local).
struct STile { int32_t run, v0, nv, pad; };

// Aligned span [lo, hi) of doubles covering [a, b): 16-byte granularity.
struct Span { int64_t lo, n; int off; };
__device__ __forceinline__ Span span16(int64_t a, int64_t b) {
    Span s;
    s.lo = a & ~int64_t(1);
    const int64_t hi = (b + 1) & ~int64_t(1);
    s.n = hi - s.lo;
    s.off = (int)(a - s.lo);
    return s;
}

constexpr int kTmaThreads = 256;
constexpr int kTmaStages = 4;

// Fused variable pass (phases m, z, u + residual partials) for class S.
// Layout of a stage (doubles): x | u | rho | alpha | z | zw, each span
// rounded to 16 bytes; `stage_doubles` is the host-computed maximum.
__global__ void __launch_bounds__(kTmaThreads) k_var_small_tma(
    PassB b, const SRun* runs, const STile* tiles, int32_t ntiles, int32_t stage_doubles,
    int64_t part_off) {
    extern __shared__ __align__(16) double tma_smem[];
    __shared__ __align__(8) uint64_t full[kTmaStages];
    __shared__ double sm[2 * (kTmaThreads / 32)];
    if (b.ctrl->stop) return;                      // uniform
    const int64_t it = b.ctrl->iter;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // issue the six copies of tile t into stage s (one thread)
    auto issue = [&](int t, int s) {
        const STile T = tiles[t];
        const SRun R = runs[T.run];
        const int64_t pe = (int64_t)R.deg * R.d;
        const Span sx = span16(R.pb0 + (int64_t)T.v0 * pe, R.pb0 + (int64_t)(T.v0 + T.nv) * pe);
        const Span se = span16(R.eb0 + (int64_t)T.v0 * R.deg, R.eb0 + (int64_t)(T.v0 + T.nv) * R.deg);
        const Span sz = span16(R.zb0 + (int64_t)T.v0 * R.d, R.zb0 + (int64_t)(T.v0 + T.nv) * R.d);
        double* base = tma_smem + (int64_t)s * stage_doubles;
        const unsigned bx = (unsigned)(sx.n * 8), be = (unsigned)(se.n * 8), bz = (unsigned)(sz.n * 8);
        mbar_expect_tx(&full[s], 2 * bx + 2 * be + 2 * bz);
        double* p = base;
        bulk_g2s(p, b.x + sx.lo, bx, &full[s]);     p += sx.n;
        bulk_g2s(p, b.uin + sx.lo, bx, &full[s]);   p += sx.n;
        bulk_g2s(p, b.rho + se.lo, be, &full[s]);   p += se.n;
        bulk_g2s(p, b.alpha + se.lo, be, &full[s]); p += se.n;
        bulk_g2s(p, b.zin + sz.lo, bz, &full[s]);     p += sz.n;
        bulk_g2s(p, b.zw + sz.lo, bz, &full[s]);
    };

    int n_mine = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) ++n_mine;
    if (threadIdx.x == 0)
        for (int k = 0; k < kTmaStages && k < n_mine; ++k)
            issue(blockIdx.x + k * gridDim.x, k);

    double pp = 0.0, dd = 0.0;
    bool bm = false, bz_ = false, bu = false;
    for (int k = 0; k < n_mine; ++k) {
        const int t = blockIdx.x + k * gridDim.x;
        const int s = k % kTmaStages;
        mbar_wait(&full[s], (unsigned)((k / kTmaStages) & 1));
        const STile T = tiles[t];
        const SRun R = runs[T.run];
        const int d = R.d, deg = R.deg;
        const int64_t pe = (int64_t)deg * d;
        const Span sx = span16(R.pb0 + (int64_t)T.v0 * pe, R.pb0 + (int64_t)(T.v0 + T.nv) * pe);
        const Span se = span16(R.eb0 + (int64_t)T.v0 * deg, R.eb0 + (int64_t)(T.v0 + T.nv) * deg);
        const Span sz = span16(R.zb0 + (int64_t)T.v0 * d, R.zb0 + (int64_t)(T.v0 + T.nv) * d);
        const double* base = tma_smem + (int64_t)s * stage_doubles;
        const double* X = base + sx.off;
        const double* U = base + sx.n + sx.off;
        const double* RH = base + 2 * sx.n + se.off;
        const double* AL = base + 2 * sx.n + se.n + se.off;
        const double* ZO = base + 2 * sx.n + 2 * se.n + sz.off;
        const double* ZW = base + 2 * sx.n + 2 * se.n + sz.n + sz.off;
        const int comps = T.nv * d;
        for (int q = threadIdx.x; q < comps; q += kTmaThreads) {
            const int vl = q / d, c = q - vl * d;
            const int64_t pl = (int64_t)vl * pe + c;          // tile-local payload
            const int64_t el = (int64_t)vl * deg;             // tile-local edge
            auto val = [&](int64_t e) {
                const double m = X[pl + e * d] + U[pl + e * d];   // phase m
                bm |= !finite(m);
                return m * RH[el + e];                            // engine.py:278
            };
            double S = val(0);                                    // reduceat a[0]
            if (deg > 1) S = S + leaf_seq(val, 1, deg - 1);
            const double zn = ddiv(S, ZW[q]);
            const double zo = ZO[q];
            const int64_t kz = R.zb0 + (int64_t)T.v0 * d + q;
            b.z[kz] = zn;
            bz_ |= !finite(zn);
            const double dz = zn - zo;
            const int64_t pg = R.pb0 + (int64_t)T.v0 * pe + pl;  // global payload
            for (int e = 0; e < deg; ++e) {
                const double t2 = X[pl + e * d] - zn;
                pp += t2 * t2;
                const double rd = RH[el + e] * dz;
                dd += rd * rd;
                const double un = U[pl + e * d] + t2 * AL[el + e];
                b.uout[pg + (int64_t)e * d] = un;
                bu |= !finite(un);
            }
        }
        __syncthreads();                       // stage s fully consumed
        if (threadIdx.x == 0 && k + kTmaStages < n_mine)
            issue(blockIdx.x + (k + kTmaStages) * gridDim.x, s);
    }
    if (bm) flag_error(b.ctrl, it, FG_PHASE_M, false);
    if (bz_) flag_error(b.ctrl, it, FG_PHASE_Z, false);
    if (bu) flag_error(b.ctrl, it, FG_PHASE_U, false);
    block_sum2<kTmaThreads>(pp, dd, sm);
    if (threadIdx.x == 0) {
        b.part[2 * (part_off + blockIdx.x)] = pp;
        b.part[2 * (part_off + blockIdx.x) + 1] = dd;
    }
}

}  // namespace fg
