// Edge pass (phase n of the previous iteration + phase x) kernels.
//
// Addressing.  Slot j of factor f lives at a var-major payload position
// pos, with z offset zo and var-major edge q.  Two modes per group:
//   * runs: the group is cut on the host into maximal runs of consecutive
//     factors over which (pos, zo, q) of every slot are affine in the
//     factor index; the kernel computes addresses arithmetically.  Every
//     benchmark family is a handful of runs per group (packing: one run
//     per disk i of the i<j triangle; SVM/MPC: 1-3 runs), so the edge pass
//     reads no per-factor index at all.
//   * index: per slot (variable, rank) tables, for irregular graphs.
// Threads map to (factor, lane) with `tpf` lanes per factor: 1 (thread
// kinds), D (element-wise kinds), 32 (warp kinds).
#pragma once

#include "fg_device.cuh"

namespace fg {

struct SlotRun {
    int64_t pos0, pos_s;     // payload position: pos0 + fl * pos_s
    int64_t z0, z_s;         // z offset
    int32_t q0, q_s;         // var-major edge
};
struct RunHdr { int64_t f0, count; };
struct BlockRef { int32_t run, item0, item1, pad; };   // CTA -> run items

// Row of disk i in var-major layout: the edge of pair (i, j) is entry
// jj = j - (j > i) of the center row (2 doubles each) and radius row.
struct DiskRow {
    int64_t pbc, pbr;        // payload of entry 0 (center row, radius row)
    int64_t zc, zr;          // z offsets
    int32_t ebc, ebr;        // var-major edge of entry 0
};

struct GroupDev {
    int32_t kind, nslots;
    int32_t dim[FG_MAX_SLOTS];
    int64_t count;
    const int32_t* svar[FG_MAX_SLOTS];   // index mode: slot variable
    const int32_t* sk[FG_MAX_SLOTS];     // index mode: edge rank in variable
    const double* fp;                    // per-factor params (AoS)
    int32_t fstride, tstride;
    const double* tab;                   // shared tables (mpc_dyn)
    const int32_t* fsys;
    int32_t ip;                          // integer param (mpc_dyn: state dim)
    int32_t tpf;                         // lanes per factor
    const RunHdr* runs;                  // run mode when non-null
    const SlotRun* sruns;                // [nruns][nslots]
    const BlockRef* blocks;              // one per CTA in run mode
    int32_t nblocks, nruns;
    // all-pairs collision groups (packing): per-disk rows + tile list
    const struct DiskRow* disks;
    const int2* tiles;                   // (bi, bj), bi <= bj
    int32_t ndisks, ntiles;
    // rows affine in the disk index (every packing graph): row i = row0 +
    // i * rowS field by field, so the tile kernel computes addresses
    int32_t rows_affine, rows_even;      // rows_even: center rows 16-byte aligned
    DiskRow row0, rowS;
    // mpc_dyn matrix form (uniform weights): K (cols x cols) on the device
    const double* kmat;
    int32_t dyn_gemm;
    int32_t unit;                        // all edge weights 1 (collision tiles)
};

struct PassA {
    VarTab vt;
    const double* z;
    const double* uin;
    const double* nsrc;      // FIRST mode: materialized n (var-major)
    double* x;
    const double* rho;       // var-major edge weights
    Ctrl* ctrl;
};

struct SlotLoc {
    int64_t pos;             // first payload slot (var-major)
    int64_t zo;              // z offset of the variable
    int32_t q;               // var-major edge index
};

struct FRef {
    int64_t f;               // factor index in the group (parameter row)
    int64_t fl;              // index inside its run
    const SlotRun* sr;       // null in index mode
};

constexpr int kEdgeThreads = 256;
constexpr int kEdgeItemsPerCta = 4 * kEdgeThreads;   // run mode
constexpr int kEdgeIndexCtas = 148 * 16;             // index mode grid cap

// Calls fn(FRef, lane) for every (factor, lane) item this thread owns.
// Items advance by blockDim, so the lanes of a warp-per-factor kernel stay
// on one factor (warp-uniform loop).
template <class F>
__device__ __forceinline__ void for_each_item(const GroupDev& g, F fn) {
    const int tpf = g.tpf;
    if (g.runs) {
        const BlockRef b = g.blocks[blockIdx.x];
        const RunHdr h = g.runs[b.run];
        const SlotRun* sr = g.sruns + (int64_t)b.run * g.nslots;
        for (int32_t item = b.item0 + (int32_t)threadIdx.x; item < b.item1;
             item += (int32_t)blockDim.x) {
            const uint32_t fl = (uint32_t)item / (uint32_t)tpf;
            const int lane = item - (int32_t)(fl * tpf);
            FRef r{h.f0 + fl, (int64_t)fl, sr};
            fn(r, lane);
        }
    } else {
        const int64_t total = g.count * tpf;
        for (int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; item < total;
             item += (int64_t)gridDim.x * blockDim.x) {
            const int64_t f = item / tpf;
            FRef r{f, f, nullptr};
            fn(r, (int)(item - f * tpf));
        }
    }
}

__device__ __forceinline__ SlotLoc locate(const VarTab& vt, const GroupDev& g,
                                          int j, const FRef& r) {
    SlotLoc s;
    if (r.sr) {
        const SlotRun& R = r.sr[j];
        s.pos = R.pos0 + r.fl * R.pos_s;
        s.zo = R.z0 + r.fl * R.z_s;
        s.q = (int32_t)(R.q0 + r.fl * R.q_s);
    } else {
        const int32_t v = g.svar[j][r.f];
        const int32_t k = g.sk[j][r.f];
        s.pos = vt.pbase[v] + (int64_t)k * g.dim[j];
        s.zo = vt.zbase[v];
        s.q = vt.ebase[v] + k;
    }
    return s;
}

template <bool FIRST>
__device__ __forceinline__ double nval(const PassA& a, const SlotLoc& s, int c,
                                       bool& badn) {
    if (FIRST) return a.nsrc[s.pos + c];
    const double v = a.z[s.zo + c] - a.uin[s.pos + c];   // n = z[zmap] - u
    badn |= !finite(v);
    return v;
}

__device__ __forceinline__ void xput(const PassA& a, int64_t p, double v,
                                     bool& badx) {
    a.x[p] = v;
    badx |= !finite(v);
}

template <bool FIRST>
__device__ __forceinline__ void passa_flags(const PassA& a, int64_t it,
                                            bool badn, bool badx) {
    if (!FIRST && badn) flag_error(a.ctrl, it - 1, FG_PHASE_N, true);
    if (badx) flag_error(a.ctrl, it, FG_PHASE_X, true);
}

// ---- collision: one thread per factor (operators.py:166-191) ------------
template <bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads, 4) k_collision(PassA a, GroupDev g) {
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int) {
        const SlotLoc s0 = locate(a.vt, g, 0, r), s1 = locate(a.vt, g, 1, r);
        const SlotLoc s2 = locate(a.vt, g, 2, r), s3 = locate(a.vt, g, 3, r);
        const double n1c0 = nval<FIRST>(a, s0, 0, bn), n1c1 = nval<FIRST>(a, s0, 1, bn);
        const double n1r = nval<FIRST>(a, s1, 0, bn);
        const double n2c0 = nval<FIRST>(a, s2, 0, bn), n2c1 = nval<FIRST>(a, s2, 1, bn);
        const double n2r = nval<FIRST>(a, s3, 0, bn);
        double c10, c11, r1, c20, c21, r2;
        prox_collision(n1c0, n1c1, n1r, n2c0, n2c1, n2r, a.rho[s0.q], a.rho[s1.q],
                       a.rho[s2.q], a.rho[s3.q], c10, c11, r1, c20, c21, r2);
        xput(a, s0.pos, c10, bx); xput(a, s0.pos + 1, c11, bx);
        xput(a, s1.pos, r1, bx);
        xput(a, s2.pos, c20, bx); xput(a, s2.pos + 1, c21, bx);
        xput(a, s3.pos, r2, bx);
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

// ---- wall: one thread per factor (operators.py:226-234) ----------------
template <bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads) k_wall(PassA a, GroupDev g) {
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int) {
        const SlotLoc s0 = locate(a.vt, g, 0, r), s1 = locate(a.vt, g, 1, r);
        const double nc0 = nval<FIRST>(a, s0, 0, bn), nc1 = nval<FIRST>(a, s0, 1, bn);
        const double nr = nval<FIRST>(a, s1, 0, bn);
        const double* P = g.fp + r.f * g.fstride;   // Q0 Q1 V0 V1
        double c0, c1, rr;
        prox_wall(nc0, nc1, nr, a.rho[s0.q], a.rho[s1.q], P[0], P[1], P[2], P[3],
                  c0, c1, rr);
        xput(a, s0.pos, c0, bx); xput(a, s0.pos + 1, c1, bx);
        xput(a, s1.pos, rr, bx);
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

// ---- element-wise kinds: one thread per (factor, component) -------------
// radius (operators.py:272-277), mpc_cost (:312-314), mpc_init (:349-354),
// svm_slack (:439-441), svm_norm (:477-479), equality (:560-564),
// nan_test (fault injector).
template <int KIND, bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads) k_elementwise(PassA a, GroupDev g) {
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int c) {
        const SlotLoc s0 = locate(a.vt, g, 0, r);
        const double n = nval<FIRST>(a, s0, c, bn);
        const double* P = g.fp + r.f * g.fstride;
        double out;
        if (KIND == FG_KIND_RADIUS) {
            out = prox_radius(n, a.rho[s0.q], P[0]);
        } else if (KIND == FG_KIND_MPC_COST) {
            out = prox_mpc_cost(n, a.rho[s0.q], P[c]);
        } else if (KIND == FG_KIND_MPC_INIT) {
            out = (c < g.fstride) ? P[c] : n;
        } else if (KIND == FG_KIND_SVM_SLACK) {
            out = prox_svm_slack(n, a.rho[s0.q], P[0]);
        } else if (KIND == FG_KIND_SVM_NORM) {
            out = prox_svm_norm(n, a.rho[s0.q], P[0]);
        } else if (KIND == FG_KIND_NAN_TEST) {
            out = (P[0] != 0.0) ? __longlong_as_double(0x7ff8000000000000ll) : n;
        } else {  // FG_KIND_EQUALITY
            const SlotLoc s1 = locate(a.vt, g, 1, r);
            const double n2 = nval<FIRST>(a, s1, c, bn);
            out = prox_equality(n, n2, a.rho[s0.q], a.rho[s1.q]);
            xput(a, s1.pos + c, out, bx);
        }
        xput(a, s0.pos + c, out, bx);
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

// ---- quadratic: one thread per factor, any slots (operators.py:131-135) -
template <bool FIRST>
__global__ void __launch_bounds__(kEdgeThreads) k_quadratic(PassA a, GroupDev g) {
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int) {
        const double* P = g.fp + r.f * g.fstride;   // per slot: targets, curvature
        int off = 0;
        for (int j = 0; j < g.nslots; ++j) {
            const SlotLoc s = locate(a.vt, g, j, r);
            const double R = a.rho[s.q];
            const int d = g.dim[j];
            const double C = P[off + d];
            for (int c = 0; c < d; ++c)
                xput(a, s.pos + c, prox_quadratic(nval<FIRST>(a, s, c, bn), R, P[off + c], C), bx);
            off += d + 1;
        }
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

// ---- svm_margin: one warp per factor (operators.py:515-525) -------------
// Slots (w: D, b: 1, xi: 1); params x (D) then y.  The two D-dim dots use a
// fixed xor-tree (deterministic; parity with NumPy's einsum is 1e-9 rel).
constexpr int kMarginLanes = 8;          // lanes per factor
constexpr int kMarginMaxD = 128;
// Each factor is served by an aligned group of 8 lanes, lane l holding
// components l, l+8, ...: 4 factors per warp keep 4x more rows in flight
// than a warp per factor.  Reductions are xor butterflies inside the group
// (fixed order: deterministic).
template <bool FIRST, int CPL>
__global__ void __launch_bounds__(kEdgeThreads, 4) k_svm_margin(PassA a, GroupDev g) {
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    const int D = g.dim[0];
    const unsigned gmask = 0xFFu << (threadIdx.x & 24);
    bool bn = false, bx = false;
    for_each_item(g, [&](const FRef& r, int lane) {   // group-uniform
        const SlotLoc s0 = locate(a.vt, g, 0, r), s1 = locate(a.vt, g, 1, r);
        const SlotLoc s2 = locate(a.vt, g, 2, r);
        const double* P = g.fp + r.f * g.fstride;
        double n1[CPL], X[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int c = lane + kMarginLanes * k;
            n1[k] = 0.0; X[k] = 0.0;
            if (c < D) {
                n1[k] = nval<FIRST>(a, s0, c, bn);
                X[k] = P[c];
            }
        }
        const double n2 = nval<FIRST>(a, s1, 0, bn), n3 = nval<FIRST>(a, s2, 0, bn);
        const double R1 = a.rho[s0.q], R2 = a.rho[s1.q], R3 = a.rho[s2.q];
        const double Y = P[D];
        double dot = 0.0, xx = 0.0;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            dot += n1[k] * X[k];
            xx += X[k] * X[k];
        }
#pragma unroll
        for (int o = 1; o < kMarginLanes; o <<= 1) {
            dot += __shfl_xor_sync(gmask, dot, o);
            xx += __shfl_xor_sync(gmask, xx, o);
        }
        const double slack = (1.0 - n3) - Y * (dot + n2);
        const double denom = (ddiv(xx, R1) + ddiv(1.0, R2)) + ddiv(1.0, R3);
        const double mu = ddiv(np_max0(slack), denom);
        const double tw = ddiv(mu, R1) * Y;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
            const int c = lane + kMarginLanes * k;
            if (c < D) xput(a, s0.pos + c, n1[k] + tw * X[k], bx);
        }
        if (lane == 0) {
            xput(a, s1.pos, n2 + ddiv(mu, R2) * Y, bx);
            xput(a, s2.pos, n3 + ddiv(mu, R3), bx);
        }
    });
    passa_flags<FIRST>(a, it, bn, bx);
}

// ---- mpc_dyn limits (operators.py:86-96, 390-404; kernels in fg_mpc.cuh) --
// Weighted projection onto {M v = 0}, M = [I+A, B, -I] (d x (2d+k)).
// With W = diag(rho0 on slot 0, rho1 on the first d of slot 1),
// S = M W^-1 M^T = G/rho0 + I/rho1, G = QLQ^T precomputed per system, so
// S^-1 = Q diag(1/(L/rho0 + 1/rho1)) Q^T (replaces the per-factor LAPACK
// gesv; parity 1e-9 rel).  Table entry: M row-major, Q row-major, L.
constexpr int kDynMaxD = 32, kDynMaxCols = 96;

// ---- collision, all-pairs tiles (packing) --------------------------------
// One CTA per 32x32 tile (bi <= bj) of the i<j pair triangle.  Pair (i, j)
// has its i-half in row i at entry j-1 and its j-half in row j at entry i,
// so a tile needs 32 contiguous entries of 32 rows for each half; every
// global access is coalesced and the DRAM traffic is the algorithmic
// minimum (k_collision_tiles_v3 below).  Two earlier forms (both halves in
// shared memory; j-half only with per-row table loads) measured slower and
// were removed (profiles/r01_pack_kernel_ab.md).
constexpr int kTile = 32;
constexpr int kTP = kTile + 1;                 // padded row (bank conflicts)

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src));
}

__device__ __forceinline__ DiskRow disk_row(const GroupDev& g, int i) {
    if (!g.rows_affine) return g.disks[i];
    DiskRow R;
    R.pbc = g.row0.pbc + (int64_t)i * g.rowS.pbc;
    R.pbr = g.row0.pbr + (int64_t)i * g.rowS.pbr;
    R.zc = g.row0.zc + (int64_t)i * g.rowS.zc;
    R.zr = g.row0.zr + (int64_t)i * g.rowS.zr;
    R.ebc = g.row0.ebc + i * g.rowS.ebc;
    R.ebr = g.row0.ebr + i * g.rowS.ebr;
    return R;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}

// Variant 3 (default when the rows are affine and 16-byte aligned):
//  * no per-row table loads: row addresses are arithmetic;
//  * the j-half (row j, entries i0..i0+31) goes to shared memory by
//    cp.async, centers as one 16-byte copy per pair;
//  * the i-half (row i, entries j0-1..) is loaded into registers for all
//    four rows of a thread BEFORE anything is stored (16-byte center loads),
//    and z of the tile's 64 rows is staged in shared memory, so a tile costs
//    one memory round trip;
//  * divisions by unit edge weights are skipped exactly (ddiv).
// A16: center entries 16-byte aligned (one 16-byte access per center pair);
// otherwise two 8-byte accesses.
// UNIT: every collision edge weight is exactly 1 (checked at sync): no
// weight loads, and the prox's weight arithmetic is the exact identity
// (1/1 = 1, mu/4 = mu*0.25, mu/1 = mu), bitwise the general form.
template <bool FIRST, bool A16, bool UNIT = false>
__global__ void __launch_bounds__(kEdgeThreads, UNIT ? 4 : 3) k_collision_tiles_v3(PassA a, GroupDev g) {
    __shared__ double2 s_c[kTile][kTile + 1];       // [jl][il]: j-half centers
    __shared__ double s_r[kTile][kTP], s_rc[kTile][kTP], s_rr[kTile][kTP];
    __shared__ double s_z[2][kTile][3];             // z of rows i0.. and j0..
    if (a.ctrl->stop) return;
    const int64_t it = a.ctrl->iter;
    const int2 t = g.tiles[blockIdx.x];
    const int i0 = t.x * kTile, j0 = t.y * kTile;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int N = g.ndisks;
    const double* __restrict__ src = FIRST ? a.nsrc : a.uin;
    const double* __restrict__ rho = a.rho;
    double* __restrict__ xo = a.x;
    bool bn = false, bx = false;
#pragma unroll
    for (int k = 0; k < kTile / 8; ++k) {
        const int jl = w + 8 * k, j = j0 + jl, i = i0 + l;
        if (j < N && i < j) {
            const DiskRow R = disk_row(g, j);
            if (A16) {
                cp_async16(&s_c[jl][l], src + R.pbc + 2 * (int64_t)i);
            } else {
                cp_async8(&s_c[jl][l].x, src + R.pbc + 2 * (int64_t)i);
                cp_async8(&s_c[jl][l].y, src + R.pbc + 2 * (int64_t)i + 1);
            }
            cp_async8(&s_r[jl][l], src + R.pbr + i);
            if (!UNIT) {
                cp_async8(&s_rc[jl][l], rho + R.ebc + i);
                cp_async8(&s_rr[jl][l], rho + R.ebr + i);
            }
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
    if (!FIRST && threadIdx.x < 2 * kTile) {
        const int h = threadIdx.x >> 5, r = (h ? j0 : i0) + l;
        if (r < N) {
            const DiskRow R = disk_row(g, r);
            s_z[h][l][0] = a.z[R.zc];
            s_z[h][l][1] = a.z[R.zc + 1];
            s_z[h][l][2] = a.z[R.zr];
        }
    }
    double2 nc[kTile / 8];
    double nr[kTile / 8], rc1[kTile / 8], rr1[kTile / 8];
#pragma unroll
    for (int k = 0; k < kTile / 8; ++k) {
        const int i = i0 + w + 8 * k, j = j0 + l;
        nc[k] = make_double2(0.0, 0.0); nr[k] = 0.0; rc1[k] = 1.0; rr1[k] = 1.0;
        if (i < N && j < N && i < j) {
            const DiskRow R = disk_row(g, i);
            const int64_t e = j - 1;
            if (A16) nc[k] = *reinterpret_cast<const double2*>(src + R.pbc + 2 * e);
            else nc[k] = make_double2(src[R.pbc + 2 * e], src[R.pbc + 2 * e + 1]);
            nr[k] = src[R.pbr + e];
            if (!UNIT) {
                rc1[k] = rho[R.ebc + e];
                rr1[k] = rho[R.ebr + e];
            }
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTile / 8; ++k) {
        const int il = w + 8 * k, i = i0 + il, j = j0 + l;
        if (i < N && j < N && i < j) {
            double n1c0 = nc[k].x, n1c1 = nc[k].y, n1r = nr[k];
            const double2 c2 = s_c[l][il];
            double n2c0 = c2.x, n2c1 = c2.y, n2r = s_r[l][il];
            if (!FIRST) {   // n = z[zmap] - u  (phase n of the previous iteration)
                n1c0 = s_z[0][il][0] - n1c0; n1c1 = s_z[0][il][1] - n1c1;
                n1r = s_z[0][il][2] - n1r;
                n2c0 = s_z[1][l][0] - n2c0; n2c1 = s_z[1][l][1] - n2c1;
                n2r = s_z[1][l][2] - n2r;
                bn |= !(finite(n1c0) && finite(n1c1) && finite(n1r) && finite(n2c0) &&
                        finite(n2c1) && finite(n2r));
            }
            double c10, c11, r1, c20, c21, r2;
            if (UNIT)
                prox_collision(n1c0, n1c1, n1r, n2c0, n2c1, n2r, 1.0, 1.0, 1.0, 1.0, c10, c11,
                               r1, c20, c21, r2);
            else
                prox_collision(n1c0, n1c1, n1r, n2c0, n2c1, n2r, rc1[k], rr1[k], s_rc[l][il],
                               s_rr[l][il], c10, c11, r1, c20, c21, r2);
            const DiskRow R = disk_row(g, i);
            const int64_t e = j - 1;
            if (A16) {
                *reinterpret_cast<double2*>(xo + R.pbc + 2 * e) = make_double2(c10, c11);
            } else {
                xo[R.pbc + 2 * e] = c10;
                xo[R.pbc + 2 * e + 1] = c11;
            }
            xo[R.pbr + e] = r1;
            bx |= !(finite(c10) && finite(c11) && finite(r1));
            s_c[l][il] = make_double2(c20, c21);
            s_r[l][il] = r2;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kTile / 8; ++k) {
        const int jl = w + 8 * k, j = j0 + jl, i = i0 + l;
        if (j < N && i < j) {
            const DiskRow R = disk_row(g, j);
            const double2 c = s_c[jl][l];
            const double r = s_r[jl][l];
            if (A16) {
                *reinterpret_cast<double2*>(xo + R.pbc + 2 * (int64_t)i) = c;
            } else {
                xo[R.pbc + 2 * (int64_t)i] = c.x;
                xo[R.pbc + 2 * (int64_t)i + 1] = c.y;
            }
            xo[R.pbr + i] = r;
            bx |= !(finite(c.x) && finite(c.y) && finite(r));
        }
    }
    passa_flags<FIRST>(a, it, bn, bx);
}

// lanes per factor of each kind's kernel
__host__ __device__ inline int kind_tpf(int kind, int dim0) {
    switch (kind) {
        case FG_KIND_SVM_MARGIN: return kMarginLanes;
        case FG_KIND_MPC_DYN: return 8;          // k_mpc_dyn8 (fg_mpc.cuh)
        case FG_KIND_RADIUS: case FG_KIND_MPC_COST: case FG_KIND_MPC_INIT:
        case FG_KIND_SVM_SLACK: case FG_KIND_SVM_NORM: case FG_KIND_EQUALITY:
        case FG_KIND_NAN_TEST: return dim0;
        default: return 1;
    }
}

}  // namespace fg
